# ncu --set full of one cfg4 launch of the pair kernel (forced with CTCB_PAIR=1)
export CTCB_PAIR=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctcb_decode_pair_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_pair_cfg4 -f python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_pair_cfg4.log 2>&1
