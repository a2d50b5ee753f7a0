# ncu --set full of the precomputed top-k kernel on cfg4 (precomp mode forced).
CTCB_TOPK_MODE=precomp timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ctcb_topk_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_topk_cfg4 -f python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_topk_cfg4.log 2>&1
