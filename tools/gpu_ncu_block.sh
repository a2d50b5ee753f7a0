timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctcb_decode_block_kernel -s 1 -c 1 \
  -o gpurun_out/ncu_block_b${BEAM:-100} -f python bench.py --workload cfg2 --beam ${BEAM:-100} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_block.log 2>&1
