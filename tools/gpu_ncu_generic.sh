# ncu --set full of the generic decode kernel on cfg2 at beam $1 (one launch)
B=${1:-100}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ctcb_decode_generic -s 1 -c 1 \
  -o gpurun_out/ncu_generic_b$B -f python bench.py --workload cfg2 --beam $B --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_generic_b$B.log 2>&1
