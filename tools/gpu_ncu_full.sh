# One ncu --set full capture of a decode kernel on a bench workload (1 launch).
set -x
K=${1:-ctcb_decode_fast_kernel}
W=${2:-cfg4}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
  -o gpurun_out/ncu_full_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_full_$W.log 2>&1
