# A/B of two library builds on the same box: python bench.py lines, alternating.
# usage: bash tools/gpu_ab.sh A.so B.so [bench args]
A=$1; B=$2; shift 2
for rep in 1 2; do for L in $A $B; do
  CTCB_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab.log
done; done
