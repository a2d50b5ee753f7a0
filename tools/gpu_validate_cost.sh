# Cost of the fused input validation on cfg4 / cfg1 / cfg3: A/B of bench.py with and without --no-validate.
O=gpurun_out/vcost
mkdir -p $O
for rep in 1 2 3; do for v in "" "--no-validate"; do for w in cfg4 cfg3; do
  timeout -s KILL 300 python bench.py --workload $w $v --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$w', '${v:-validate}', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> $O/ab.log
done; done; done
