# Overlap sweep: top-k blocks per SM beside the walk (CTCB_OVERLAP_BPS) on cfg3 / cfg1 / shards.
O=gpurun_out/ov2
mkdir -p $O
for cfg in "CTCB_OVERLAP=0" "CTCB_OVERLAP_BPS=1" "CTCB_OVERLAP_BPS=2" "CTCB_OVERLAP_BPS=3" "CTCB_OVERLAP_BPS=8"; do
  for w in cfg3 cfg1; do
    env $cfg timeout -s KILL 200 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$w', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> $O/sweep.log
  done
  env $cfg timeout -s KILL 300 python tools/shard_modes.py 8 4 2>/dev/null | sed "s/^/$cfg /" >> $O/sweep.log
done
