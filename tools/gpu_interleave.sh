# A/B: interleaved first items (CTCB_INTERLEAVE=1) vs the plain longest-first queue.
O=gpurun_out/il
mkdir -p $O
for rep in 1 2; do for il in 0 1; do
  CTCB_INTERLEAVE=$il timeout -s KILL 300 python tools/shard_modes.py 8 4 2>/dev/null | sed "s/^/il=$il /" >> $O/ab.log
  CTCB_INTERLEAVE=$il timeout -s KILL 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('il=$il cfg4', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> $O/ab.log
done; done
CTCB_INTERLEAVE=1 CTCB_TOPK_MODE=precomp timeout -s KILL 300 python tools/parity_full.py 1 3 > $O/parity_il.log 2>&1
