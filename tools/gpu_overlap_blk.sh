# Block kernel (beam 50/100) with the wide top-k beside it: parity tests + A/B.
O=gpurun_out/ovb
mkdir -p $O
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "overlapped" > $O/pytest_overlap.log 2>&1; echo "rc=$?" >> $O/pytest_overlap.log
for rep in 1 2; do for ov in 0 1; do for b in 50 100; do
  CTCB_OVERLAP=$ov timeout -s KILL 200 python bench.py --workload cfg2 --beam $b --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ov=$ov', 'beam=$b', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> $O/ab.log
done; done; done
