# A/B: input screen fused into the global-row top-k's first pass (new) vs a separate scalar pass (base), cfg3.
O=gpurun_out/scr
mkdir -p $O
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "overlapped or validat or cfg3" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do for L in variants/libctcb_base.so variants/libctcb_new.so; do for ov in 1 0; do
  CTCB_LIB=$L CTCB_OVERLAP=$ov timeout -s KILL 200 python bench.py --workload cfg3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L ov=$ov', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> $O/ab.log
done; done; done
timeout 600 python tools/parity_full.py 3 > $O/parity_cfg3.log 2>&1
