# A/B: packed fp32x2 input screen (new2, new3 = + integer verdict) vs scalar (base2) on cfg4; validation tests.
O=gpurun_out/f2
mkdir -p $O
CTCB_LIB=variants/libctcb_new3.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "validat or invalid or headline or cfg1_full" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2 3; do for L in variants/libctcb_base2.so variants/libctcb_new2.so variants/libctcb_new3.so; do
  CTCB_LIB=$L timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" >> $O/ab.log
done; done
