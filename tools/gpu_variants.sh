# bench build variants (CTCB_LIB) on cfg4 and cfg1, plus cfg4 parity for each
for v in variants/libctcb_horner.so variants/libctcb_estrin.so; do
  echo "== $v"
  for w in cfg4 cfg1; do
    CTCB_LIB=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['ms_per_step'], d['value']/1e6, d['roofline']['frac'])"
  done
  CTCB_LIB=$v timeout 300 python tools/parity_full.py 4 2>/dev/null | cut -c1-150
done
