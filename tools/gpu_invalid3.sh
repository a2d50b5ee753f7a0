O=gpurun_out/inv3
mkdir -p $O
for r in 1 2; do
timeout -s KILL 300 python -m pytest tests/test_lm.py -q -m gpu -k "invalid_rows" -rf > $O/pytest_lm_invalid_$r.log 2>&1; echo "rc=$?" >> $O/pytest_lm_invalid_$r.log
done
timeout -s KILL 300 python -m pytest tests/test_lm.py -q -m gpu > $O/pytest_lm.log 2>&1; echo "rc=$?" >> $O/pytest_lm.log
