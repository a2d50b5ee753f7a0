O=gpurun_out/inv2
mkdir -p $O
for r in 1 2; do
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "never_walk_invalid or validation" -rf > $O/pytest_invalid_$r.log 2>&1; echo "rc=$?" >> $O/pytest_invalid_$r.log
done
