# Invalid-row regression + repeated full GPU suites (the final4 fault was intermittent).
O=gpurun_out/inv
mkdir -p $O
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "never_walk_invalid or validation" > $O/pytest_invalid.log 2>&1; echo "rc=$?" >> $O/pytest_invalid.log
for r in 1 2 3; do
  timeout -s KILL 900 python -m pytest tests -q -m gpu > $O/full_$r.log 2>&1; echo "rc=$?" >> $O/full_$r.log
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-e2e > $O/bench_cfg1.json 2> $O/bench_cfg1.err
