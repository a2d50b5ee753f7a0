# Overlap default (V > 512 only): new parity tests, full GPU suite, cfg3 / cfg1 / cfg4 lines.
O=gpurun_out/ov3
mkdir -p $O
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k overlapped > $O/pytest_overlap.log 2>&1; echo "rc=$?" >> $O/pytest_overlap.log
timeout -s KILL 1200 python -m pytest tests -q -m gpu -rx > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for w in cfg3 cfg1; do timeout -s KILL 200 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout -s KILL 600 python bench.py > $O/bench.json 2> $O/bench.err
