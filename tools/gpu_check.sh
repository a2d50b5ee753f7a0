# Quick state check on one box: GPU tests, cfg4 bench line, cfg1 / cfg3 lines, smoke.
set -x
O=gpurun_out/check
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -rx -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
