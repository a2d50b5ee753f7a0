# Round-2 check: GPU test suite, default bench line (cpu baselines, parity, e2e), smoke.
set -x
timeout 1200 python -m pytest tests -q -m gpu -rx > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
