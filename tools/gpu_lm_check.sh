set -x
timeout 900 python -m pytest tests/test_lm.py tests/test_gpu_parity.py -q -m gpu -k "lm or regression" -rx > gpurun_out/pytest_lm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lm.log
timeout 600 python tools/bench_lm.py > gpurun_out/bench_lm.json 2> gpurun_out/bench_lm.err
