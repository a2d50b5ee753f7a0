set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
lscpu > gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
