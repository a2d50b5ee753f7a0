# Round 2, session 2: state of the restored tree (GPU tests, cfg4/cfg1/cfg2/cfg3 lines).
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -rx > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-validate > gpurun_out/bench_cfg4_nv.json 2> gpurun_out/bench_cfg4_nv.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 300 python bench.py --workload cfg2 --beam 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_b50.json 2> gpurun_out/bench_cfg2_b50.err
timeout 300 python bench.py --workload cfg2 --beam 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg2_b100.json 2> gpurun_out/bench_cfg2_b100.err
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
