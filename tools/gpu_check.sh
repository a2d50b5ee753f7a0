# GPU parity tests + quick bench lines (no CPU baseline / e2e) into gpurun_out/.
set -x
make -s -C paper_2310_17864_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in cfg4 cfg1 cfg3; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/q_$w.json 2> gpurun_out/q_$w.err
done
for b in 10 50; do
  timeout 300 python bench.py --workload cfg2 --beam $b --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/q_cfg2_b$b.json 2> gpurun_out/q_cfg2_b$b.err
done
