# Block kernel quick loop: its GPU tests, cfg2 parity at beams 50/100, cfg2 benches.
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "block_kernel or threshold_tie" > gpurun_out/block_pytest0.log 2>&1; echo "rc=$?" >> gpurun_out/block_pytest0.log
for b in 50 100; do
  timeout 150 python tools/parity_full.py 2 --beam $b >> gpurun_out/block_par.jsonl 2>> gpurun_out/block_par.err
  timeout 150 python bench.py --workload cfg2 --beam $b --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/block_bench_b$b.json 2>/dev/null
done
