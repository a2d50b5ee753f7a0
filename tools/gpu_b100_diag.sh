for b in 50 100; do
  timeout 600 python tools/parity_full.py 2 --beam $b > gpurun_out/diag_b$b.jsonl 2> gpurun_out/diag_b$b.err
  timeout 600 python bench.py --workload cfg2 --beam $b --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/diag_bench_b$b.json 2>/dev/null
done
