# Final bench lines after the longer pre-region spin (3 runs of the default line, cfg1).
O=gpurun_out/final7
mkdir -p $O
for r in 1 2 3; do timeout 900 python bench.py > $O/bench_$r.json 2> $O/bench_$r.err; done
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
