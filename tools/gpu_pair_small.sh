for w in cfg1 cfg2 cfg3; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/small_def_$w.json 2>/dev/null
  CTCB_PAIR=1 timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/small_pair_$w.json 2>/dev/null
done
