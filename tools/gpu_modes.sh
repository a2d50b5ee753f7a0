# cfg4 bench in fused vs precomputed-top-k mode
for m in fused precomp; do
  CTCB_TOPK_MODE=$m timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/q_cfg4_$m.json 2> gpurun_out/q_cfg4_$m.err
done
CTCB_TOPK_MODE=precomp timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_precomp.csv python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
