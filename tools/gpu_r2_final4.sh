# Final verification of the round-2 code (block-kernel overlap default): GPU suite, bench lines, shards, smoke,
# and the kernel launch list of one 8-GPU cfg4 shard (512 utterances) in precomputed mode.
O=gpurun_out/final4
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -rx > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --workload cfg2 --beam 50 --no-cpu-baseline --no-e2e > $O/bench_cfg2_b50.json 2> $O/bench_cfg2_b50.err
timeout 300 python bench.py --workload cfg2 --beam 100 --no-cpu-baseline --no-e2e > $O/bench_cfg2_b100.json 2> $O/bench_cfg2_b100.err
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
CTCB_TOPK_MODE=precomp timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_shard8.csv python tools/shard_modes.py 8 > $O/ncu_shard.log 2>&1
timeout 600 python tools/parity_full.py 2 --beam 50 > $O/parity_cfg2_b50.log 2>&1
timeout 900 python tools/parity_full.py 2 --beam 100 > $O/parity_cfg2_b100.log 2>&1
