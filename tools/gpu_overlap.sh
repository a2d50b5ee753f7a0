# Overlapped precomputed top-k: GPU parity suite, then A/B of CTCB_OVERLAP=0/1 on cfg1, cfg3 and the cfg4 shards.
set -x
O=gpurun_out/ov
mkdir -p $O
timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cfg1 or cfg3 or cfg0 or golden" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for ov in 1 0; do
  CTCB_OVERLAP=$ov timeout -s KILL 200 python bench.py --workload cfg1 --no-cpu-baseline --no-e2e > $O/cfg1_ov$ov.json 2> $O/cfg1_ov$ov.err
  CTCB_OVERLAP=$ov timeout -s KILL 200 python bench.py --workload cfg3 --no-cpu-baseline --no-e2e > $O/cfg3_ov$ov.json 2> $O/cfg3_ov$ov.err
  CTCB_OVERLAP=$ov timeout -s KILL 300 python tools/shard_modes.py 8 4 > $O/shards_ov$ov.log 2>&1
done
timeout -s KILL 1200 python -m pytest tests -q -m gpu -rx > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
