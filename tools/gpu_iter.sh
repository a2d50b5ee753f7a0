# Iteration check: GPU tests, full-batch parity, fuzz, cfg4 bench line, utterance timeline.
set -x
timeout 1200 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/parity_full.py 4 1 0 > gpurun_out/parity.log 2>&1
timeout 600 python tools/parity_full.py 2 --beam 10 >> gpurun_out/parity.log 2>&1
timeout 600 python tools/fuzz_parity.py ${FUZZ_N:-300} 91 > gpurun_out/fuzz_pre.log 2>&1
CTCB_TOPK_MODE=fused timeout 600 python tools/fuzz_parity.py ${FUZZ_N:-300} 92 > gpurun_out/fuzz_fused.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
timeout 300 python tools/utt_timeline.py 4 > gpurun_out/tl4.json 2>&1
timeout 300 python tools/utt_counters.py 4 1546 2255 2480 2899 1248 1101 1731 1792 > gpurun_out/uc.log 2>&1
