# Pair-kernel iteration: parity on cfg4 (all 4096 utterances), bench, one ncu capture.
set -x
timeout 300 python tools/parity_full.py 4 > gpurun_out/pair_cfg4.jsonl 2> gpurun_out/pair_cfg4.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/pair_bench.json 2> gpurun_out/pair_bench.err
if [ "${NCU:-1}" = "1" ]; then bash tools/gpu_ncu_full.sh ctcb_decode_pair_kernel cfg4; fi
