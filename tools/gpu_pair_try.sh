set -x
export CTCB_PAIR=1
timeout 120 python tools/parity_full.py 0 > gpurun_out/pair_cfg0.jsonl 2> gpurun_out/pair_cfg0.err
timeout 180 python tools/parity_full.py 1 > gpurun_out/pair_cfg1.jsonl 2> gpurun_out/pair_cfg1.err
timeout 300 python tools/parity_full.py 4 > gpurun_out/pair_cfg4.jsonl 2> gpurun_out/pair_cfg4.err
unset CTCB_PAIR
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/pair_bench.json 2> gpurun_out/pair_bench.err
