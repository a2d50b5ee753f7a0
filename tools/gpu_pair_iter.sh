# Pair-kernel iteration: parity on cfg4 (all 4096 utterances) + cfg2 beams, bench, optional ncu.
export CTCB_PAIR=1
timeout 300 python tools/parity_full.py 4 > gpurun_out/pair_cfg4.jsonl 2> gpurun_out/pair_cfg4.err
timeout 300 python tools/parity_full.py 2 --beam 16 > gpurun_out/pair_cfg2.jsonl 2> gpurun_out/pair_cfg2.err
timeout 300 python tools/parity_full.py 2 --beam 3 >> gpurun_out/pair_cfg2.jsonl 2>> gpurun_out/pair_cfg2.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/pair_bench.json 2> gpurun_out/pair_bench.err
if [ "${NCU:-0}" = "1" ]; then bash tools/gpu_ncu_pair.sh; fi
