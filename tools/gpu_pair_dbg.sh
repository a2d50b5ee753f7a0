export CTCB_PAIR=1
timeout 120 python tools/parity_full.py 0 1 > gpurun_out/dbg_cfg01.jsonl 2> gpurun_out/dbg_cfg01.err
timeout 300 python tools/parity_full.py 4 > gpurun_out/dbg_cfg4.jsonl 2> gpurun_out/dbg_cfg4.err
timeout 300 python tools/parity_full.py 2 --beam 10 > gpurun_out/dbg_cfg2.jsonl 2> gpurun_out/dbg_cfg2.err
timeout 300 python tools/parity_full.py 2 --beam 16 >> gpurun_out/dbg_cfg2.jsonl 2>> gpurun_out/dbg_cfg2.err
timeout 300 python tools/parity_full.py 2 --beam 1 >> gpurun_out/dbg_cfg2.jsonl 2>> gpurun_out/dbg_cfg2.err
timeout 300 python tools/parity_full.py 2 --beam 3 >> gpurun_out/dbg_cfg2.jsonl 2>> gpurun_out/dbg_cfg2.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/pair_bench.json 2> gpurun_out/pair_bench.err
