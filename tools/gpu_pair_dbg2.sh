export CTCB_PAIR=1
timeout 120 python tools/parity_full.py 1 > gpurun_out/dbg2_cfg1.jsonl 2> gpurun_out/dbg2_cfg1.err
timeout 120 python tools/parity_full.py 2 --beam 10 > gpurun_out/dbg2_cfg2.jsonl 2> gpurun_out/dbg2_cfg2.err
timeout 300 python tools/parity_full.py 4 > gpurun_out/dbg2_cfg4.jsonl 2> gpurun_out/dbg2_cfg4.err
