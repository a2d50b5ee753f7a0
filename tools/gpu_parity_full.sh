set -x
timeout 600 python tools/parity_full.py 4 > gpurun_out/parity_cfg4.jsonl 2> gpurun_out/parity_cfg4.err
timeout 600 python tools/parity_full.py 1 3 > gpurun_out/parity_cfg13.jsonl 2> gpurun_out/parity_cfg13.err
timeout 600 python tools/parity_full.py 2 --beam 10 > gpurun_out/parity_cfg2.jsonl 2>> gpurun_out/parity_cfg2.err
timeout 600 python tools/parity_full.py 2 --beam 1 >> gpurun_out/parity_cfg2.jsonl 2>> gpurun_out/parity_cfg2.err
timeout 600 python tools/parity_full.py 1 --mode fused >> gpurun_out/parity_cfg13.jsonl 2>> gpurun_out/parity_cfg13.err
