set -x
export CTCB_PAIR=1
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/parity_full.py 0 > gpurun_out/san_pair_cfg0.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/parity_full.py 1 > gpurun_out/san_pair_cfg1.log 2>&1
