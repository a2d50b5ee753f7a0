# Parity of the final build: full batches (cfg4 / cfg1 / cfg3, cfg2 beams 50 / 100) and randomised decodes in both top-k modes.
O=gpurun_out/pf
mkdir -p $O
timeout 600 python tools/parity_full.py 4 1 3 > $O/parity_full.log 2>&1
timeout 600 python tools/parity_full.py 2 --beam 50 > $O/parity_cfg2_b50.log 2>&1
timeout 900 python tools/parity_full.py 2 --beam 100 > $O/parity_cfg2_b100.log 2>&1
timeout 900 python tools/fuzz_parity.py 250 501 > $O/fuzz_parity_s501.log 2>&1
CTCB_TOPK_MODE=fused timeout 900 python tools/fuzz_parity.py 250 502 > $O/fuzz_parity_fused_s502.log 2>&1
