# Long randomised parity sweeps (fast / block / generic kernels in both top-k modes, fused LM) against the oracle.
mkdir -p gpurun_out/fuzz
timeout 1500 python tools/fuzz_parity.py 2000 201 > gpurun_out/fuzz/fuzz_parity_s201.log 2>&1
CTCB_TOPK_MODE=fused timeout 1500 python tools/fuzz_parity.py 2000 202 > gpurun_out/fuzz/fuzz_parity_fused_s202.log 2>&1
timeout 1200 python tools/fuzz_lm.py 600 203 > gpurun_out/fuzz/fuzz_lm_s203.log 2>&1
