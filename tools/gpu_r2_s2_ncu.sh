set -x
bash tools/gpu_ncu_full.sh ctcb_decode_fast_small_kernel cfg4
bash tools/gpu_sanitize.sh
