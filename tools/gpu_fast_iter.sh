# Fast-kernel iteration: full cfg4 parity through the fused kernel, GPU parity tests, bench; optional ncu.
set -x
timeout 300 python tools/parity_full.py 4 > gpurun_out/fast_cfg4.jsonl 2> gpurun_out/fast_cfg4.err
timeout 300 python tools/parity_full.py 1 --mode fused > gpurun_out/fast_cfg1f.jsonl 2> gpurun_out/fast_cfg1f.err
timeout 300 python tools/parity_full.py 2 --beam 3 --mode fused >> gpurun_out/fast_cfg1f.jsonl 2>> gpurun_out/fast_cfg1f.err
timeout 300 python tools/parity_full.py 2 --beam 15 --mode fused >> gpurun_out/fast_cfg1f.jsonl 2>> gpurun_out/fast_cfg1f.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_properties.py -q -m gpu -x > gpurun_out/fast_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fast_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/fast_bench.json 2> gpurun_out/fast_bench.err
if [ "${NCU:-0}" = "1" ]; then bash tools/gpu_ncu_full.sh ctcb_decode_fast_small_kernel cfg4; fi
