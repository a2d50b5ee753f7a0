set -x
timeout 900 python -m pytest tests/test_cli.py tests/test_align.py tests/test_lm.py tests/test_ctcforge_api.py tests/test_gpu_parity.py -q -m gpu -k "cli or align or lm or ctcforge or multi_device or regression" -rx > gpurun_out/pytest_glue.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_glue.log
