# compute-sanitizer memcheck / racecheck / synccheck over every device kernel
# (tools/sanitize_cases.py: tiny inputs, each decode also checked against the oracle).
set -x
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize_cases.py \
    > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san_$tool.log
done
