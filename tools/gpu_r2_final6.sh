# Final round-2 measurement (session 3, after the packed input screen): GPU suite, bench lines, launch list, ncu --set full, checked-build cases, smoke.
# Round 2 measurement set: GPU tests, bench lines (cfg4 with CPU baselines / e2e / parity,
# reference arm, cfg1, cfg2 beam 50/100, cfg3), launch list, ncu --set full of the
# headline kernel, utterance timeline, checked-build sanitizer substitute, smoke.
set -x
mkdir -p gpurun_out/final6
O=gpurun_out/final6
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > $O/host_cpu.txt
timeout 1200 python -m pytest tests -q -m gpu -rx > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python bench.py --workload cfg1 --no-cpu-baseline > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 300 python bench.py --workload cfg2 --beam 50 --no-cpu-baseline --no-e2e > $O/bench_cfg2_b50.json 2> $O/bench_cfg2_b50.err
timeout 300 python bench.py --workload cfg2 --beam 100 --no-cpu-baseline --no-e2e > $O/bench_cfg2_b100.json 2> $O/bench_cfg2_b100.err
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ctcb_decode_fast_small -s 3 -c 1 -o $O/ncu_full_cfg4 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
python tools/sanitize_cases.py > $O/checks_plain.log 2>&1; echo "rc=$?" >> $O/checks_plain.log
if [ -f variants/libctcb_chk.so ]; then CTCB_LIB=variants/libctcb_chk.so python tools/sanitize_cases.py > $O/checks_fchk.log 2>&1; echo "rc=$?" >> $O/checks_fchk.log; fi
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
