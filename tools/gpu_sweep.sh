# Bench cfg4 (and cfg1) with each library variant in variants/ plus the default build.
set -x
for lib in paper_2310_17864_b200/libctcb.so variants/*.so; do
  n=$(basename $lib .so)
  CTCB_LIB=$PWD/$lib timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/q_cfg4_$n.json 2> gpurun_out/q_cfg4_$n.err
done
