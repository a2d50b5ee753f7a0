"""Copy a round's measurement outputs from gpurun_out/ into profiles/<dir>/ and
summarise the ncu capture of the decode kernel
(usage: python tools/save_profiles.py profiles/r01/s2 [gpurun_out/subdir])."""
import csv, io, json, os, shutil, subprocess, sys

dst = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
os.makedirs(dst, exist_ok=True)
for f in ("bench.json", "bench_ref.json", "bench_cfg1.json", "launches.csv", "host_cpu.txt", "gpu.txt", "pytest_gpu.log",
          "smoke.log"):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
rep = os.path.join(src, "ncu_full_cfg4.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    si, mi, vi, ui = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    keep = {"Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Executed Instructions",
            "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Block Size", "Grid Size",
            "Dynamic Shared Memory Per Block", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "SM Frequency"}
    lines = [f"{x[si]} | {x[mi]} = {x[vi]} {x[ui]}" for x in rows[1:] if x[mi] in keep]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    name = r[2][r[0].index("Kernel Name")] if "Kernel Name" in r[0] else "?"
    dram = 0.0
    for i, n in enumerate(r[0]):
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum") or ("pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued")):
            lines.append(f"{n} {r[1][i]} {r[2][i]}")
        if n in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r[1][i]]
            dram += float(r[2][i].replace(",", "")) * scale
    with open(os.path.join(dst, "ncu_decode_summary.txt"), "w") as fh:
        fh.write(f"# ncu --set full, one cfg4 launch of {name}\n" + "\n".join(lines) + "\n")
    hot = subprocess.run([sys.executable, "tools/ncu_hot_lines.py", rep, "40"], capture_output=True, text=True).stdout
    open(os.path.join(dst, "ncu_decode_hot_lines.txt"), "w").write(hot)
    ops = subprocess.run([sys.executable, "tools/ncu_opcodes.py", rep, "2041806"], capture_output=True, text=True).stdout
    open(os.path.join(dst, "ncu_decode_opcodes_per_frame.txt"), "w").write(ops)
    kname = name.split("(")[0].split("::")[-1]
    with open("profiles/ncu_traffic.json", "w") as fh:
        json.dump({"workload": "cfg4-whole-box", "n_gpus": 1, "kernel": kname, "dram_bytes_per_launch": int(dram),
                   "source": f"{dst}/ncu_decode_summary.txt: dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full, "
                             "one launch of bench.py --workload cfg4 --steps 1 --warmup 3"}, fh, indent=1)
print(sorted(os.listdir(dst)))
