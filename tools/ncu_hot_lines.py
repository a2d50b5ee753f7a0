"""Aggregate an ncu --import-source report by CUDA source line (all inlined call
sites summed):  python tools/ncu_hot_lines.py REP.ncu-rep [N]"""
import csv, io, os, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, recs, tot_i, tot_s = "?", [], 0.0, 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1]); continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        smp, ins = float(r[4]), float(r[7])
    except (ValueError, IndexError):
        continue
    tot_i += ins; tot_s += smp
    recs.append((ins, smp, f"{fname}:{r[0]}", r[1].strip()[:100]))
print(f"samples {tot_s:.0f} instr {tot_i:.0f}")
for ins, smp, ln, src in sorted(recs, key=lambda x: -x[1])[:n]:
    print(f"{ln:>22} samp {100*smp/max(tot_s,1):5.1f}% inst {100*ins/max(tot_i,1):5.1f}%  {src}")
