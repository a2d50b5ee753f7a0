"""Dynamic SASS opcode mix of an ncu --import-source report:
python tools/ncu_opcodes.py REP.ncu-rep [units]  (counts ÷ units, e.g. frames)."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
tot = 0.0
for r in csv.reader(io.StringIO(out)):
    if len(r) < 6 or not r[0].startswith("0x"):
        continue
    try:
        n = float(r[5])
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[1])
    if not m:
        continue
    agg[m.group(2)] += n
    tot += n
print(f"total {tot / units:.1f}")
for op, n in agg.most_common(40):
    print(f"{op:14s} {n / units:8.1f}  {100 * n / tot:5.1f}%")
