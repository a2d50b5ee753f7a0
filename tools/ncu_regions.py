"""Executed warp-instruction breakdown of an ncu --import-source report by
kernel code region.

    python tools/ncu_regions.py REP.ncu-rep FILE.cu UNITS START:NAME [START:NAME ...]

The cuda+sass source view lists a SASS instruction once under every source
line of its inline call stack; instructions are deduplicated by address and
attributed (executed instructions and warp-state samples) to the deepest line of FILE.cu at or after the first region start
(the call site inside the kernel body), else to the region of the preceding
address.  Counts are divided by UNITS (e.g. warp-frames).
"""
import csv
import io
import os
import subprocess
import sys

rep, fname, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
regions = sorted((int(a.split(":")[0]), a.split(":")[1]) for a in sys.argv[4:])
first = regions[0][0]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, cur_line = "?", 0
count, samp, lines = {}, {}, {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = os.path.basename(r[1])
        continue
    if r[0] == "" and len(r) > 7 and r[2].startswith("0x"):
        a = int(r[2], 16)
        try:
            count[a] = float(r[7])
        except ValueError:
            count.setdefault(a, 0.0)
        try:
            samp[a] = float(r[4])
        except ValueError:
            samp.setdefault(a, 0.0)
        if cur_file == fname and cur_line >= first:
            lines.setdefault(a, []).append(cur_line)
    else:
        try:
            cur_line = int(r[0])
        except ValueError:
            pass


def region_of(line):
    name = None
    for start, nm in regions:
        if line >= start:
            name = nm
    return name


agg, sagg, last = {}, {}, "prologue"
for a in sorted(count):
    if a in lines:
        last = region_of(max(lines[a]))
    agg[last] = agg.get(last, 0.0) + count[a]
    sagg[last] = sagg.get(last, 0.0) + samp.get(a, 0.0)
tot = sum(agg.values())
stot = sum(sagg.values()) or 1.0
print(f"{'region':24s} {'inst/unit':>9s}  {'inst%':>5s}  {'stall-samples%':>14s}")
for k, v in sorted(agg.items(), key=lambda x: -sagg[x[0]]):
    print(f"{k:24s} {v / units:9.1f}  {100 * v / tot:5.1f}  {100 * sagg[k] / stot:14.1f}")
print(f"{'total':24s} {tot / units:9.1f}")
