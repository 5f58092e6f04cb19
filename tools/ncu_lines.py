"""Per-source-line warp-stall / instruction shares of one kernel in an ncu report
(run here on a report from the GPU box): python tools/ncu_lines.py rep.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, ex, src = collections.Counter(), collections.Counter(), {}
fname = hdr = cur = None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        cur = r[0]
        src[(fname, cur)] = r[1]
    try:
        st, e = float(r[4]), float(r[7])
    except (ValueError, IndexError):
        continue
    agg[(fname, cur)] += st
    ex[(fname, cur)] += e
tot, te = sum(agg.values()) or 1, sum(ex.values()) or 1
print(f"stall samples {tot:.0f}, instructions {te:.0f}")
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{v / tot * 100:5.1f}% stall  {ex[k] / te * 100:5.1f}% inst  {k[0]}:{k[1]}  {src.get(k, '').strip()[:80]}")
