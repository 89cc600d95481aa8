"""Per-source-line warp-stall samples from `ncu -i X --page source --csv
--print-source cuda,sass` output. usage: ncu_lines.py file.csv [top]"""
import csv
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lines, si, fname = [], None, "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or len(r) <= si or not r[0]:
        continue
    try:
        lines.append((float(r[si] or 0), f"{fname}:{r[0]}", r[1][:110]))
    except ValueError:
        continue
tot = sum(v for v, _, _ in lines) or 1
print(f"total samples {tot:.0f}")
for v, ln, s in sorted(lines, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {ln:<18} {s}")
