"""Summarise an ncu source page (cuda,sass view) into per-CUDA-line stall samples.

usage: ncu -i rep --page source --csv --print-source=cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [topN]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
func, hdr, per, src, path = None, None, {}, {}, ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1][:60]
        per.setdefault(func, defaultdict(float))
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if func and hdr and len(r) == len(hdr) and r[0].isdigit():
        line = (path, int(r[0]))
        src.setdefault((func, line), r[1])
        try:
            per[func][line] += float(r[4] or 0)
        except ValueError:
            pass
for f, d in per.items():
    tot = sum(d.values()) or 1.0
    print("==", f, f"(samples {tot:.0f})")
    for line, v in sorted(d.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {line[0]}:{line[1]:<5} {src[(f, line)].strip()[:90]}")
