"""Share of GPU time per kernel from an ncu launch list
(ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file x.csv ...).

usage: python tools/launch_summary.py launches.csv [header line of the command]
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = next(r for r in rows if "Kernel Name" in r)
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt, units = defaultdict(float), defaultdict(int), set()
for r in rows:
    if r is hdr or len(r) <= max(ik, iv) or r[ik] == "Kernel Name":
        continue
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1.0, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9}.get(r[iu], 1.0)
    units.add(r[iu])
    tot[r[ik]] += v * scale
    cnt[r[ik]] += 1
if len(sys.argv) > 2:
    print(sys.argv[2])
total = sum(tot.values()) or 1.0
print(f"total GPU time {total / 1e9:.3f} s over {sum(cnt.values())} launches "
      f"(serialised per-launch times, units seen {sorted(units)})")
print("share of GPU time per kernel:")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{100 * v / total:7.3f}%  x{cnt[k]:3d}  {k[:100]}")
