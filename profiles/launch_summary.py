"""Summarise an `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L` launch
list (profiles/README_r02.md): launches, total, share and average per kernel, largest first.
    python profiles/launch_summary.py LAUNCHES.csv [CMD-NOTE] > SUMMARY.txt"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*$", "", r[ki])
    name = re.sub(r"^(void )?", "", name)
    name = re.sub(r"<.*$", "", name)
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
allt = sum(tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none launch list (cold-cache, serialised; compare SHARES)")
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print(f"# {sum(cnt.values())} launches, {allt / 1e3:.3f} ms in total")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:40]:40s} {cnt[k]:6d} launches {tot[k] / 1e3:10.3f} ms {100 * tot[k] / allt:6.1f}%  avg {tot[k] / cnt[k]:9.2f} us")
