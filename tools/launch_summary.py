"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv):
total time, launches and DRAM bytes per kernel name.  usage: python tools/launch_summary.py file.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
L = {}
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    L.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for v in L.values():
    name = re.sub(r"\(.*", "", v["k"]).replace("void ", "")
    a = agg[name]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0.0)
    a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{a[1] / 1e6:9.3f} ms {a[0]:5d} launches {a[2] / 1e9:8.2f} GB  {name}")
print(f"{tot / 1e6:9.3f} ms total")
