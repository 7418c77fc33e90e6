"""Warp-stall samples per CUDA source line from an ncu report (--import-source, -lineinfo build).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, agg, src, cur = None, {}, {}, None
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if not r[0]:  # SASS rows under a source line (the line row carries their sum)
        continue
    cur = r[0]
    src[cur] = r[1]
    try:
        v = float(r[4] or 0)
    except ValueError:
        v = 0.0
    agg[cur] = agg.get(cur, 0.0) + v
tot = sum(agg.values()) or 1.0
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{ln:>5s} {v / tot * 100:5.1f}%  {src.get(ln, '')[:110]}")
