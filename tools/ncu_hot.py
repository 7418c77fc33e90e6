"""Top source lines by warp-stall samples from an ncu report (reads `ncu --page source --csv`)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_all = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter(); src = {}; reasons = collections.defaultdict(collections.Counter)
for r in rows:
    if len(r) <= i_all or not r[0].isdigit():
        continue
    try:
        v = int(r[i_all])
    except ValueError:
        continue
    agg[r[0]] += v; src[r[0]] = r[1][:95]
    for k in stall_cols:
        try:
            reasons[r[0]][hdr[k]] += int(r[k])
        except (ValueError, IndexError):
            pass
tot = sum(agg.values()) or 1
print("total samples", tot)
for line, v in agg.most_common(n):
    top = ", ".join(f"{k[6:]}={c}" for k, c in reasons[line].most_common(3))
    print(f"{v:7d} {100*v/tot:5.1f}% L{line}: {src[line]}  [{top}]")
