"""Per-launch DRAM traffic of the lifting kernels from an `ncu --set full` report
-> profiles/traffic_rNN.json (the bench's roofline.traffic).
usage: python tools/traffic_from_ncu.py report.ncu-rep profiles/traffic_r01.json"""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
idx = {k: hdr.index(k) for k in keep if k in hdr}
units = rows[1]
launches = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    launches.append({k: r[i] for k, i in idx.items()})
def mb(v, u):
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
    return float(v.replace(",", "")) * scale
res = {}
for name, keys in (("K1_forward", ("fwd_persistent", "fwd_shallow")), ("K2_inverse", ("inv_persistent",))):
    sel = [l for l in launches if any(k in l["Kernel Name"] for k in keys)]
    if not sel:
        continue
    ur, uw = units[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_write.sum"]]
    tot = [mb(l["dram__bytes_read.sum"], ur) + mb(l["dram__bytes_write.sum"], uw) for l in sel]
    res[name] = int(sum(tot) / len(tot) * 1e6)
res["source"] = ("ncu --set full --clock-control none on tools/lift_one.py 1 2 4 8 (config-2 cube): "
                 "dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over L = 1, 2, 4, 8; "
                 "algorithmic = 1073741824 B per launch")
res["units"] = {"dram__bytes_read.sum": units[idx["dram__bytes_read.sum"]]}
res["per_launch"] = launches
json.dump(res, open(out, "w"), indent=1)
print({k: v for k, v in res.items() if k.startswith("K")})
