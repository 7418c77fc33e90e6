"""Summarise an ncu launch list (csv: gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) of ONE K4 call into per-phase time / DRAM bytes and write
profiles/traffic_r02.json's K4 entry.  usage: python tools/k4_traffic.py launches.csv cfg out.json"""
import collections
import csv
import json
import sys

path, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
iname, imet, iunit, ival = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
iid = hdr.index("ID")
k = collections.defaultdict(dict)
for r in rows[1:]:
    k[r[iid]]["name"] = r[iname]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "second": 1.0}.get(r[iunit], 1.0)
    k[r[iid]][r[imet]] = float(r[ival].replace(",", "")) * scale


def phase(n):
    for key, ph in (("sbr_update_mult", "two-stage: trailing pass (update + Z = A22 V)"), ("sbr_panel", "two-stage: panel QR"),
                    ("sbr_w", "two-stage: W"), ("sbr_chase", "two-stage: band chase"),
                    ("sbr_apply_q2", "two-stage: stage-2 back-transformation"),
                    ("tridiag_panel", "tridiagonalization panels"), ("gemm_f64", "K3 GEMMs (Gram, trailing, NS, back-transform, X V0)"),
                    ("tri_bisect", "bisection"), ("tri_multisect", "bisection"), ("tri_inviter", "inverse iteration"), ("cluster_mgs", "cluster MGS"),
                    ("svd_sweep_kernel", "Jacobi sweeps"), ("ns_", "Newton-Schulz bookkeeping"), ("wy_larft", "larft"), ("sbr_larft_merge", "larft")):
        if key in n:
            return ph
    return "other (copy-in, sort, permute, flags)"


agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for v in k.values():
    a = agg[phase(v["name"])]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0.0)
    a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
tot_t = sum(a[1] for a in agg.values())
tot_b = sum(a[2] for a in agg.values())
res = {"launches": len(k), "serialized_ms": round(tot_t * 1e3, 3), "dram_bytes_per_call": int(tot_b),
       "phases": {p: {"launches": a[0], "ms": round(a[1] * 1e3, 3), "dram_GB": round(a[2] / 1e9, 3)}
                  for p, a in sorted(agg.items(), key=lambda x: -x[1][1])},
       "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 f"--clock-control none on tools/k4_launches.py {cfg} (one K4 call, NVTX range k4call); "
                 "launches serialized and cold: shares, not absolute times"}
try:
    allres = json.load(open(out))
except Exception:  # noqa: BLE001
    allres = {}
allres[f"K4_cfg{cfg}"] = res
json.dump(allres, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
