"""Per-phase cycles of K4 at low occupancy (<= 1 CTA per SM): the latency floor (diagnostics).
usage: WT_OPT_SVD_PROFILE=1 python tools/svd_latency.py [n] [batch]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E
E.options_from_env()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
a = torch.randn(b, n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); sig, vec, info = E.svd(a, n); e.record(); torch.cuda.synchronize()
print(f"n={n} batch={b}: {s.elapsed_time(e):.2f} ms, sweeps {E.last_sweeps()}")
