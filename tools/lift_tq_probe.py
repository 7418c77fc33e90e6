"""Median GB/s of K1 / K2 at config 2 for several L (diagnostics; env WT_LIFT_TQ_MAX)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E
x = torch.randn(512, 512, 256, dtype=torch.float64, device="cuda")
n = x.numel()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); return 2 * n * 8 / ts[len(ts) // 2] / 1e6
res = []
for L in [int(a) for a in os.environ.get("LS", "1 2 4 6 8").split()]:
    buf = E.lift_forward(x, L)
    out = torch.empty_like(x)
    f = t(lambda: E.lift_forward(x, L))
    i = t(lambda: E.lift_inverse(buf, 512, 512, 256, L))
    y = E.lift_inverse(buf, 512, 512, 256, L)
    ok = float((y - x).abs().max()) < 1e-12
    res.append(f"L={L} fwd {f:.0f} inv {i:.0f} {'ok' if ok else 'BAD'}")
print(os.environ.get("WT_LIFT_TQ_MAX", "16"), " | ".join(res))
