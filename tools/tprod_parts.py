"""Time the pieces of the t-product at a p^3 cube (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import baselines as B, engine as E
p = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = torch.randn(p, p, p, dtype=torch.float64, device="cuda")
def t(name, fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): r = fn()
    e.record(); torch.cuda.synchronize(); print(f"{name:28s} {s.elapsed_time(e)/reps*1e3:8.1f} us"); return r
spec = t("rfft", lambda: torch.fft.rfft(a, dim=2))
f = t("_spectrum (no delta)", lambda: B._spectrum(a, exact_dc=False))
t("t_product", lambda: B.t_product(a, a)); sys.exit(0)
h = p // 2 + 1
fc = torch.empty((2 * h, p, p), dtype=torch.float64, device="cuda")
t("gemm re.re", lambda: E.gemm(f[:h], f[:h], out=fc[:h]))
t("4 gemms", lambda: (E.gemm(f[:h], f[:h], out=fc[:h]), E.gemm(f[h:], f[h:], alpha=-1.0, beta=1.0, out=fc[:h]),
                      E.gemm(f[:h], f[h:], out=fc[h:]), E.gemm(f[h:], f[:h], beta=1.0, out=fc[h:])))
t("_synthesis", lambda: B._synthesis(fc, p))
t("t_product", lambda: B.t_product(a, a))
