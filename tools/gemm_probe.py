"""K3 throughput on the config-5 face product shape (128 x 512^3) and others."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_08228_b200 import engine as E

E.options_from_env()  # WT_OPT_GEMM_TMA=0: the cp.async ring instead of the tensor-map variant

for (b, m, n, k) in [(128, 512, 512, 512), (32, 1024, 1024, 1024), (192, 256, 256, 256), (32, 64, 40, 48)]:
    A = torch.randn(b, m, k, dtype=torch.float64, device="cuda")
    B = torch.randn(b, k, n, dtype=torch.float64, device="cuda")
    C = torch.empty(b, m, n, dtype=torch.float64, device="cuda")
    for ta, tb in [(False, False), (False, True), (True, False), (True, True)]:
        a = A.transpose(1, 2).contiguous() if ta else A
        bb = B.transpose(1, 2).contiguous() if tb else B
        for _ in range(3):
            E.gemm(a, bb, ta, tb, out=C)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            E.gemm(a, bb, ta, tb, out=C)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        ref = torch.bmm(A, B)
        err = float((C - ref).norm() / ref.norm())
        print(f"batch {b} {m}x{n}x{k} tA={int(ta)} tB={int(tb)}: {ms*1e3:8.1f} us  {2*b*m*n*k/ms/1e9:6.2f} TF/s  relerr {err:.1e}", flush=True)
    # cuBLAS fp64 for context (library reference point, not the product path)
    for _ in range(3): torch.bmm(A, B, out=C)
    s.record()
    for _ in range(10): torch.bmm(A, B, out=C)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"   cuBLAS bmm fp64: {ms*1e3:8.1f} us  {2*b*m*n*k/ms/1e9:6.2f} TF/s", flush=True)
