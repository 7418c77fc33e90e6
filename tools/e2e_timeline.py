"""Timeline of one numpy sp_w_svd call on the config-4 cube (upload + K1, K4 + K5,
K2 + download), from CUDA events around the decomposition inside
engine.host_slices_pipeline.  usage: python tools/e2e_timeline.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08228_b200 as W  # noqa: E402
from paper_2601_08228_b200 import decomposition as D, synth  # noqa: E402

x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
if len(sys.argv) > 1 and sys.argv[1] == "pinned":  # the cube in page-locked memory: DMA in place
    xp = W.pinned_empty(x.shape)
    xp[...] = x
    x = xp
marks = {}
inner = D._coarse_truncate


def wrapped(r, tol=0.0):
    f = inner(r, tol)

    def decompose(coarse):
        marks["t_dec0"] = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        out = f(coarse)
        e1.record()
        marks["ev"] = (e0, e1)
        return out
    return decompose


D._coarse_truncate = wrapped
keep = []
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s0 = torch.cuda.Event(enable_timing=True)
    s0.record()
    y = W.sp_w_svd(x, 30, 4)
    s1 = torch.cuda.Event(enable_timing=True)
    s1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    keep = [y]
    e0, e1 = marks["ev"]
    print(f"call {rep}: wall {1e3 * (t1 - t0):6.1f} ms | upload+K1 (to decompose start) {s0.elapsed_time(e0):6.1f} ms"
          f" | K4+K5 {e0.elapsed_time(e1):6.1f} ms | K2+download {e1.elapsed_time(s1):6.1f} ms"
          f" | host time to decompose call {1e3 * (marks['t_dec0'] - t0):6.1f} ms", flush=True)
