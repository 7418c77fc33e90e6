"""inverse_w(forward_w(numpy cube)) on the config-2 cube: pageable vs page-locked input."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_08228_b200 as W
x = np.random.default_rng(0).standard_normal((512, 512, 256))
xp = W.pinned_empty(x.shape); xp[...] = x
for name, a in (("pageable", x), ("pinned", xp), ("pageable", x), ("pinned", xp)):
    for _ in range(2):
        for L in (1, 2, 4, 8):
            W.inverse_w(W.forward_w(a, L))
    tf = ti = 0.0
    for L in (1, 2, 4, 8):
        t0 = time.perf_counter(); pyr = W.forward_w(a, L); t1 = time.perf_counter(); o = W.inverse_w(pyr); t2 = time.perf_counter()
        tf += t1 - t0; ti += t2 - t1
    print(f"{name}: forward {tf * 250:.1f} ms/call, inverse {ti * 250:.1f} ms/call, {4 * 4 * x.nbytes / (tf + ti) / 1e9:.1f} GB/s", flush=True)
