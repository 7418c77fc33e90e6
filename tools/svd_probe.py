"""Probe K4 accuracy/sweeps/time on the config-3/4 wavelet slices (diagnostics).
usage: python tools/svd_probe.py [inner_sweeps ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_08228_b200 import engine as E, synth

inners = sys.argv[1:] or ["16"]
cases = [(256, 256, 192, 3, 20), (1024, 1024, 256, 4, 30)]
for (n1, n2, p, L, r) in cases:
    x = torch.from_numpy(synth.hyperspectral_cube(n1, n2, p, seed=0)).cuda()
    pyr = E.lift_forward(x, L)
    sel = pyr if n1 == 256 else pyr[p - 2 * (p >> L):]
    a = sel.cpu().numpy()
    k = min(6, a.shape[0])
    ref = np.linalg.svd(a[:k], compute_uv=False)
    for inner in inners:
        os.environ["WT_SVD_INNER_SWEEPS"] = inner
        for rep in range(2):
            torch.cuda.synchronize(); t = time.perf_counter()
            sigma, vec, info = E.svd(sel, r)
            torch.cuda.synchronize(); dt = time.perf_counter() - t
        s = sigma.cpu().numpy()[:k]
        err = np.abs(s - ref) / ref[:, :1]
        print(f"{n1}x{n2} batch {sel.shape[0]} inner {inner}: {dt*1e3:.1f} ms, sweeps {E.last_sweeps()}, "
              f"info {int(info.abs().sum())}, max sigma err {err.max():.3e}", flush=True)
