"""K4 preconditioner phase times (WT_OPT_EIG_PROFILE) and K4 call times on the config-3
(192 x 256^2) and config-4 (32 x 1024^2) wavelet slices.  usage: python tools/eig_phases.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E, synth  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t) * 1e3)
    return best


for name, (shape, L, last) in {"cfg3": ((256, 256, 192), 3, None), "cfg4": ((1024, 1024, 256), 4, 32)}.items():
    x = synth.hyperspectral_cube(*shape, seed=0)
    s, d = O.lift_forward(x, L)
    a = O.packed_slices(s, d)
    if last:
        a = a[-last:]
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    full = timed(lambda: E.svd(at, 0))
    topk = timed(lambda: E.svd_truncated_recon(at, 30)) if a.shape[1] >= 512 else float("nan")
    print(f"{name}: full K4 {full:.2f} ms, rank-30 leading-triplet recon {topk:.2f} ms", flush=True)
    with E.option("eig_profile", 1):
        E.svd(at, 0)
        if a.shape[1] >= 512:
            E.svd_truncated_recon(at, 30)
        torch.cuda.synchronize()
