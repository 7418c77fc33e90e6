"""Two-stage (eig_sbr.cuh) vs one-stage tridiagonalization inside K4's leading-triplet mode:
rank-r reconstructions against LAPACK, bit-repeatability, times and preconditioner phases.
usage: python tools/sbr_check.py [quick]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import _native as N, engine as E, synth  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"


def lapack_trunc(a, r):
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    return u[:, :, :r] @ (s[:, :r, None] * vh[:, :r, :])


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t) * 1e3)
    return out, best


def run(name, a, r):
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ref = lapack_trunc(a, r)
    rel = lambda x: float(np.linalg.norm((x.cpu().numpy() - ref).ravel()) / np.linalg.norm(ref.ravel()))  # noqa: E731
    out = {}
    for two in (1, 0):
        with E.option("eig_twostage", two):
            rec, ms = timed(lambda: E.svd_truncated_recon(at, r))
            sw, fb = E.last_sweeps(), int(N.load().wt_svd_last_fallbacks())
            rec2 = E.svd_truncated_recon(at, r)
            out[two] = (rel(rec), ms, sw, fb, bool(torch.equal(rec, rec2)))
    for two in (1, 0):
        e, ms, sw, fb, same = out[two]
        print(f"{name:26s} r={r:3d} {'two-stage' if two else 'one-stage'}: {ms:7.2f} ms, {sw} sweeps, fallbacks {fb}, "
              f"err vs LAPACK {e:.1e}, repeat-identical {same}", flush=True)


rng = np.random.default_rng(0)
run("rand 2x512^2", rng.standard_normal((2, 512, 512)), 30)
run("rand 3x700x600", rng.standard_normal((3, 700, 600)), 20)
run("rand 2x1024^2", rng.standard_normal((2, 1024, 1024)), 30)
g = rng.standard_normal((2, 1024, 1024))
u, _, vh = np.linalg.svd(g, full_matrices=False)
run("graded 2x1024^2", u @ (np.logspace(0, -10, 1024)[None, :, None] * vh), 30)
run("rand 2x1030x1034", rng.standard_normal((2, 1034, 1030)), 30)
if not quick:
    x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
    s, d = O.lift_forward(x, 4)
    a = O.packed_slices(s, d)[-32:]
    run("cfg4 coarse 32x1024^2", a, 30)
    run("cfg4 8-GPU share 4x1024^2", a[:4], 30)
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for two in (1, 0):
        with E.option("eig_twostage", two), E.option("eig_profile", 1):
            E.svd_truncated_recon(at, 30)
            torch.cuda.synchronize()
