"""K4 with / without the Gram-eigenbasis preconditioner (eig.cu): singular values vs
LAPACK, sweeps, fallbacks, time.  usage: python tools/precond_check.py [quick]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import _native as N, engine as E, synth  # noqa: E402
E.options_from_env()
from oracle import wten_oracle as O  # noqa: E402


def run(name, a):
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ref = np.linalg.svd(a, compute_uv=False)
    lib = N.load()
    out = {}
    for reps in (1, 3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            s, vec, info = E.svd(at, 0)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / reps * 1e3
    s = s.cpu().numpy()
    err = np.max(np.abs(s - ref) / np.maximum(ref[:, :1], 1e-300))
    print(f"{name:34s} ms {ms:8.2f} sweeps {E.last_sweeps():3d} fallbacks {lib.wt_svd_last_fallbacks():4d} "
          f"sigma err {err:.1e} info {int(info.max())}", flush=True)
    return err


def cases(quick):
    rng = np.random.default_rng(0)
    yield "rand 4x128^2", rng.standard_normal((4, 128, 128))
    yield "rand 3x200x150", rng.standard_normal((3, 200, 150))
    yield "rand 2x150x260", rng.standard_normal((2, 150, 260))
    yield "rand 8x256^2", rng.standard_normal((8, 256, 256))
    x = synth.hyperspectral_cube(256, 256, 192, seed=0)
    s, d = O.lift_forward(x, 3)
    pyr = O.packed_slices(s, d)
    yield "cfg3 192x256^2", pyr
    u = np.linalg.qr(rng.standard_normal((256, 256)))[0]
    v = np.linalg.qr(rng.standard_normal((256, 256)))[0]
    g = (u * np.logspace(0, -10, 256)) @ v.T
    yield "graded 1e-10 256^2", np.stack([g, g.T])
    z = np.zeros((3, 256, 256)); z[1] = rng.standard_normal((256, 256))
    yield "zero+rand 3x256^2", z
    yield "blur 2x512^2", np.stack([synth.toeplitz_blur(512)] * 2)
    if quick:
        return
    yield "rand 4x512^2", rng.standard_normal((4, 512, 512))
    x = synth.hyperspectral_cube(1024, 1024, 32, seed=0)
    s, d = O.lift_forward(x, 4)
    yield "cfg4 coarse 4x1024^2", O.packed_slices(s, d)[-4:]
    x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
    s, d = O.lift_forward(x, 4)
    yield "cfg4 32x1024^2", O.packed_slices(s, d)[-32:]


if __name__ == "__main__":
    quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
    mode = os.environ.get("WT_OPT_SVD_PRECOND", "1")
    print("WT_OPT_SVD_PRECOND =", mode)
    worst = 0.0
    for name, a in cases(quick):
        worst = max(worst, run(name, a))
    print("worst sigma err %.1e" % worst)
