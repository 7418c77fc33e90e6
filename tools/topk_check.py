"""Rank-r reconstructions through K4's leading-triplet mode (wt_svd_topk_f64) vs the full
K4 and LAPACK: relative error and time.  usage: python tools/topk_check.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08228_b200 import engine as E, synth  # noqa: E402
from oracle import wten_oracle as O  # noqa: E402

E.options_from_env()


def lapack_trunc(a, r):
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    return u[:, :, :r] @ (s[:, :r, None] * vh[:, :r, :])


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t) * 1e3


def run(name, a, r):
    at = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ref = lapack_trunc(a, r)
    k = E.topk_width(min(a.shape[1:]), r)

    def full():
        s, v, info = E.svd(at, r)
        E.raise_if_failed(info)
        return E.truncated_recon(at, s, v, r)

    rec_t, ms_t = timed(lambda: E.svd_truncated_recon(at, r))
    sw_t = E.last_sweeps()
    rec_f, ms_f = timed(full)
    rel = lambda x: float(np.linalg.norm((x.cpu().numpy() - ref).ravel()) / np.linalg.norm(ref.ravel()))  # noqa: E731
    print(f"{name:28s} r={r:3d} k={k:3d}: topk {ms_t:7.2f} ms ({sw_t} sweeps) err {rel(rec_t):.1e} | "
          f"full {ms_f:7.2f} ms err {rel(rec_f):.1e}", flush=True)


rng = np.random.default_rng(0)
run("rand 8x256^2", rng.standard_normal((8, 256, 256)), 20)
run("rand 4x512x300", rng.standard_normal((4, 512, 300)), 30)
x = synth.hyperspectral_cube(256, 256, 192, seed=0)
s, d = O.lift_forward(x, 3)
run("cfg3 coarse (s3, d3) 48x256^2", O.packed_slices(s, d)[-48:], 20)
x = synth.hyperspectral_cube(1024, 1024, 256, seed=0)
s, d = O.lift_forward(x, 4)
run("cfg4 coarse 32x1024^2", O.packed_slices(s, d)[-32:], 30)
