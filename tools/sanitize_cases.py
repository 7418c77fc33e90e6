"""Small invocations of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): K1/K2 at every L (TMA paths, shallow / persistent /
ancestor-chain variants, peer tables), K3 orientations, K4 plain / cluster-split
(S = 2, 4, 8 through WT_OPT_SVD_SPLIT) / preconditioned (single CTA and cluster
panels), the epilogues, the orthonormal completion and the LU pivot check.
Checks results against numpy so a silent corruption also fails.
usage: [WT_OPT_SVD_SPLIT=S] python tools/sanitize_cases.py [lift|gemm|svd|all]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_08228_b200 as W  # noqa: E402
from paper_2601_08228_b200 import engine as E  # noqa: E402
E.options_from_env()
from oracle import wten_oracle as O  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300))


if what in ("lift", "all"):
    x = rng.standard_normal((24, 20, 256))
    for L in (1, 2, 3, 4, 5, 6, 7, 8):
        pyr = W.forward_w(torch.from_numpy(x).cuda(), L)
        s, d = O.lift_forward(x, L)
        assert np.array_equal(pyr.smooth.cpu().numpy(), s)
        assert np.array_equal(W.inverse_w(pyr).cpu().numpy(), O.lift_inverse(s, d))
    y = rng.standard_normal((40, 16, 64))
    assert rel(W.sp_w_svd(y, 4, 2), O.sp_w_svd(y, 4, 2)) < 1e-8
    print("lift ok", flush=True)

if what in ("gemm", "all"):
    for ta in (0, 1):
        for tb in (0, 1):
            a = rng.standard_normal((3, 70, 50))
            b = rng.standard_normal((3, 50, 90))
            A = torch.from_numpy(a.transpose(0, 2, 1).copy() if ta else a).cuda()
            B = torch.from_numpy(b.transpose(0, 2, 1).copy() if tb else b).cuda()
            c = E.gemm(A, B, trans_a=bool(ta), trans_b=bool(tb)).cpu().numpy()
            assert rel(c, a @ b) < 1e-13
    print("gemm ok", flush=True)

if what in ("svd", "all"):
    for shape in [(4, 48, 40), (2, 128, 128), (2, 160, 150), (3, 40, 130)]:
        a = rng.standard_normal(shape)
        s, vec, info = E.svd(torch.from_numpy(a).cuda(), min(shape[1:]))
        E.raise_if_failed(info)
        ref = np.linalg.svd(a, compute_uv=False)
        assert np.max(np.abs(s.cpu().numpy() - ref)) < 1e-12 * ref.max(), shape
    cube = rng.standard_normal((6, 5, 8))
    cube[:, :, 4:] = cube[:, :, 3:4]  # constant tail: zero detail slices (rank-deficient blocks)
    f, rec = W.w_svd(cube, 3, 2)
    assert rel(rec, O.w_svd(cube, 3, 2)["recon"]) < 1e-8
    u, sv, v = W.matrix_svd(np.zeros((4, 3)))
    assert np.abs(u.T @ u - np.eye(3)).max() < 1e-12
    pinv = W.pinv_w(rng.standard_normal((12, 10, 8)), 2)
    inv = W.inverse_tensor(rng.standard_normal((6, 6, 4)) + 4 * np.eye(6)[:, :, None], 1)
    print("svd ok", flush=True)
