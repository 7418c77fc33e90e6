"""The SPEC's acceptance criteria that are properties rather than fixtures,
through the GPU product path:

AC2 perfect reconstruction over random tensors and every valid L; AC3 the
algebraic laws (associativity, transpose / inverse reversal, bilinearity,
trace); AC4 Penrose conditions, dagger identities and the two-route
uniqueness; AC5 wavelet-domain Eckart-Young == truncation_bound; plus the
invariant sweep of SURVEY.md section 4 (U * S * V^T == recon, orthonormal U
blocks in the wavelet domain, sp-w-svd == w-svd at L = 1).
"""

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import engine as E
from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu


def test_ac2_perfect_reconstruction_random_sweep():
    """200 random tensors up to 32 x 32 x 64, every valid L: ||inv(fwd(t)) - t|| <= 1e-12 ||t||,
    and the pyramid is bit-identical to the oracle's."""
    rng = np.random.default_rng(2026)
    for k in range(200):
        n1, n2 = (int(v) for v in rng.integers(1, 33, size=2))
        p = int(2 ** rng.integers(0, 7)) * int(rng.choice([1, 3]))
        p = min(p, 64) if p % 3 else min(p, 48)
        L = int(rng.integers(1, W.max_levels(p) + 1)) if W.max_levels(p) >= 1 else None
        if L is None:
            continue
        t = rng.standard_normal((n1, n2, p)) * 10.0 ** float(rng.integers(-3, 4))
        dev = k % 2 == 0
        x = torch.from_numpy(t).cuda() if dev else t
        pyr = W.forward_w(x, L)
        s_ref, d_ref = O.lift_forward(t, L)
        sm = pyr.smooth.cpu().numpy() if dev else pyr.smooth
        assert np.array_equal(sm, s_ref)
        y = W.inverse_w(pyr)
        y = y.cpu().numpy() if dev else y
        assert np.linalg.norm((y - t).ravel()) <= 1e-12 * np.linalg.norm(t.ravel())


def test_ac3_algebraic_laws():
    rng = np.random.default_rng(3)
    L = 2
    wp = lambda a, b: W.w_product(a, b, L)  # noqa: E731
    for _ in range(10):
        a = rng.standard_normal((6, 6, 8)) + 3.0 * np.eye(6)[:, :, None]
        b = rng.standard_normal((6, 6, 8)) + 3.0 * np.eye(6)[:, :, None]
        c = rng.standard_normal((6, 6, 8))
        # associativity, scaled as SPEC.md:246
        err = np.linalg.norm((wp(wp(a, b), c) - wp(a, wp(b, c))).ravel())
        assert err <= 1e-10 * np.linalg.norm(a) * np.linalg.norm(b) * np.linalg.norm(c)
        assert relerr(W.transpose(wp(a, b)), wp(W.transpose(b), W.transpose(a))) < 1e-12
        inv_ab = W.inverse_tensor(wp(a, b), L)
        assert relerr(inv_ab, wp(W.inverse_tensor(b, L), W.inverse_tensor(a, L))) < 1e-8
        a2 = rng.standard_normal(a.shape)
        assert relerr(wp(2.0 * a - 0.5 * a2, b), 2.0 * wp(a, b) - 0.5 * wp(a2, b)) < 1e-12
        assert abs(W.trace(wp(a, b)) - W.trace(wp(b, a))) <= 1e-10 * abs(W.trace(wp(a, b))) + 1e-12
        lhs, rhs = W.trace(wp(W.transpose(a), b)), W.trace(wp(a, W.transpose(b)))
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)
        assert abs(W.trace(a) - W.trace(W.transpose(a))) <= 1e-12 * abs(W.trace(a))


def test_ac4_penrose_dagger_uniqueness():
    rng = np.random.default_rng(4)
    L = 3
    wp = lambda a, b: W.w_product(a, b, L)  # noqa: E731
    for shape in [(12, 8, 8), (8, 12, 8), (10, 10, 8)]:
        a = rng.standard_normal(shape)
        x = W.pinv_w(a, L)
        assert relerr(wp(wp(a, x), a), a) < 1e-8
        assert relerr(wp(wp(x, a), x), x) < 1e-8
        assert relerr(W.transpose(wp(a, x)), wp(a, x)) < 1e-8
        assert relerr(W.transpose(wp(x, a)), wp(x, a)) < 1e-8
        assert relerr(W.pinv_w_via_factors(a, L), x) < 1e-8            # two routes
        assert relerr(W.pinv_w(x, L), a) < 1e-7                         # (a+)+ = a
        assert relerr(W.pinv_w(W.transpose(a), L), W.transpose(x)) < 1e-7
        aat = wp(a, W.transpose(a))
        assert relerr(W.pinv_w(aat, L), wp(W.pinv_w(W.transpose(a), L), x)) < 1e-7
        assert relerr(x, wp(W.transpose(a), W.pinv_w(aat, L))) < 1e-7
        # trace property 5: Tr(a+ b a) = Tr(b) for b = a a+ c
        if shape[0] == shape[1]:
            c = rng.standard_normal((shape[0], shape[0], 8))
            bb = wp(wp(a, x), c)
            assert abs(W.trace(wp(wp(x, bb), a)) - W.trace(bb)) <= 1e-8 * max(abs(W.trace(bb)), 1.0)


def test_ac5_eckart_young_and_invariant_sweep():
    rng = np.random.default_rng(5)
    for k in range(30):
        n1, n2 = (int(v) for v in rng.integers(2, 13, size=2))
        L = int(rng.integers(1, 4))
        p = 8
        r = int(rng.integers(1, min(n1, n2) + 1))
        a = rng.standard_normal((n1, n2, p))
        f, rec = W.w_svd(a, r, L)
        # wavelet-domain residual^2 == sum of discarded sigma^2 == truncation_bound^2
        pa = E.lift_forward(torch.from_numpy(a).cuda(), L).cpu().numpy()
        pr = E.lift_forward(torch.from_numpy(rec).cuda(), L).cpu().numpy()
        res = np.linalg.norm((pa - pr).ravel())
        bound = W.truncation_bound(f, r).bound
        assert abs(res - bound) <= 1e-8 * bound + 1e-13 * np.linalg.norm(pa.ravel())
        # U * S * V^T == recon
        usv = W.w_product(W.w_product(f.U, f.S, L), W.transpose(f.V), L)
        assert relerr(usv, rec) < 1e-10
        # wavelet-domain U blocks orthonormal where sigma > 0
        pu = E.lift_forward(torch.from_numpy(np.ascontiguousarray(f.U)).cuda(), L).cpu().numpy()
        sig = np.concatenate([s for _, s in f.sigma_table])
        for k2 in range(p):
            keep = sig[k2, :r] > 1e-12 * max(sig[k2, 0], 1e-300)
            u = pu[k2][:, keep]
            assert np.abs(u.T @ u - np.eye(u.shape[1])).max() < 1e-10
    # sp-w-svd == w-svd at L = 1
    a = rng.standard_normal((9, 7, 8))
    assert relerr(W.sp_w_svd(a, 3, 1), W.w_svd(a, 3, 1)[1]) < 1e-14
