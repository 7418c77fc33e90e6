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
        # wavelet-domain U and V blocks orthonormal, every column --
        # zero / rank-deficient slices included (K6 completes them like LAPACK)
        for fac in (f.U, f.V):
            pu = E.lift_forward(torch.from_numpy(np.ascontiguousarray(fac)).cuda(), L).cpu().numpy()
            for k2 in range(p):
                u = pu[k2]
                assert np.abs(u.T @ u - np.eye(u.shape[1])).max() < 1e-10
    # sp-w-svd == w-svd at L = 1
    a = rng.standard_normal((9, 7, 8))
    assert relerr(W.sp_w_svd(a, 3, 1), W.w_svd(a, 3, 1)[1]) < 1e-14


def graded_cube(n1, n2, p, lo_exp, seed):
    """(n1, n2, p) cube whose every frontal slice has singular values logspace(0, lo_exp)."""
    rng = np.random.default_rng(seed)
    q = min(n1, n2)
    out = np.empty((n1, n2, p))
    for k in range(p):
        u = np.linalg.qr(rng.standard_normal((n1, q)))[0]
        v = np.linalg.qr(rng.standard_normal((n2, q)))[0]
        out[:, :, k] = (u * np.logspace(0, lo_exp, q)) @ v.T
    return out


@pytest.mark.parametrize("shape", [(48, 40, 8), (40, 48, 8), (160, 144, 4)])
def test_graded_spectrum_full_rank_w_svd(shape):
    """sigma down to 1e-10 sigma_1, full rank: singular values and the
    reconstruction vs the oracle, U / V wavelet blocks orthonormal to 1e-10 (K6's
    short-side factor (A v) / s is re-orthonormalised), U * S * V^T == recon."""
    n1, n2, p = shape
    L = 2
    r = min(n1, n2)
    a = graded_cube(n1, n2, p, -10.0, seed=n1)
    f, rec = W.w_svd(a, r, L)
    want = O.w_svd(a, r, L)
    assert relerr(rec, want["recon"]) < 1e-8
    for (_, s1), (_, s2) in zip(f.sigma_table, want["sigma_table"]):
        assert np.max(np.abs(s1 - s2) / s2[:, :1]) < 1e-8
    for fac in (f.U, f.V):
        pu = E.lift_forward(torch.from_numpy(np.ascontiguousarray(fac)).cuda(), L).cpu().numpy()
        for k in range(p):
            assert np.abs(pu[k].T @ pu[k] - np.eye(r)).max() < 1e-10
    usv = W.w_product(W.w_product(f.U, f.S, L), W.transpose(f.V), L)
    assert relerr(usv, rec) < 1e-10


def test_graded_spectrum_pinv_via_factors():
    """pinv_w_via_factors on sigma down to 1e-10 sigma_1 (full rank): equals pinv_w and the
    oracle to the conditioning (cond 1e10 -> agreement ~eps * cond), and the Penrose
    identities A A+ A = A, A+ A A+ = A+ hold."""
    a = graded_cube(32, 32, 8, -10.0, seed=3)
    L = 2
    x1 = W.pinv_w_via_factors(a, L)
    x2 = W.pinv_w(a, L)
    ref = O.pinv_w(a, L)
    assert relerr(x1, ref) < 1e-4 and relerr(x2, ref) < 1e-4
    assert relerr(x1, x2) < 1e-4
    aa = W.w_product(W.w_product(a, x2, L), a, L)
    assert relerr(aa, a) < 1e-6  # eps * cond(1e10)


def test_matrix_svd_orthonormal_for_zero_and_rank_one():
    """tensor.matrix_svd (SPEC: U^T U = I to 1e-12, zero matrix included)."""
    rng = np.random.default_rng(5)
    cases = [np.zeros((3, 3)), np.zeros((5, 2)), np.outer(rng.standard_normal(7), rng.standard_normal(4)),
             np.outer(rng.standard_normal(3), rng.standard_normal(6)), rng.standard_normal((6, 6))]
    for m in cases:
        u, s, v = W.matrix_svd(m)
        q = min(m.shape)
        assert u.shape == (m.shape[0], q) and v.shape == (m.shape[1], q)
        assert np.abs(u.T @ u - np.eye(q)).max() < 1e-12
        assert np.abs(v.T @ v - np.eye(q)).max() < 1e-12
        assert np.abs((u * s) @ v.T - m).max() <= 1e-12 * max(1.0, np.abs(m).max())
        np.testing.assert_allclose(s, np.linalg.svd(m, compute_uv=False), atol=1e-12 * max(1.0, s.max()))
