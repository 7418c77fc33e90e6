"""Config 5 (w-pinv deblurring) and the imaging helpers on the GPU.

PSNR/SSIM have no reference code; the oracle follows the
PAPER/SPEC formulas, so these parities are pinned to that restatement.
Bars (north_star): PSNR within 1e-6 dB, SSIM within 1e-6; pseudo-inverse and
recovered images within 1e-8 relative.
"""

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import imaging, synth
from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu


def test_psnr_ssim_match_oracle():
    rng = np.random.default_rng(41)
    x = rng.random((40, 30, 16))
    y = np.clip(x + 0.05 * rng.standard_normal(x.shape), 0, 1)
    assert abs(imaging.psnr(x, y) - O.psnr(x, y)) < 1e-9
    assert abs(imaging.ssim(x, y) - O.ssim(x, y)) < 1e-12
    assert abs(imaging.psnr(x, y, 2.0) - O.psnr(x, y, 2.0)) < 1e-9
    assert imaging.psnr(x, x) == float("inf")
    assert abs(imaging.ssim(x, x) - 1.0) < 1e-15
    assert imaging.psnr(np.ones((2, 2, 2)), np.zeros((2, 2, 2)), 1.0) == 0.0


def test_blur_operator_spec_examples():
    av, ah = imaging.blur_operator(2, 1, 4, 3, 4)
    np.testing.assert_allclose(av[:, :, 0][0], [1 / 3, 1 / 6, 0, 0])
    np.testing.assert_allclose(ah[:, :, 2], np.eye(3) / 3)
    # slice-constant operators have exactly-zero detail blocks
    pyr = W.forward_w(av, 2)
    assert all(not d.any() for d in pyr.details)


def test_config5_deblur_full_size():
    """BASELINE configs[4]: 512x512x128, 12 endmembers, 9x9 Gaussian PSF sigma=2, L=3, tol 1e-3."""
    x, av, ah, eta = synth.deblur_problem()
    xd, avd, ahd, etad = (torch.from_numpy(t).cuda() for t in (x, av, ah, eta))
    b = imaging.blur(xd, avd, ahd, 3) + etad
    xr = imaging.deblur(b, avd, ahd, 3, "w", tol=1e-3)
    # oracle pipeline on the same bytes
    b_ref = O.w_product(O.w_product(av, x, 3), O.transpose(ah), 3) + eta
    assert relerr(b.cpu().numpy(), b_ref) < 1e-12
    left = O.pinv_w(av, 3, 1e-3)
    right = O.pinv_w(O.transpose(ah), 3, 1e-3)
    assert relerr(W.pinv_w(avd, 3, 1e-3).cpu().numpy(), left) < 1e-8
    xr_ref = O.w_product(O.w_product(left, b_ref, 3), right, 3)
    xr_h = xr.cpu().numpy()
    assert relerr(xr_h, xr_ref) < 1e-8
    assert abs(imaging.psnr(xd, xr) - O.psnr(x, xr_ref)) < 1e-6
    assert abs(imaging.ssim(xd, xr) - O.ssim(x, xr_ref)) < 1e-6
    # deblur-w == deblur-spw for slice-constant operators
    xs = imaging.deblur(b, avd, ahd, 3, "spw", tol=1e-3)
    assert relerr(xs.cpu().numpy(), xr_h) < 1e-12


def test_deblur_t_method_matches_oracle():
    """SPEC.md:495-499 method t: t_pinv sandwich under the t-product (the paper's comparator)."""
    x, av, ah, eta = synth.deblur_problem(n=96, p=24, endmembers=6, noise=0.005)
    b = O.t_product(O.t_product(av, x), O.transpose(ah)) + eta
    got = imaging.deblur(b, av, ah, 3, "t", tol=1e-3)
    left = O.t_pinv(av, 1e-3)
    right = O.t_pinv(O.transpose(ah), 1e-3)
    want = O.t_product(O.t_product(left, b), right)
    assert relerr(got, want) < 1e-8
    assert abs(imaging.psnr(x, got) - O.psnr(x, want)) < 1e-6
    # the slice-constant operator's t-pseudo-inverse is itself slice-constant
    tp = W.baselines.t_pinv(av, 1e-3)
    assert np.abs(tp - tp[:, :, :1]).max() <= 1e-15 * np.abs(tp).max()


def test_ac9_blur_semantics_follow_the_reference_code():
    """SPEC.md:489-503 claims blur == per-band A_v X_k A_h^T and deblur(blur(x)) ~ x.
    Under the reference's lazy-wavelet w-product a slice-constant operator has zero
    detail blocks, so the product keeps only the smooth (band-averaged) content:
    the blurred cube is piecewise constant over 2^L-band groups and the SPEC claims
    do not hold for the shipped code (code governs).  We pin
    the code's behaviour: oracle parity, the piecewise-constant structure, and
    deblur-w == deblur-spw."""
    rng = np.random.default_rng(9)
    x = rng.random((64, 64, 8))
    av, ah = imaging.blur_operator(3, 3, 64, 64, 8)
    b = imaging.blur(x, av, ah, 3)
    want = O.w_product(O.w_product(av, x, 3), O.transpose(ah), 3)
    assert relerr(b, want) < 1e-12
    assert np.abs(b - b[:, :, :1]).max() <= 1e-12 * np.abs(b).max()     # constant over the 8 bands
    per_band = np.stack([av[:, :, 0] @ x[:, :, k] @ ah[:, :, 0].T for k in range(8)], axis=2)
    assert relerr(b.mean(axis=2), per_band.mean(axis=2)) < 1e-12         # = per-band product of the band mean
    xw = imaging.deblur(b, av, ah, 3, "w")
    assert relerr(xw, imaging.deblur(b, av, ah, 3, "spw")) < 1e-12
    assert relerr(xw, np.broadcast_to(x.mean(axis=2, keepdims=True), x.shape)) < 1e-6


# ---- generator / operator construction on the GPU ----

def test_blur_operator_device_bit_identical():
    for (bv, bh, n1, n2, p) in [(2, 1, 4, 3, 4), (5, 7, 33, 70, 9), (3, 3, 128, 65, 32), (9, 2, 1, 1, 1)]:
        av, ah = imaging.blur_operator(bv, bh, n1, n2, p)
        avd, ahd = imaging.blur_operator(bv, bh, n1, n2, p, device="cuda")
        assert avd.is_cuda and tuple(avd.shape) == av.shape and tuple(ahd.shape) == ah.shape
        assert np.array_equal(avd.cpu().numpy(), av) and np.array_equal(ahd.cpu().numpy(), ah)


def test_toeplitz_operator_matches_host_psf_operator():
    for n, p in [(40, 6), (7, 5), (64, 16)]:
        ref = synth.slice_constant(synth.toeplitz_blur(n, 9, 2.0), p)
        got = imaging.toeplitz_operator(synth.gaussian_taps(9, 2.0)[4:], n, p)
        assert np.array_equal(got.cpu().numpy(), ref)
    assert tuple(imaging.toeplitz_operator([1.0], 0, 3).shape) == (0, 0, 3)


def test_gauss_smooth_matches_scipy_reflect():
    from scipy.ndimage import gaussian_filter

    from paper_2601_08228_b200 import engine as E

    rng = np.random.default_rng(5)
    w = torch.from_numpy(synth.gaussian_half_kernel(4.0)).cuda()
    for shape in [(50, 37, 3), (9, 70, 2), (5, 4, 1), (128, 96, 10)]:   # (9, ..) / (5, 4, ..): radius 16 > extent
        x = rng.random(shape)
        ref = np.stack([gaussian_filter(x[:, :, e], sigma=4, mode="reflect") for e in range(shape[2])], axis=2)
        got = E.gauss_smooth2d(torch.from_numpy(x).cuda(), w).cpu().numpy()
        assert np.abs(got - ref).max() <= 4e-16, shape


def test_hyperspectral_cube_device_matches_host_generator():
    for (n1, n2, p, e, seed) in [(48, 40, 24, 10, 0), (33, 21, 17, 12, 3)]:
        ref = synth.hyperspectral_cube(n1, n2, p, e, seed=seed)
        got = synth.hyperspectral_cube_device(n1, n2, p, e, seed=seed, noise_source="numpy")
        assert got.is_cuda and tuple(got.shape) == ref.shape
        assert np.abs(got.cpu().numpy() - ref).max() < 1e-13
    clean_ref = synth.hyperspectral_cube(32, 32, 16, noise=0.0)
    clean = synth.hyperspectral_cube_device(32, 32, 16, noise=0.0)
    assert np.abs(clean.cpu().numpy() - clean_ref).max() < 1e-13


def test_hyperspectral_cube_device_philox_noise():
    n1, n2, p = 96, 96, 64
    a = synth.hyperspectral_cube_device(n1, n2, p, seed=7)
    b = synth.hyperspectral_cube_device(n1, n2, p, seed=7)
    c = synth.hyperspectral_cube_device(n1, n2, p, seed=8)
    assert torch.equal(a, b) and not torch.equal(a, c)            # seeded, deterministic
    assert float(a.min()) >= 0.0 and float(a.max()) <= 1.0
    clean = synth.hyperspectral_cube_device(n1, n2, p, seed=7, noise=0.0)
    inside = (clean > 0.06) & (clean < 0.94)                        # 6 sigma from the clip bounds
    z = ((a - clean)[inside] / 0.01).cpu().numpy()
    assert z.size > 1e5
    assert abs(z.mean()) < 5 / np.sqrt(z.size) and abs(z.std() - 1.0) < 0.01
    assert abs(np.mean(z ** 3)) < 0.05 and abs(np.mean(z ** 4) - 3.0) < 0.1
    # neighbouring samples (the two Box-Muller outputs of one counter, and adjacent counters) uncorrelated
    flat = ((a - clean) / 0.01).reshape(-1)
    ok = (inside.reshape(-1)[:-1] & inside.reshape(-1)[1:])
    corr = float((flat[:-1] * flat[1:])[ok].mean())
    assert abs(corr) < 0.01
