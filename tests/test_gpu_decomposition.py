"""K4 (block-Jacobi SVD) + K5/K6/K7 epilogues on the GPU.

Bars (BASELINE.json north_star): singular values and rank-k reconstructions
within 1e-8 relative; sigma compared per slice as max|dsigma| / sigma_max.
Singular vectors carry sign/rotation freedom, so U, V are checked through the
invariants (U *_w S *_w V^T = recon, orthonormality), never entry-wise.
"""

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import engine as E
from paper_2601_08228_b200 import synth
from oracle import wten_oracle as O
from wt_helpers import relerr
from wt_paper_examples import MP, MP_A, MP_B

pytestmark = pytest.mark.gpu
TOL = 1e-8


def sigma_err(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    scale = np.maximum(want[:, :1], 1e-300)
    return float(np.max(np.abs(got - want) / scale)) if want.size else 0.0


@pytest.mark.parametrize("name,r,L", [("sq", 3, 2), ("wide", 4, 3), ("tall", 2, 4)])
def test_reference_fixtures(golden, name, r, L):
    g = golden("decomposition.npz")
    x = g[f"{name}_x"]
    f, rec = W.w_svd(x, r, L)
    assert [t for t, _ in f.sigma_table] == [f"d{j}" for j in range(1, L + 1)] + ["s"]
    for tag, s in f.sigma_table:
        assert sigma_err(s, g[f"{name}_sigma_{tag}"]) < 1e-12
    assert relerr(rec, g[f"{name}_recon"]) < 1e-10
    assert relerr(f.S, g[f"{name}_S"]) < 1e-12
    usv = W.w_product(W.w_product(f.U, f.S, L), W.transpose(f.V), L)
    assert relerr(usv, rec) < 1e-10
    assert abs(W.truncation_bound(f, r).bound - float(g[f"{name}_bound"])) < 1e-10
    assert relerr(W.sp_w_svd(x, r, L), g[f"{name}_sp"]) < 1e-10


def test_pinv_fixtures_and_counterexample(golden):
    g = golden("decomposition.npz")
    x = g["pinv_x"]
    assert relerr(W.pinv_w(x, 3), g["pinv_L3_default"]) < 1e-10
    assert relerr(W.pinv_w(x, 1, 1e-1), g["pinv_L1_tol1e-1"]) < 1e-10
    assert relerr(W.sp_pinv_w(x, 2), g["sp_pinv_L2"]) < 1e-10
    assert relerr(W.pinv_w_via_factors(x, 2), g["pinv_via_factors_L2"]) < 1e-9
    assert np.array_equal(W.pinv_w(np.zeros((4, 5, 4)), 2), g["pinv_zero"])
    # PAPER.md:604-704, printed values are exact
    ab = W.w_product(MP_A, MP_B, 1)
    c = W.pinv_w(ab, 1)
    assert np.abs(c - MP["C"]).max() < 1e-12
    d = W.w_product(W.pinv_w(MP_B, 1), W.pinv_w(MP_A, 1), 1)
    assert np.abs(d - MP["D"]).max() < 1e-12


@pytest.mark.parametrize("shape,r,L", [((40, 40, 8), 5, 3), ((30, 70, 4), 30, 2),
                                       ((70, 30, 4), 7, 1), ((1, 9, 4), 1, 2), ((65, 33, 16), 33, 4)])
def test_against_oracle_random(shape, r, L):
    x = np.random.default_rng(sum(shape) + r).standard_normal(shape)
    want = O.w_svd(x, r, L)
    f, rec = W.w_svd(x, r, L)
    for (t1, s1), (t2, s2) in zip(f.sigma_table, want["sigma_table"]):
        assert t1 == t2 and sigma_err(s1, s2) < 1e-12
    assert relerr(rec, want["recon"]) < 1e-10
    assert relerr(W.sp_w_svd(x, r, L), O.sp_w_svd(x, r, L)) < 1e-10
    assert relerr(W.pinv_w(x, L), O.pinv_w(x, L)) < 1e-9


def test_penrose_identities():
    x = np.random.default_rng(21).standard_normal((9, 6, 8))
    L = 2
    xp = W.pinv_w(x, L)
    wp = lambda a, b: W.w_product(a, b, L)  # noqa: E731
    assert relerr(wp(wp(x, xp), x), x) < 1e-10
    assert relerr(wp(wp(xp, x), xp), xp) < 1e-10
    axp = wp(x, xp)
    assert relerr(W.transpose(axp), axp) < 1e-10
    xpa = wp(xp, x)
    assert relerr(W.transpose(xpa), xpa) < 1e-10


def test_nan_raises_linalgerror_like_reference():
    a = np.ones((3, 3, 4))
    a[0, 0, 0] = np.nan
    with pytest.raises(np.linalg.LinAlgError, match="SVD did not converge"):
        W.w_svd(a, 1, 1)
    with pytest.raises(np.linalg.LinAlgError, match="SVD did not converge"):
        W.pinv_w(a, 1)


def test_engine_svd_orthogonality_and_sort():
    rng = np.random.default_rng(22)
    a = torch.from_numpy(rng.standard_normal((5, 100, 300))).cuda()
    sigma, vec, info = E.svd(a, 100)
    assert int(info.abs().sum()) == 0
    s = sigma.cpu().numpy()
    assert np.all(np.diff(s, axis=1) <= 0)
    v = vec.cpu().numpy()
    gram = v @ np.swapaxes(v, 1, 2)
    assert np.abs(gram - np.eye(100)).max() < 1e-12
    want = np.linalg.svd(a.cpu().numpy(), compute_uv=False)
    assert sigma_err(s, want) < 1e-13


def test_config3_full_size():
    """w-svd rank 20 of the 256x256x192 hyperspectral cube, L=3 (BASELINE config 3)."""
    x = synth.hyperspectral_cube(256, 256, 192, endmembers=10, seed=0)
    want = O.w_svd(x, 20, 3)
    f, rec = W.w_svd(torch.from_numpy(x).cuda(), 20, 3)
    for (t1, s1), (t2, s2) in zip(f.sigma_table, want["sigma_table"]):
        assert t1 == t2 and sigma_err(s1.cpu().numpy(), s2) < TOL
    assert relerr(rec.cpu().numpy(), want["recon"]) < TOL
    assert relerr(f.S.cpu().numpy(), want["S"]) < TOL
    assert abs(O.psnr(x, rec.cpu().numpy()) - O.psnr(x, want["recon"])) < 1e-6
    assert abs(O.ssim(x, rec.cpu().numpy()) - O.ssim(x, want["recon"])) < 1e-6


def test_config4_full_size():
    """sp-w-svd rank 30 of the 1024x1024x256 cube, L=4 (BASELINE config 4)."""
    x = synth.hyperspectral_cube(1024, 1024, 256, endmembers=10, seed=0)
    want = O.sp_w_svd(x, 30, 4)
    got = W.sp_w_svd(torch.from_numpy(x).cuda(), 30, 4).cpu().numpy()
    assert relerr(got, want) < TOL
    # piecewise constant in blocks of 2^(L-1) bands (finer details zeroed)
    assert np.array_equal(got[..., 0::8], got[..., 7::8])
    # the numpy drop-in call streams the cube through the GPU in row chunks
    # (engine.host_slices_pipeline): same kernels on the same bytes -> same bits
    assert np.array_equal(W.sp_w_svd(x, 30, 4), got)


def test_determinism():
    x = torch.from_numpy(np.random.default_rng(23).standard_normal((64, 64, 32))).cuda()
    r1 = W.sp_w_svd(x, 8, 2)
    r2 = W.sp_w_svd(x, 8, 2)
    assert torch.equal(r1, r2)


@pytest.mark.parametrize("knob", ["svd_persist", "svd_pair_skip"])
def test_scheduling_knobs_do_not_change_bits(knob):
    """K4's persistent dependency-scheduled sweeps and the clean-pair skip only
    change WHEN visits run or drop visits that rotate nothing: sigma and vectors
    are bit-identical with either switched off (one launch per round / every
    pair re-tested).  256 columns: cross-only rounds and 16 blocks.  The
    one-launch-per-round path has no cluster-split visits, so the comparison
    pins the split to 1 (a split changes the Gram's summation order)."""
    a = torch.from_numpy(np.random.default_rng(29).standard_normal((6, 300, 256))).cuda()
    outs = []
    with E.option("svd_split", 1):
        for v in (1, 0):
            with E.option(knob, v):
                sigma, vec, info = E.svd(a, 256)
                E.raise_if_failed(info)
                outs.append((sigma.clone(), vec.clone(), E.last_sweeps()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


@pytest.mark.parametrize("split", [1, 2, 4, 8, 0])
@pytest.mark.parametrize("precond", [1, 0])
def test_cluster_split_visits(split, precond):
    """Visits split over 2/4/8-CTA clusters (rows of the panel, partial Grams
    summed in rank order through distributed shared memory; 9 row chunks, so
    uneven row ranges), with and without the Gram-eigenbasis preconditioner:
    sigma against LAPACK, orthonormal vectors, and the clean-pair skip (decided
    by the cluster leader) leaves the bits unchanged."""
    rng = np.random.default_rng(31)
    a_np = rng.standard_normal((3, 520, 512)) * np.linspace(1.0, 1e-3, 512)
    a = torch.from_numpy(a_np).cuda()
    outs = []
    with E.option("svd_split", split), E.option("svd_precond", precond):
        for skip in (1, 0):
            with E.option("svd_pair_skip", skip):
                sigma, vec, info = E.svd(a, 512)
                E.raise_if_failed(info)
                outs.append((sigma.cpu().numpy(), vec.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    sigma, vec = outs[0]
    ref = np.linalg.svd(a_np, compute_uv=False)
    assert np.max(np.abs(sigma - ref) / ref[:, :1]) < 1e-12
    # long side (520) singular vectors, orthonormal
    for b in range(3):
        g = vec[b] @ vec[b].T
        assert np.max(np.abs(g - np.eye(512))) < 1e-11


@pytest.mark.parametrize("shape", [(1, 70, 130), (2, 200, 33), (5, 64, 64)])
def test_cluster_split_small_and_ragged(shape):
    """Forced 8-CTA clusters on panels with fewer row chunks than CTAs (the host
    clamps the split to one chunk per CTA), wide and tall slices."""
    a_np = np.random.default_rng(sum(shape)).standard_normal(shape)
    with E.option("svd_split", 8):
        sigma, vec, info = E.svd(torch.from_numpy(a_np).cuda(), min(shape[1:]))
    E.raise_if_failed(info)
    assert sigma_err(sigma.cpu().numpy(), np.linalg.svd(a_np, compute_uv=False)) < 1e-12


def test_concurrent_host_threads_on_own_streams():
    """The API is pure (SPEC concurrency sections): host threads driving their own
    CUDA streams get the serial results bit for bit (per-thread host state in K4)."""
    import threading

    xs = [np.random.default_rng(50 + i).standard_normal((48, 40, 16)) for i in range(4)]
    serial = [W.sp_w_svd(x, 5, 2) for x in xs] + [W.pinv_w(x, 2) for x in xs]
    out = [None] * (2 * len(xs))
    errs = []

    def work(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[i] = W.sp_w_svd(xs[i], 5, 2)
                out[len(xs) + i] = W.pinv_w(xs[i], 2)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for a, b in zip(out, serial):
        assert np.array_equal(a, b)


def test_batches_above_grid_limit():
    """K4 and the epilogue kernels chunk batches above 65535 matrices internally."""
    rng = np.random.default_rng(61)
    a = rng.standard_normal((70001, 3, 2))
    at = torch.from_numpy(a).cuda()
    sigma, vec, info = E.svd(at, 2)
    assert int(info.abs().max()) == 0
    np.testing.assert_allclose(sigma.cpu().numpy(), np.linalg.svd(a, compute_uv=False), rtol=0, atol=1e-13)
    pinv = E.pinv_blocks(at, sigma, vec, 1e-12).cpu().numpy()
    np.testing.assert_allclose(pinv, np.linalg.pinv(a), rtol=0, atol=1e-10)
    rec = E.truncated_recon(at, sigma, vec, 2).cpu().numpy()
    np.testing.assert_allclose(rec, a, rtol=0, atol=1e-12)


@pytest.mark.parametrize("n1,n2", [(40, 24), (24, 40), (33, 33)])
def test_ranked_pinv_matches_full_and_oracle(n1, n2):
    """K7 with per-slice rank limits (wt_pinv_from_svd_ranked_f64, used by pinv_blocks):
    zero slices, rank-deficient slices and tol cutoffs give the same bits as the
    full-width assembly (wt_pinv_from_svd_f64) and match the oracle's _pinv_stack."""
    from paper_2601_08228_b200 import _native as N

    rng = np.random.default_rng(5)
    k = 9
    a = rng.standard_normal((k, n1, n2))
    a[1] = 0.0                                                    # all-zero slice: rank 0
    a[2] = np.outer(rng.standard_normal(n1), rng.standard_normal(n2))  # rank 1
    q = min(n1, n2)
    u = np.linalg.qr(rng.standard_normal((n1, q)))[0]
    v = np.linalg.qr(rng.standard_normal((n2, q)))[0]
    a[3] = (u * np.logspace(0, -6, q)) @ v.T                      # graded: cutoff inside
    ad = torch.from_numpy(a).cuda()
    for tol in (1e-12, 1e-3):
        sigma, vec, info = E.svd(ad, q)
        E.raise_if_failed(info)
        got = E.pinv_blocks(ad, sigma, vec, tol).cpu().numpy()
        full = torch.empty((k, n2, n1), dtype=torch.float64, device="cuda")
        t = torch.empty((k, q, q), dtype=torch.float64, device="cuda")
        lib = N.require_gpu()
        N.check(lib.wt_pinv_from_svd_f64(ad.data_ptr(), n2, n1 * n2, n1, n2, k, sigma.data_ptr(),
                                         vec.data_ptr(), tol, full.data_ptr(), n1, n1 * n2,
                                         t.data_ptr(), torch.cuda.current_stream().cuda_stream),
                "wt_pinv_from_svd_f64")
        assert np.array_equal(got, full.cpu().numpy())
        assert not got[1].any()
        want = np.stack([O.pinv_stack(a[i][:, :, None], tol)[:, :, 0] for i in range(k)])
        assert relerr(got, want) < 1e-8


@pytest.mark.parametrize("n1,n2", [(2048, 2048), (700, 2100)])
def test_large_slices_against_lapack(n1, n2):
    """Large single slices: 128 column blocks (the largest with the clean-pair
    records) and 2100 columns (132 blocks: records off), against LAPACK."""
    rng = np.random.default_rng(31)
    a = rng.standard_normal((1, n1, n2))
    a[0, :, ::7] *= 1e-3                                   # a graded spectrum
    sigma, vec, info = E.svd(torch.from_numpy(a).cuda(), 8)
    E.raise_if_failed(info)
    want = np.linalg.svd(a[0], compute_uv=False)[None]
    assert sigma_err(sigma.cpu().numpy(), want) < TOL


def test_sweep_limit_raises_linalgerror_like_dgesdd():
    """K4 info == 2 (no convergence within max_sweeps) raises LinAlgError('SVD did not
    converge') like np.linalg.svd when dgesdd fails (decomposition.py:66)."""
    a = torch.from_numpy(np.random.default_rng(0).standard_normal((2, 64, 64))).cuda()
    sigma, vec, info = E.svd(a, 0, max_sweeps=1)
    assert int(info.max()) == 2
    with pytest.raises(np.linalg.LinAlgError, match="SVD did not converge"):
        E.raise_if_failed(info)


def test_pinv_tiny_and_huge_scales():
    """pinv of 1e-160 * I and 1e+150 * I: 1/s is applied twice on the operands, never
    squared (1/s^2 overflows below ~1.5e-154 and underflows above ~1e154)."""
    ident = W.identity_tensor(4, 8, 2)
    for scale in (1e-160, 1e150):
        a = ident * scale
        x = W.pinv_w(a, 2)
        assert np.all(np.isfinite(x))
        assert relerr(x * scale, ident) < 1e-12
        y = W.inverse_tensor(a, 2)
        assert relerr(y * scale, ident) < 1e-12


def test_sp_pinv_w_empty():
    for shape in [(0, 3, 4), (3, 0, 4)]:
        out = W.sp_pinv_w(np.zeros(shape), 1)
        assert out.shape == (shape[1], shape[0], shape[2]) and not out.any()


@pytest.mark.parametrize("shape,r", [((6, 256, 256), 20), ((3, 300, 512), 30), ((2, 520, 256), 8)])
def test_topk_truncation_matches_full_and_lapack(shape, r):
    """K4's leading-triplet mode (wt_svd_topk_f64, used by sp_w_svd's rank-r truncation):
    the k leading singular values equal the full K4's / LAPACK's, the rank-r
    reconstruction equals the full path's and LAPACK's; graded and noise-like slices."""
    rng = np.random.default_rng(sum(shape) + r)
    a = rng.standard_normal(shape)
    a[0] = (np.linalg.qr(rng.standard_normal((shape[1], shape[1])))[0][:, :min(shape[1:])]
            * np.logspace(0, -9, min(shape[1:]))) @ np.linalg.qr(rng.standard_normal((shape[2], min(shape[1:]))))[0].T
    at = torch.from_numpy(a).cuda()
    k = E.topk_width(min(shape[1:]), r)
    assert k >= 2 * r
    s_k, v_k, info = E.svd_topk(at, k, r)
    E.raise_if_failed(info)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(s_k.cpu().numpy() - ref[:, :k]) / ref[:, :1]) < 1e-12
    rec = E.svd_truncated_recon(at, r).cpu().numpy()
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    want = u[:, :, :r] @ (s[:, :r, None] * vh[:, :r, :])
    assert relerr(rec, want) < 1e-10
    s_f, v_f, _ = E.svd(at, r)
    full = E.truncated_recon(at, s_f, v_f, r).cpu().numpy()
    assert relerr(rec, full) < 1e-10


@pytest.mark.parametrize("shape,rank", [((6, 123, 245), 60), ((6, 245, 123), 41), ((4, 100, 100), 30),
                                        ((3, 200, 300), 50), ((2, 640, 512), 100)])
def test_rank_deficient_slices_with_many_null_columns_converge(shape, rank):
    """More numerically-null columns than one pair visit holds (32): the visits made of null columns
    only must not keep the sweeps alive (found by tools/fuzz_parity.py on 123 x 245 rank-82 detail
    slices: 40 sweeps without progress, LinAlgError).  Singular values vs LAPACK, orthonormal factor
    blocks and the reconstruction through the public API."""
    rng = np.random.default_rng(sum(shape) + rank)
    b, m, n = shape
    a = rng.standard_normal((b, m, rank)) @ rng.standard_normal((b, rank, n))
    at = torch.from_numpy(a).cuda()
    q = min(m, n)
    sig, vec, info = E.svd(at, q)
    E.raise_if_failed(info)
    assert E.last_sweeps() <= 30  # (plain Jacobi below 128 columns: 12-17 sweeps on full-rank slices, ~22 here)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.abs(sig.cpu().numpy() - ref).max() <= 1e-12 * ref.max()
    cube = np.ascontiguousarray(np.moveaxis(a, 0, 2))[:, :, : 2 * (b // 2)]     # (m, n, p), p even
    want = O.w_svd(cube, rank // 2, 1)
    f, rec = W.w_svd(cube, rank // 2, 1)
    assert relerr(rec, want["recon"]) < TOL
    full, rec_full = W.w_svd(cube, q, 1)                                         # every triplet, null ones included
    assert relerr(rec_full, cube) < 1e-10
    for blk in (full.U, full.V):
        pyr = W.forward_w(blk, 1)
        for st in [pyr.smooth] + list(pyr.details):
            for k in range(st.shape[2]):
                g = st[:, :, k].T @ st[:, :, k]
                assert np.abs(g - np.eye(g.shape[0])).max() < 1e-10


def test_truncation_with_null_triplets_whose_noise_vector_is_parallel_to_a_real_one():
    """Two parallel columns: the third Jacobi column is exactly-proportional noise (norm 1e-32) whose
    normalised direction equals a real left vector.  K4 completes null vectors orthonormally, so the
    rank-q truncation (projector U_r U_r^T A) counts no direction twice (tools/fuzz_parity.py seed 1
    case 294: the reconstruction doubled a row)."""
    a = np.zeros((12, 3, 4))
    rng = np.random.default_rng(3)
    for k in range(4):
        a[2, 1, k], a[2, 2, k] = rng.standard_normal(2)          # columns 1, 2 both multiples of e_2
        a[[4, 8, 9], 0, k] = rng.standard_normal(3)
    for L in (1, 2):
        for r in (2, 3):
            want = O.w_svd(a, r, L)
            f, rec = W.w_svd(a, r, L)
            assert relerr(rec, want["recon"]) < TOL
            assert relerr(W.sp_w_svd(a, r, L), O.sp_w_svd(a, r, L)) < TOL
            at = np.ascontiguousarray(np.transpose(a, (1, 0, 2)))   # wide slices: the right-vector side
            assert relerr(W.w_svd(at, r, L)[1], O.w_svd(at, r, L)["recon"]) < TOL
    sig, vec, info = E.svd(torch.from_numpy(np.ascontiguousarray(np.moveaxis(a, 2, 0))).cuda(), 3)
    v = vec.cpu().numpy()
    for b in range(v.shape[0]):
        assert np.abs(v[b] @ v[b].T - np.eye(3)).max() < 1e-12
