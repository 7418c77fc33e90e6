"""K3 (DMMA GEMM) and the w-product on the GPU against the reference fixtures
and the oracle.  Bar (BASELINE.json north_star): w-product within 1e-10
relative Frobenius error in float64."""

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import engine as E
from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu
TOL = 1e-10


def test_config1_against_reference_fixture(golden):
    g = golden("w_product.npz")
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (64, 48, 32))
    b = rng.uniform(-1, 1, (48, 40, 32))
    c = W.w_product(a, b, 1)
    assert isinstance(c, np.ndarray) and c.shape == (64, 40, 32)
    assert relerr(c, g["cfg1_c"]) < TOL
    # transform round trips of both operands (config 1 parity list)
    for t in (a, b):
        assert relerr(W.inverse_w(W.forward_w(t, 1)), t) < 1e-15
    for L in (1, 2, 3):
        assert relerr(W.w_product(g["small_a"], g["small_b"], L), g[f"small_c_L{L}"]) < TOL


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("mnk", [(1, 1, 1), (7, 5, 3), (33, 65, 17), (130, 129, 200), (256, 256, 64)])
def test_gemm_all_orientations(ta, tb, mnk):
    M, Nn, K = mnk
    rng = np.random.default_rng(M * 7 + Nn * 3 + K)
    batch = 3
    a = rng.standard_normal((batch, K, M) if ta else (batch, M, K))
    b = rng.standard_normal((batch, Nn, K) if tb else (batch, K, Nn))
    c0 = rng.standard_normal((batch, M, Nn))
    opa = np.swapaxes(a, 1, 2) if ta else a
    opb = np.swapaxes(b, 1, 2) if tb else b
    want = 0.5 * (opa @ opb) - 2.0 * c0
    cd = torch.from_numpy(c0).cuda()
    E.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), ta, tb, alpha=0.5, beta=-2.0, out=cd)
    assert relerr(cd.cpu().numpy(), want) < 1e-14


@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("shape", [(200, 130, 70, 66), (160, 256, 192, 100), (3, 1030, 1034, 72), (1, 2048, 2048, 64)])
def test_gemm_tensor_map_variant(ta, tb, shape):
    """K3's tensor-map (TMA) variant: ragged even sizes (zero-filled edge boxes and K tails), strided
    row pitches, batch 1, both warp tilings -- against numpy and against the cp.async kernel."""
    batch, M, Nn, K = shape
    rng = np.random.default_rng(M + 3 * Nn + 5 * K + ta + 2 * tb)
    pad = 6  # row pitch larger than the extent: operands are views of wider buffers
    abuf = rng.standard_normal((batch, K, M + pad) if ta else (batch, M, K + pad))
    bbuf = rng.standard_normal((batch, Nn, K + pad) if tb else (batch, K, Nn + pad))
    at = torch.from_numpy(abuf).cuda()[:, :, :(M if ta else K)]
    bt = torch.from_numpy(bbuf).cuda()[:, :, :(K if tb else Nn)]
    a = abuf[:, :, :(M if ta else K)]
    b = bbuf[:, :, :(K if tb else Nn)]
    c0 = rng.standard_normal((batch, M, Nn))
    opa = np.swapaxes(a, 1, 2) if ta else a
    opb = np.swapaxes(b, 1, 2) if tb else b
    want = 1.5 * (opa @ opb) + 0.25 * c0
    got = {}
    for tma in (1, 0):
        with E.option("gemm_tma", tma):
            cd = torch.from_numpy(c0).cuda()
            E.gemm(at, bt, ta, tb, alpha=1.5, beta=0.25, out=cd)
            got[tma] = cd.cpu().numpy()
    assert relerr(got[1], want) < 1e-14
    assert relerr(got[1], got[0]) < 1e-15


def test_gemm_config5_size():
    rng = np.random.default_rng(9)
    a = rng.standard_normal((128, 512, 512))
    b = rng.standard_normal((128, 512, 512))
    c = E.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    assert relerr(c, a @ b) < 1e-14


def test_w_product_matches_oracle_config5_shape():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((512, 512, 128))
    b = rng.standard_normal((512, 512, 128))
    want = O.w_product(a, b, 3)
    got = W.w_product(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), 3)
    assert relerr(got.cpu().numpy(), want) < TOL


def test_slicewise_transpose_identity_face_product():
    rng = np.random.default_rng(12)
    a = rng.standard_normal((6, 4, 8))
    b = rng.standard_normal((4, 5, 8))
    assert relerr(W.slicewise_matmul(a, b), O.face_matmul(a, b)) < 1e-15
    assert np.array_equal(W.transpose(a), O.transpose(a))
    ident = W.identity_tensor(6, 8, 3)
    assert relerr(W.w_product(ident, a, 3), a) < 1e-14
    pa, pb = W.forward_w(a, 2), W.forward_w(b, 2)
    fp = W.face_product(pa, pb)
    assert relerr(W.inverse_w(fp), O.w_product(a, b, 2)) < 1e-14
    # device pyramids take the packed fast path
    da, db = W.forward_w(torch.from_numpy(a).cuda(), 2), W.forward_w(torch.from_numpy(b).cuda(), 2)
    assert relerr(W.inverse_w(W.face_product(da, db)).cpu().numpy(), O.w_product(a, b, 2)) < 1e-14


def test_w_product_laws():
    rng = np.random.default_rng(13)
    a = rng.standard_normal((5, 4, 16))
    b = rng.standard_normal((4, 6, 16))
    c = rng.standard_normal((6, 3, 16))
    for L in (1, 2, 4):
        ab_c = W.w_product(W.w_product(a, b, L), c, L)
        a_bc = W.w_product(a, W.w_product(b, c, L), L)
        assert relerr(ab_c, a_bc) < 1e-12                      # associativity
        lhs = W.transpose(W.w_product(a, b, L))
        rhs = W.w_product(W.transpose(b), W.transpose(a), L)
        assert relerr(lhs, rhs) < 1e-12                        # transpose reversal
        assert relerr(W.w_product(2 * a + a, b, L), 3 * W.w_product(a, b, L)) < 1e-12


def test_nan_propagates_silently_like_reference():
    a = np.ones((3, 3, 4))
    a[0, 0, 0] = np.nan
    c = W.w_product(a, np.ones((3, 2, 4)), 1)
    assert np.isnan(c).any()


def test_determinism():
    rng = np.random.default_rng(14)
    a = torch.from_numpy(rng.standard_normal((96, 80, 64))).cuda()
    b = torch.from_numpy(rng.standard_normal((80, 72, 64))).cuda()
    assert torch.equal(W.w_product(a, b, 3), W.w_product(a, b, 3))


def test_ring_constructors_match_reference(golden):
    import json
    import os

    from wt_helpers import GOLDEN

    g = golden("ring.npz")
    assert relerr(W.inverse_tensor(g["inv_x"], 2), g["inv_L2"]) < 1e-10
    assert relerr(W.inverse_tensor(g["inv_x"], 3), g["inv_L3"]) < 1e-10
    assert relerr(W.identity_tensor(4, 8, 2), g["identity_4_8_2"]) < 1e-15
    assert relerr(W.orthogonal_tensor(g["orth_q"], 8, 3), g["orth_5_8_3"]) < 1e-14
    errs = {e["call"]: e for e in json.load(open(os.path.join(GOLDEN, "errors.json")))["errors"]}
    gi = golden("ring_inputs.npz")
    for name, call in (("sing", "inverse_tensor(singular smooth)"),
                       ("sing_d2", "inverse_tensor(zero d2 slice 0)")):
        with pytest.raises(W.SingularSliceError) as ei:
            W.inverse_tensor(gi[name], 2)
        assert (ei.value.level, ei.value.slice_index) == (errs[call]["level"], errs[call]["slice_index"])


@pytest.mark.parametrize("shape", [(7, 5, 3), (33, 17, 1), (64, 48, 32), (5, 9, 130)])
def test_transpose_one_pass_exact(shape):
    """wt_tube_transpose_f64: bit-exact slicewise transpose for odd / unit / even p,
    including a view whose data pointer is not 16-byte aligned."""
    x = np.random.default_rng(41).standard_normal(shape)
    assert np.array_equal(W.transpose(x), O.transpose(x))
    big = torch.from_numpy(np.random.default_rng(42).standard_normal((shape[0] + 1,) + shape[1:])).cuda()
    view = big[1:]  # contiguous, offset by one row of tubes
    assert torch.equal(W.transpose(view), view.permute(1, 0, 2).contiguous())


def test_inverse_tensor_follows_lu_semantics():
    """inverse_tensor raises only where np.linalg.inv does (an exactly zero LU pivot, or a
    non-finite inverse): finite ill-conditioned slices are inverted (algebra.py:77-83)."""
    from paper_2601_08228_b200.errors import SingularSliceError

    rng = np.random.default_rng(11)
    q = np.linalg.qr(rng.standard_normal((4, 4)))[0]
    ill = (q * np.array([1.0, 1e-3, 1e-7, 1e-12])) @ q.T          # cond 1e12, no zero pivot
    # wavelet domain (L = 1): smooth slices [ill, I], detail slices [2 I, ill^T]
    sm = np.stack([ill, np.eye(4)], axis=2)
    dt = np.stack([2 * np.eye(4), ill.T.copy()], axis=2)
    a = O.lift_inverse(sm, [dt])
    # a slice-constant cube has exactly zero detail slices: both raise, same (level, slice)
    with pytest.raises(ValueError):
        O.inverse_tensor(np.stack([ill] * 4, axis=2), 1)
    with pytest.raises(SingularSliceError):
        W.inverse_tensor(np.stack([ill] * 4, axis=2), 1)
    got = W.inverse_tensor(a, 1)                                      # reference inverts: no error
    want = O.inverse_tensor(a, 1)
    assert np.all(np.isfinite(got))
    assert relerr(got, want) < 1e-3                                    # agreement ~ eps * cond
    # smooth slice exactly singular (dyadic values: the round trip is exact), detail slice I
    sing = O.lift_inverse(np.array([[1.0, 2.0], [2.0, 4.0]])[:, :, None], [np.eye(2)[:, :, None]])
    with pytest.raises(SingularSliceError) as e:
        W.inverse_tensor(sing, 1)
    with pytest.raises(ValueError) as e2:
        O.inverse_tensor(sing, 1)
    assert (e.value.level, e.value.slice_index) == e2.value.args[0]


def test_one_call_w_product_graph_replay():
    """wt_w_product_f64: repeated calls with the same arguments replay a captured CUDA
    graph; the graph reads the buffers at replay time (in-place input updates are seen),
    and new arguments run eagerly.  Every result equals the oracle."""
    from paper_2601_08228_b200.algebra import w_product_device

    rng = np.random.default_rng(12)
    a = rng.uniform(-1, 1, (20, 12, 16))
    b = rng.uniform(-1, 1, (12, 9, 16))
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = torch.empty((20, 9, 16), dtype=torch.float64, device="cuda")
    for _ in range(4):  # eager, eager + capture, replay, replay
        w_product_device(ad, bd, 2, out=out)
        assert relerr(out.cpu().numpy(), O.w_product(a, b, 2)) < 1e-13
    a2 = rng.uniform(-1, 1, a.shape)
    ad.copy_(torch.from_numpy(a2))  # same pointer, new data
    w_product_device(ad, bd, 2, out=out)
    assert relerr(out.cpu().numpy(), O.w_product(a2, b, 2)) < 1e-13
    fresh = w_product_device(bd.transpose(0, 1).contiguous(), ad.transpose(0, 1).contiguous(), 2)
    assert relerr(fresh.cpu().numpy(), O.w_product(np.swapaxes(b, 0, 1), np.swapaxes(a2, 0, 1), 2)) < 1e-13
