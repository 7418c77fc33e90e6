"""Pin the CPU oracle (oracle/wten_oracle.py) before trusting it:
  * the paper's worked examples (exact),
  * golden fixtures produced by running the reference itself
    (tests/golden/make_golden.py),
  * the SPEC's known answers (max_levels, identity tube, PSNR examples).
CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import wten_oracle as O
from wt_helpers import GOLDEN, relerr
from wt_paper_examples import EX2, EX2_A, EX2_B, MP, MP_A, MP_B


def test_example2_every_intermediate():
    sa1, da1 = O.lift_forward(EX2_A, 1)
    sb1, db1 = O.lift_forward(EX2_B, 1)
    assert np.array_equal(sa1, EX2["A_s1"]) and np.array_equal(da1[0], EX2["A_d1"])
    assert np.array_equal(sb1, EX2["B_s1"]) and np.array_equal(db1[0], EX2["B_d1"])
    sa2, da2 = O.lift_forward(EX2_A, 2)
    sb2, db2 = O.lift_forward(EX2_B, 2)
    assert np.array_equal(sa2, EX2["A_s2"]) and np.array_equal(da2[1], EX2["A_d2"])
    assert np.array_equal(sb2, EX2["B_s2"]) and np.array_equal(db2[1], EX2["B_d2"])
    cd1 = O.face_matmul(da2[0], db2[0])
    cs2 = O.face_matmul(sa2, sb2)
    cd2 = O.face_matmul(da2[1], db2[1])
    assert np.array_equal(cd1, EX2["C_d1"])
    assert np.array_equal(cs2, EX2["C_s2"]) and np.array_equal(cd2, EX2["C_d2"])
    assert np.array_equal(O.lift_inverse(cs2, [cd2]), EX2["C_s1"])
    assert np.array_equal(O.w_product(EX2_A, EX2_B, 2), EX2["C"])


def test_moore_penrose_counterexample():
    sa, da = O.lift_forward(MP_A, 1)
    sb, db = O.lift_forward(MP_B, 1)
    assert np.array_equal(sa, MP["A_s"]) and np.array_equal(da[0], MP["A_d"])
    assert np.array_equal(sb, MP["B_s"]) and np.array_equal(db[0], MP["B_d"])
    ab = O.w_product(MP_A, MP_B, 1)
    s, d = O.lift_forward(ab, 1)
    assert np.allclose(s, MP["AB_s"], atol=1e-15) and np.allclose(d[0], MP["AB_d"], atol=1e-15)
    c = O.pinv_w(ab, 1)
    cs, cd = O.lift_forward(c, 1)
    assert np.abs(cs - MP["C_s"]).max() < 1e-12 and np.abs(cd[0] - MP["C_d"]).max() < 1e-12
    assert np.abs(c - MP["C"]).max() < 1e-12
    ap = O.pinv_w(MP_A, 1)
    bp = O.pinv_w(MP_B, 1)
    s, d = O.lift_forward(ap, 1)
    assert np.abs(s - MP["Apinv_s"]).max() < 1e-12 and np.abs(d[0] - MP["Apinv_d"]).max() < 1e-12
    s, d = O.lift_forward(bp, 1)
    assert np.abs(s - MP["Bpinv_s"]).max() < 1e-12 and np.abs(d[0] - MP["Bpinv_d"]).max() < 1e-12
    dd = O.w_product(bp, ap, 1)
    assert np.abs(dd - MP["D"]).max() < 1e-12


def test_lifting_matches_reference_fixtures(golden):
    g = golden("lifting.npz")
    meta = json.load(open(os.path.join(GOLDEN, "errors.json")))["lifting_cases"]
    for case in meta:
        ci = case["case"]
        x = g[f"c{ci}_x"]
        for L in case["levels"]:
            s, d = O.lift_forward(x, L)
            assert np.array_equal(s, g[f"c{ci}_L{L}_smooth"]), (ci, L)
            for j in range(1, L + 1):
                assert np.array_equal(d[j - 1], g[f"c{ci}_L{L}_d{j}"]), (ci, L, j)
            assert np.array_equal(O.lift_inverse(s, d), g[f"c{ci}_L{L}_inv"]), (ci, L)


def test_w_product_matches_reference_fixtures(golden):
    g = golden("w_product.npz")
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (64, 48, 32))
    b = rng.uniform(-1, 1, (48, 40, 32))
    assert np.array_equal(np.array([a.sum(), b.sum()]), g["cfg1_a_sum"])  # generator drift guard
    assert relerr(O.w_product(a, b, 1), g["cfg1_c"]) < 1e-14
    for L in (1, 2, 3):
        assert relerr(O.w_product(g["small_a"], g["small_b"], L), g[f"small_c_L{L}"]) < 1e-14


@pytest.mark.parametrize("name,r,L", [("sq", 3, 2), ("wide", 4, 3), ("tall", 2, 4)])
def test_decompositions_match_reference_fixtures(golden, name, r, L):
    g = golden("decomposition.npz")
    x = g[f"{name}_x"]
    out = O.w_svd(x, r, L)
    for tag, s in out["sigma_table"]:
        np.testing.assert_allclose(s, g[f"{name}_sigma_{tag}"], rtol=0, atol=1e-13)
    assert relerr(out["recon"], g[f"{name}_recon"]) < 1e-12
    assert relerr(out["S"], g[f"{name}_S"]) < 1e-12
    # U, V carry sign freedom: compare the product U *_w S *_w V^T
    usv = O.w_product(O.w_product(out["U"], out["S"], L), O.transpose(out["V"]), L)
    ref = O.w_product(O.w_product(g[f"{name}_U"], g[f"{name}_S"], L), O.transpose(g[f"{name}_V"]), L)
    assert relerr(usv, ref) < 1e-12
    assert abs(O.truncation_bound(out["sigma_table"], r) - float(g[f"{name}_bound"])) < 1e-12
    assert relerr(O.sp_w_svd(x, r, L), g[f"{name}_sp"]) < 1e-12


def test_pinv_matches_reference_fixtures(golden):
    g = golden("decomposition.npz")
    x = g["pinv_x"]
    assert relerr(O.pinv_w(x, 3), g["pinv_L3_default"]) < 1e-12
    assert relerr(O.pinv_w(x, 1, 1e-1), g["pinv_L1_tol1e-1"]) < 1e-12
    assert relerr(O.sp_pinv_w(x, 2), g["sp_pinv_L2"]) < 1e-12
    assert np.array_equal(O.pinv_w(np.zeros((4, 5, 4)), 2), g["pinv_zero"])


def test_max_levels_known_answers():
    errs = json.load(open(os.path.join(GOLDEN, "errors.json")))["errors"]
    for e in errs:
        if e["call"].startswith("max_levels(") and "value" in e:
            p = int(e["call"][len("max_levels("):-1])
            assert O.max_levels(p) == e["value"]


def test_spec_identity_tube_and_constant_tube():
    # tube [1,1] at L=1 is smooth 1.0? identity tube n=1,p=2 -> [1.5, 0.5]
    one = np.zeros((1, 1, 2))
    one[0, 0, :] = [1.0, 1.0]
    s, d = O.lift_forward(one, 1)
    assert s[0, 0, 0] == 1.0 and d[0][0, 0, 0] == 0.0  # constant tube -> zero detail
    ident = O.lift_inverse(np.ones((1, 1, 1)), [np.ones((1, 1, 1))])
    assert np.array_equal(ident[0, 0], [1.5, 0.5])
    ident4 = O.lift_inverse(np.ones((1, 1, 1)), [np.ones((1, 1, 2)), np.ones((1, 1, 1))])
    assert np.array_equal(ident4[0, 0], [2.0, 1.0, 1.0, 0.0])


def test_psnr_ssim_spec_examples():
    x1 = np.ones((2, 2, 2))
    x0 = np.zeros((2, 2, 2))
    assert O.psnr(x1, x0, 1.0) == 0.0
    y = np.random.default_rng(3).random((4, 5, 3))
    z = y + 0.01
    assert abs(O.psnr(y, y + 0.1, 1.0) - (O.psnr(y, y + 0.01, 1.0) - 20.0)) < 1e-9
    assert O.psnr(y, y) == float("inf")
    assert abs(O.ssim(y, y) - 1.0) < 1e-15
    # SPEC.md:532 "x2 = -x1 -> value < 0" holds for zero-mean bands; with a
    # non-zero mean both SSIM factors flip sign and the product is positive.
    yc = y - y.mean(axis=(0, 1), keepdims=True)
    assert O.ssim(yc, -yc, 1.0) < 0
    assert abs(O.ssim(z, z) - 1.0) < 1e-15


def test_ring_constructors_match_reference_fixtures(golden):
    g = golden("ring.npz")
    x = g["inv_x"]
    assert relerr(O.inverse_tensor(x, 2), g["inv_L2"]) < 1e-12
    assert relerr(O.inverse_tensor(x, 3), g["inv_L3"]) < 1e-12
    eye = lambda k: np.broadcast_to(np.eye(6)[:, :, None], (6, 6, k)).copy()  # noqa: E731
    ident = O.lift_inverse(eye(2), [eye(4), eye(2)])  # every wavelet block = I (algebra.py:54-59)
    assert relerr(O.w_product(x, O.inverse_tensor(x, 2), 2), ident) < 1e-12
    gi = golden("ring_inputs.npz")
    for name, want in (("sing", (0, 0)), ("sing_d2", (2, 0))):
        with pytest.raises(ValueError) as ei:
            O.inverse_tensor(gi[name], 2)
        assert ei.value.args[0] == want


# ------------------------------------------------ comparator products ----

BL_PRODUCTS = ["t1", "t2", "t3", "t4", "t5"]


@pytest.mark.parametrize("name", BL_PRODUCTS)
def test_t_and_m_product_match_reference_fixtures(golden, name):
    g = golden("baselines.npz")
    a, b = g[f"{name}_a"], g[f"{name}_b"]
    assert relerr(O.t_product(a, b), g[f"{name}_t"]) < 1e-13
    if f"{name}_m" in g.files:
        m = O.dct_matrix(a.shape[2])
        assert np.abs(m - g[f"{name}_dct"]).max() < 1e-14
        assert relerr(O.m_product(a, b, m, m.T), g[f"{name}_m"]) < 1e-13


@pytest.mark.parametrize("seed", range(20))
def test_t_product_equals_block_circulant_product(seed):
    """FFT t-product == brute-force block-circulant product to 1e-10."""
    rng = np.random.default_rng(seed)
    n1, n2, n3 = (int(v) for v in rng.integers(1, 7, size=3))
    p = int(rng.integers(1, 9))
    a = rng.standard_normal((n1, n2, p))
    b = rng.standard_normal((n2, n3, p))
    assert relerr(O.t_product(a, b), O.t_product_circulant(a, b)) < 1e-10


@pytest.mark.parametrize("name", ["s1", "s2", "s3"])
def test_t_svd_t_pinv_match_reference_fixtures(golden, name):
    g = golden("baselines.npz")
    x = g[f"{name}_x"]
    r = {"s1": 2, "s2": 3, "s3": 7}[name]
    assert relerr(O.t_svd(x, r), g[f"{name}_tsvd"]) < 1e-12
    assert relerr(O.t_pinv(x), g[f"{name}_tpinv"]) < 1e-12
    assert relerr(O.t_pinv(x, 1e-1), g[f"{name}_tpinv_1e-1"]) < 1e-12


def test_identities_and_constant_tubes_match_reference(golden):
    g = golden("baselines.npz")
    assert np.array_equal(O.tube_identity(3, 5), g["tube_identity_3_5"])
    m = O.dct_matrix(6)
    assert np.abs(O.m_identity(3, 6, m.T) - g["m_identity_3_6"]).max() < 1e-14
    assert relerr(O.t_pinv(g["const_x"]), g["const_tpinv"]) < 1e-12
    assert relerr(O.t_svd(g["const_x"], 2), g["const_tsvd_2"]) < 1e-12
