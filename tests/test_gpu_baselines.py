"""GPU parity of the comparator products (t-product, m-product, t-svd, t-pinv)
against the reference's own outputs (tests/golden/baselines.npz) and the oracle
(numpy FFT + LAPACK restatement of baselines.py).  Tolerance: 1e-10 relative,
the SPEC's t-product accuracy contract."""

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu
B = W.baselines
TOL = 1e-10


@pytest.mark.parametrize("name", ["t1", "t2", "t3", "t4", "t5"])
def test_products_match_reference_fixtures(golden, name):
    g = golden("baselines.npz")
    a, b = g[f"{name}_a"], g[f"{name}_b"]
    got = B.t_product(a, b)
    assert isinstance(got, np.ndarray) and got.flags.c_contiguous
    assert relerr(got, g[f"{name}_t"]) < TOL
    if f"{name}_m" in g.files:
        assert relerr(B.m_product(a, b, B.dct_transform(a.shape[2])), g[f"{name}_m"]) < TOL


@pytest.mark.parametrize("name,r", [("s1", 2), ("s2", 3), ("s3", 7)])
def test_t_svd_t_pinv_match_reference_fixtures(golden, name, r):
    g = golden("baselines.npz")
    x = g[f"{name}_x"]
    assert relerr(B.t_svd(x, r), g[f"{name}_tsvd"]) < TOL
    assert relerr(B.t_pinv(x), g[f"{name}_tpinv"]) < TOL
    assert relerr(B.t_pinv(x, 1e-1), g[f"{name}_tpinv_1e-1"]) < TOL


def test_identities_and_constant_tubes(golden):
    g = golden("baselines.npz")
    assert np.array_equal(B.tube_identity(3, 5), g["tube_identity_3_5"])
    assert np.abs(B.m_identity(3, 6, B.dct_transform(6)) - g["m_identity_3_6"]).max() < 1e-14
    assert relerr(B.t_pinv(g["const_x"]), g["const_tpinv"]) < TOL
    assert relerr(B.t_svd(g["const_x"], 2), g["const_tsvd_2"]) < TOL


@pytest.mark.parametrize("shape", [(64, 48, 40, 32), (33, 17, 70, 102), (128, 96, 80, 7), (5, 130, 3, 1)])
def test_t_product_vs_oracle(shape):
    n1, n2, n3, p = shape
    rng = np.random.default_rng(n1 * p)
    a = rng.standard_normal((n1, n2, p))
    b = rng.standard_normal((n2, n3, p))
    assert relerr(B.t_product(a, b), O.t_product(a, b)) < TOL
    # the tube identity is the neutral element
    assert relerr(B.t_product(a, B.tube_identity(n2, p)), a) < TOL


@pytest.mark.parametrize("seed", range(5))
def test_t_product_block_circulant_small(seed):
    """all shapes <= 6 x 6 x 8 agree with brute-force block-circulant products."""
    rng = np.random.default_rng(100 + seed)
    for _ in range(20):
        n1, n2, n3 = (int(v) for v in rng.integers(1, 7, size=3))
        p = int(rng.integers(1, 9))
        a = rng.standard_normal((n1, n2, p))
        b = rng.standard_normal((n2, n3, p))
        assert relerr(B.t_product(a, b), O.t_product_circulant(a, b)) < TOL


def test_m_product_properties():
    """identity element, associativity and bilinearity with the DCT."""
    rng = np.random.default_rng(7)
    p = 24
    tr = B.dct_transform(p)
    a = rng.standard_normal((20, 16, p))
    b = rng.standard_normal((16, 12, p))
    c = rng.standard_normal((12, 9, p))
    m = tr.M
    assert relerr(B.m_product(a, b, tr), O.m_product(a, b, m, m.T)) < TOL
    assert relerr(B.m_product(a, B.m_identity(16, p, tr), tr), a) < TOL
    ab_c = B.m_product(B.m_product(a, b, tr), c, tr)
    a_bc = B.m_product(a, B.m_product(b, c, tr), tr)
    assert relerr(ab_c, a_bc) < TOL
    b2 = rng.standard_normal(b.shape)
    lin = B.m_product(a, 2.0 * b - 3.0 * b2, tr)
    assert relerr(lin, 2.0 * B.m_product(a, b, tr) - 3.0 * B.m_product(a, b2, tr)) < TOL
    ident = B.ModeTransform(kind="matrix", M=np.eye(p), Minv=np.eye(p))
    assert relerr(B.m_product(a, b, ident), O.face_matmul(a, b)) < TOL


@pytest.mark.parametrize("shape,r", [((40, 30, 12), 5), ((24, 36, 9), 24), ((50, 20, 16), 1)])
def test_t_svd_vs_oracle(shape, r):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    assert relerr(B.t_svd(x, r), O.t_svd(x, r)) < TOL


def test_t_svd_full_rank_is_identity():
    x = np.random.default_rng(3).standard_normal((12, 9, 10))
    assert relerr(B.t_svd(x, 9), x) < TOL


@pytest.mark.parametrize("shape,tol", [((24, 24, 16), 1e-12), ((30, 20, 10), 1e-3), ((16, 40, 7), 1e-12)])
def test_t_pinv_vs_oracle(shape, tol):
    rng = np.random.default_rng(shape[0] + shape[2])
    x = rng.standard_normal(shape)
    got = B.t_pinv(x, tol)
    assert got.shape == (shape[1], shape[0], shape[2])
    assert relerr(got, O.t_pinv(x, tol)) < TOL


def test_t_pinv_zero_and_device_roundtrip():
    z = B.t_pinv(np.zeros((4, 5, 6)))
    assert z.shape == (5, 4, 6) and not np.any(z)
    x = np.random.default_rng(9).standard_normal((10, 8, 6))
    xd = torch.from_numpy(x).cuda()
    got = B.t_pinv(xd)
    assert isinstance(got, torch.Tensor) and got.is_cuda
    assert relerr(got.cpu().numpy(), O.t_pinv(x)) < TOL
    prod = B.t_product(xd, torch.from_numpy(B.tube_identity(8, 6)).cuda())
    assert prod.is_cuda and relerr(prod.cpu().numpy(), x) < TOL


def test_t_svd_nan_raises_like_lapack():
    x = np.ones((3, 3, 4))
    x[0, 0, 0] = np.nan
    with pytest.raises(np.linalg.LinAlgError):
        B.t_svd(x, 1)
