"""K1/K2 parity on the GPU: bit-exact against the reference fixtures, the paper's
Example 2 and the CPU oracle, at small and full (config 2) sizes."""

import json
import os

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import _native as N
from paper_2601_08228_b200 import engine as E
from oracle import wten_oracle as O
from wt_helpers import GOLDEN
from wt_paper_examples import EX2, EX2_A, EX2_B

pytestmark = pytest.mark.gpu


def test_reference_fixtures_bit_exact(golden):
    g = golden("lifting.npz")
    meta = json.load(open(os.path.join(GOLDEN, "errors.json")))["lifting_cases"]
    for case in meta:
        ci = case["case"]
        x = g[f"c{ci}_x"]
        for L in case["levels"]:
            pyr = W.forward_w(x, L)
            assert isinstance(pyr.smooth, np.ndarray) and pyr.smooth.flags.c_contiguous
            assert np.array_equal(pyr.smooth, g[f"c{ci}_L{L}_smooth"]), (ci, L)
            for j in range(1, L + 1):
                assert np.array_equal(pyr.details[j - 1], g[f"c{ci}_L{L}_d{j}"]), (ci, L, j)
            assert np.array_equal(W.inverse_w(pyr), g[f"c{ci}_L{L}_inv"]), (ci, L)
            # device mode gives the same bytes
            dp = W.forward_w(torch.from_numpy(x).cuda(), L)
            assert np.array_equal(dp.smooth.cpu().numpy(), g[f"c{ci}_L{L}_smooth"])
            assert np.array_equal(W.inverse_w(dp).cpu().numpy(), g[f"c{ci}_L{L}_inv"])


def test_example2_intermediates():
    for L in (1, 2):
        pa = W.forward_w(EX2_A, L)
        pb = W.forward_w(EX2_B, L)
        assert np.array_equal(pa.smooth, EX2[f"A_s{L}"]) and np.array_equal(pb.smooth, EX2[f"B_s{L}"])
        assert np.array_equal(pa.details[L - 1], EX2[f"A_d{L}"])
        assert np.array_equal(pb.details[L - 1], EX2[f"B_d{L}"])
    assert np.array_equal(W.w_product(EX2_A, EX2_B, 2), EX2["C"])
    c = W.face_product(W.forward_w(EX2_A, 2), W.forward_w(EX2_B, 2))
    assert np.array_equal(c.smooth, EX2["C_s2"]) and np.array_equal(c.details[1], EX2["C_d2"])
    assert np.array_equal(c.details[0], EX2["C_d1"])


@pytest.mark.parametrize("L", [1, 2, 4, 8])
def test_config2_full_size_bit_exact(L):
    x = np.random.default_rng(0).standard_normal((512, 512, 256))
    s_ref, d_ref = O.lift_forward(x, L)
    xd = torch.from_numpy(x).cuda()
    buf = E.lift_forward(xd, L)
    want = O.packed_slices(s_ref, d_ref)
    assert torch.equal(buf.cpu(), torch.from_numpy(want))
    y = E.lift_inverse(buf, 512, 512, 256, L)
    assert torch.equal(y.cpu(), torch.from_numpy(O.lift_inverse(s_ref, d_ref)))
    # round trip against the input: exact-rounding closeness (1e-12 rel)
    rel = float((y - xd).norm() / xd.norm())
    assert rel < 1e-12


@pytest.mark.parametrize("shape,L", [((7, 5, 6), 1), ((3, 11, 192), 3), ((33, 1, 64), 6),
                                     ((1, 1, 2), 1), ((2, 3, 8192), 13), ((5, 4, 24), 3),
                                     ((64, 64, 1024), 10), ((9, 9, 96), 5)])
def test_odd_shapes_bit_exact(shape, L):
    x = np.random.default_rng(sum(shape) + L).standard_normal(shape)
    s_ref, d_ref = O.lift_forward(x, L)
    pyr = W.forward_w(x, L)
    assert np.array_equal(pyr.smooth, s_ref)
    for a, b in zip(pyr.details, d_ref):
        assert np.array_equal(a, b)
    assert np.array_equal(W.inverse_w(pyr), O.lift_inverse(s_ref, d_ref))
    buf = E.lift_forward(torch.from_numpy(x).cuda(), L)
    assert np.array_equal(buf.cpu().numpy(), O.packed_slices(s_ref, d_ref))


def test_unaligned_input_takes_plain_path():
    n1, n2, p, L = 13, 7, 32, 3
    x = np.random.default_rng(5).standard_normal((n1, n2, p))
    base = torch.zeros(n1 * n2 * p + 1, dtype=torch.float64, device="cuda")
    xd = base[1:].view(n1, n2, p)
    xd.copy_(torch.from_numpy(x))
    assert xd.data_ptr() % 16 == 8
    buf = E.lift_forward(xd, L)
    s_ref, d_ref = O.lift_forward(x, L)
    assert np.array_equal(buf.cpu().numpy(), O.packed_slices(s_ref, d_ref))
    out = torch.zeros(n1 * n2 * p + 1, dtype=torch.float64, device="cuda")[1:].view(n1, n2, p)
    E.lift_inverse(buf, n1, n2, p, L, out=out)
    assert np.array_equal(out.cpu().numpy(), O.lift_inverse(s_ref, d_ref))


@pytest.mark.parametrize("shape", [(5, 6, 7), (300, 257, 33), (1, 1, 1)])
def test_level0_is_a_transpose(shape):
    x = np.random.default_rng(1).standard_normal(shape)
    buf = E.lift_forward(torch.from_numpy(x).cuda(), 0)
    assert np.array_equal(buf.cpu().numpy(), np.moveaxis(x, 2, 0))
    y = E.lift_inverse(buf, *shape, 0)
    assert np.array_equal(y.cpu().numpy(), x)


@pytest.mark.parametrize("L", [1, 3, 4])
def test_sparse_mask_compact_buffers(L):
    n1, n2, p = 17, 9, 64
    x = np.random.default_rng(L).standard_normal((n1, n2, p))
    s_ref, d_ref = O.lift_forward(x, L)
    m = p >> L
    mask = E.level_mask(L, smooth=True, details=[L])
    xd = torch.from_numpy(x).cuda()
    coarse = E.lift_forward(xd, L, mask=mask, slice_base=p - 2 * m)
    assert coarse.shape == (2 * m, n1, n2)
    assert np.array_equal(coarse.cpu().numpy(), O.packed_slices(s_ref, d_ref)[p - 2 * m:])
    y = E.lift_inverse(coarse, n1, n2, p, L, mask=mask, slice_base=p - 2 * m)
    zeros = [np.zeros_like(d) for d in d_ref[:-1]] + [d_ref[-1]]
    assert np.array_equal(y.cpu().numpy(), O.lift_inverse(s_ref, zeros))


def test_tube_major_layout_is_reference_layout():
    x = np.random.default_rng(2).standard_normal((6, 10, 16))
    buf = E.lift_forward(torch.from_numpy(x).cuda(), 2, layout=N.LAYOUT_TUBE).cpu().numpy().ravel()
    s_ref, d_ref = O.lift_forward(x, 2)
    want = np.concatenate([d.ravel() for d in d_ref] + [s_ref.ravel()])
    assert np.array_equal(buf, want)


def test_user_built_and_mutated_pyramids():
    x = np.random.default_rng(3).standard_normal((4, 5, 8))
    dp = W.forward_w(torch.from_numpy(x).cuda(), 2)
    dp.details[0] = torch.zeros_like(dp.details[0])  # replaced block -> repack path
    s_ref, d_ref = O.lift_forward(x, 2)
    want = O.lift_inverse(s_ref, [np.zeros_like(d_ref[0]), d_ref[1]])
    assert np.array_equal(W.inverse_w(dp).cpu().numpy(), want)
    dp2 = W.forward_w(torch.from_numpy(x).cuda(), 2)
    dp2.smooth.mul_(2.0)                              # in-place edit of a view -> packed buffer sees it
    want2 = O.lift_inverse(2.0 * s_ref, d_ref)
    assert np.array_equal(W.inverse_w(dp2).cpu().numpy(), want2)
    cp = W.constant_pyramid(np.eye(3), 8, 3)
    assert np.array_equal(W.inverse_w(cp), W.identity_tensor(3, 8, 3))


def test_energy_ratio_and_empty():
    x = np.random.default_rng(4).standard_normal((6, 6, 16))
    s, d = O.lift_forward(x, 3)
    got = W.fine_detail_energy_ratio(W.forward_w(x, 3))
    assert abs(got - O.fine_detail_energy_ratio(s, d)) < 1e-14
    e = W.forward_w(np.zeros((0, 3, 4)), 1)
    assert e.smooth.shape == (0, 3, 2)
    assert W.inverse_w(e).shape == (0, 3, 4)


@pytest.mark.parametrize("shape,L", [((2, 3, 1 << 14), 14), ((3, 1, 1 << 15), 15), ((2, 2, 1 << 14), 13)])
def test_very_deep_levels_per_level_path(shape, L):
    """2^L-band chunks beyond one tile (L > 13) take the per-level path; still bit-exact."""
    x = np.random.default_rng(L).standard_normal(shape)
    s_ref, d_ref = O.lift_forward(x, L)
    pyr = W.forward_w(x, L)
    assert np.array_equal(pyr.smooth, s_ref)
    assert all(np.array_equal(a, b) for a, b in zip(pyr.details, d_ref))
    assert np.array_equal(W.inverse_w(pyr), O.lift_inverse(s_ref, d_ref))
    buf = E.lift_forward(torch.from_numpy(x).cuda(), L)
    assert np.array_equal(buf.cpu().numpy(), O.packed_slices(s_ref, d_ref))
    y = E.lift_inverse(buf, shape[0], shape[1], shape[2], L)
    assert np.array_equal(y.cpu().numpy(), O.lift_inverse(s_ref, d_ref))


def test_odd_band_counts_in_transposes():
    x = np.random.default_rng(8).standard_normal((5, 4, 7))
    b = np.random.default_rng(9).standard_normal((4, 3, 7))
    assert np.array_equal(W.transpose(x), O.transpose(x))
    got = W.slicewise_matmul(x, b)
    assert np.max(np.abs(got - O.face_matmul(x, b))) < 1e-14


@pytest.mark.parametrize("shape,L", [((6, 10, 16), 2), ((64, 64, 256), 8), ((33, 7, 96), 5), ((512, 9, 64), 1)])
def test_tube_major_fast_route_masks_and_bases(shape, L):
    """TUBE layout through the fast slice-major kernels + block transposes
    (wt_lift_*_f64 with WT_LAYOUT_TUBE_MAJOR): full, compact [dL|sL] and round trip."""
    n1, n2, p = shape
    x = np.random.default_rng(p + L).standard_normal(shape)
    s_ref, d_ref = O.lift_forward(x, L)
    xd = torch.from_numpy(x).cuda()
    buf = E.lift_forward(xd, L, layout=N.LAYOUT_TUBE)
    want = np.concatenate([d.ravel() for d in d_ref] + [s_ref.ravel()])
    assert np.array_equal(buf.cpu().numpy().ravel(), want)
    y = E.lift_inverse(buf, n1, n2, p, L, layout=N.LAYOUT_TUBE)
    assert np.array_equal(y.cpu().numpy(), O.lift_inverse(s_ref, d_ref))
    m = p >> L
    mask = E.level_mask(L, smooth=True, details=[L])
    coarse = E.lift_forward(xd, L, layout=N.LAYOUT_TUBE, mask=mask, slice_base=p - 2 * m)
    assert np.array_equal(coarse.cpu().numpy().ravel(),
                          np.concatenate([d_ref[-1].ravel(), s_ref.ravel()]))
    y2 = E.lift_inverse(coarse, n1, n2, p, L, layout=N.LAYOUT_TUBE, mask=mask, slice_base=p - 2 * m)
    zeros = [np.zeros_like(d) for d in d_ref[:-1]] + [d_ref[-1]]
    assert np.array_equal(y2.cpu().numpy(), O.lift_inverse(s_ref, zeros))


def test_host_input_conventions_and_streamed_path():
    """np.asarray(x, float64) semantics (lifting.py:83): lists, float32, Fortran order and
    strided views all work; cubes from 4 M elements take the chunked host pipeline."""
    rng = np.random.default_rng(77)
    x = rng.standard_normal((130, 129, 256))           # 4.3 M elements -> streamed path
    for src in (x, np.asfortranarray(x), x.astype(np.float32)):
        s_ref, d_ref = O.lift_forward(np.asarray(src, dtype=np.float64), 4)
        pyr = W.forward_w(src, 4)
        assert np.array_equal(pyr.smooth, s_ref) and all(np.array_equal(a, b) for a, b in zip(pyr.details, d_ref))
        y = W.inverse_w(pyr)
        assert isinstance(y, np.ndarray) and y.flags.c_contiguous
        assert np.array_equal(y, O.lift_inverse(s_ref, d_ref))
    f32 = x.astype(np.float32)
    assert np.array_equal(W.forward_w(f32, 2).smooth, O.lift_forward(f32.astype(np.float64), 2)[0])
    view = x[::2, 1:, :128]                              # strided view
    assert np.array_equal(W.forward_w(view, 3).smooth, O.lift_forward(np.ascontiguousarray(view), 3)[0])
    lst = x[:2, :3, :8].tolist()
    assert np.array_equal(W.forward_w(lst, 1).smooth, O.lift_forward(np.asarray(lst), 1)[0])


def test_host_results_pool_and_pageable_fallback():
    """Large numpy results come from a pool of a few (engine._POOL_PER_SIZE) pinned buffers per size that no
    caller still references; a caller keeping every result gets pageable results (staged
    through the pinned download ring) instead of a fresh page-locked block per call, with
    identical values -- for the streamed transform, its inverse and the sp_w_svd pipeline."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((256, 256, 128))            # 8.4 M elements = 64 MiB results
    s_ref, d_ref = O.lift_forward(x, 3)
    x_back = O.lift_inverse(s_ref, d_ref)
    from paper_2601_08228_b200 import engine as E

    P = E._POOL_PER_SIZE
    kept = [W.forward_w(x, 3) for _ in range(P + 2)]    # all alive: the pool is exhausted
    pinned = [torch.from_numpy(k.smooth).is_pinned() for k in kept]
    assert pinned[:P] == [True] * P and pinned[P:] == [False, False]
    for pyr in kept:
        assert np.array_equal(pyr.smooth, s_ref) and all(np.array_equal(a, b) for a, b in zip(pyr.details, d_ref))
        assert np.array_equal(W.inverse_w(pyr), x_back)  # pinned and pageable pyramids both stream back
    del kept, pyr
    import gc
    gc.collect()
    again = W.forward_w(x, 3)                           # a freed pooled buffer is reused
    assert torch.from_numpy(again.smooth).is_pinned()
    assert np.array_equal(again.smooth, s_ref)
    ys = [W.sp_w_svd(x, 20, 3) for _ in range(P + 1)]  # streamed sp_w_svd, results kept
    assert not torch.from_numpy(ys[P]).is_pinned()
    ref = O.sp_w_svd(x, 20, 3)
    for y in ys:
        assert np.array_equal(y, ys[0])
        assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 1e-10


def test_host_results_pool_evicts_other_sizes_at_the_cap(monkeypatch):
    """At the pool's byte cap, unreferenced pinned buffers of other result sizes are given up
    instead of sending the new size's results to pageable memory."""
    import gc

    rng = np.random.default_rng(6)
    xa = rng.standard_normal((256, 256, 128))            # 64 MiB results
    xb = rng.standard_normal((256, 288, 128))            # 72 MiB results
    with E._pool_lock:
        E._pool.clear()
    monkeypatch.setattr(E, "_POOL_BYTES", 150 << 20)     # room for two buffers
    a1, a2 = W.forward_w(xa, 2), W.forward_w(xa, 2)
    assert torch.from_numpy(a1.smooth).is_pinned() and torch.from_numpy(a2.smooth).is_pinned()
    b_held = W.forward_w(xb, 2)                          # cap reached, both A buffers referenced: pageable
    assert not torch.from_numpy(b_held.smooth).is_pinned()
    del a1, a2, b_held
    gc.collect()
    b1 = W.forward_w(xb, 2)                              # the free A buffers make room
    assert torch.from_numpy(b1.smooth).is_pinned()
    s_ref, d_ref = O.lift_forward(xb, 2)
    assert np.array_equal(b1.smooth, s_ref) and all(np.array_equal(u, v) for u, v in zip(b1.details, d_ref))
    with E._pool_lock:
        E._pool.clear()
