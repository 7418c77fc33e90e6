"""Race / ordering stress in place of compute-sanitizer, which this GPU pool has
closed ("runs under it have left GPUs needing a reset"): every kernel family
runs repeatedly -- under different scheduling (resident CTAs per SM, cluster
splits, concurrent host threads) -- and must give bit-identical results that
also match the CPU oracle.  A shared-memory race, a missing fence between the
TMA refill and the generic-proxy reads, a lost update in the K4 ticket
scheduler or in the preconditioner's cluster exchanges shows up as a changed
bit in some repetition.  (tools/sanitize_cases.py holds the small cases the
sanitizer runs would use.)"""

import threading

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import engine as E
from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu


def test_lifting_every_level_repeated():
    x = torch.from_numpy(np.random.default_rng(1).standard_normal((96, 80, 256))).cuda()
    for L in range(1, 9):
        buf0 = E.lift_forward(x, L)
        y0 = E.lift_inverse(buf0, 96, 80, 256, L)
        for _ in range(5):
            assert torch.equal(E.lift_forward(x, L), buf0)
            assert torch.equal(E.lift_inverse(buf0, 96, 80, 256, L), y0)
        s, d = O.lift_forward(x.cpu().numpy(), L)
        assert np.array_equal(buf0.cpu().numpy(), O.packed_slices(s, d))


@pytest.mark.parametrize("shape", [(24, 256, 256), (4, 1024, 1024), (6, 512, 384)])
def test_svd_preconditioned_repeated(shape):
    """K4 with the eig.cu preconditioner (single-CTA and 2 / 4 / 8-CTA cluster panels):
    ten runs bit-identical, singular values vs LAPACK."""
    a = torch.from_numpy(np.random.default_rng(shape[1]).standard_normal(shape)).cuda()
    s0, v0, _ = E.svd(a, 8)
    for _ in range(9):
        s, v, info = E.svd(a, 8)
        E.raise_if_failed(info)
        assert torch.equal(s, s0) and torch.equal(v, v0)
    ref = np.linalg.svd(a[:2].cpu().numpy(), compute_uv=False)
    assert np.max(np.abs(s0[:2].cpu().numpy() - ref)) < 1e-12 * ref.max()


@pytest.mark.parametrize("opt", [("svd_split", 2), ("svd_split", 4), ("svd_split", 8), ("svd_ctas_per_sm", 1)])
def test_svd_scheduling_stress(opt):
    a = torch.from_numpy(np.random.default_rng(7).standard_normal((3, 512, 512))).cuda()
    with E.option(*opt):
        s0, v0, _ = E.svd(a, 4)
        for _ in range(4):
            s, v, _ = E.svd(a, 4)
            assert torch.equal(s, s0) and torch.equal(v, v0)
    ref = np.linalg.svd(a.cpu().numpy(), compute_uv=False)
    assert np.max(np.abs(s0.cpu().numpy() - ref)) < 1e-12 * ref.max()


def test_concurrent_streams_preconditioned():
    """Four host threads, each on its own stream, run preconditioned SVDs at once: every
    result equals the serial one (the workspace, ring buffers and diagnostics are per call
    or per thread)."""
    rng = np.random.default_rng(3)
    xs = [torch.from_numpy(rng.standard_normal((6, 256, 256))).cuda() for _ in range(4)]
    serial = [E.svd(x, 4)[0] for x in xs]
    out = [None] * 4

    def run(i):
        with torch.cuda.stream(torch.cuda.Stream()):
            out[i] = E.svd(xs[i], 4)[0]
            torch.cuda.current_stream().synchronize()

    th = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(out, serial):
        assert torch.equal(a, b)


def test_host_streamed_sp_w_svd_repeated():
    x = np.random.default_rng(9).standard_normal((256, 128, 256))
    y0 = W.sp_w_svd(x, 6, 3)
    for _ in range(3):
        assert np.array_equal(W.sp_w_svd(x, 6, 3), y0)
    assert relerr(y0, O.sp_w_svd(x, 6, 3)) < 1e-8


def test_pinned_numpy_inputs_are_uploaded_in_place_with_the_same_bits():
    """Cubes in page-locked memory (W.pinned_empty) skip the staging ring on the streamed host
    paths (engine.host_slices_pipeline, engine.host_lift); the results are those of the pageable
    path bit for bit, and the input array is left untouched."""
    import paper_2601_08228_b200 as W

    rng = np.random.default_rng(23)
    x = rng.standard_normal((160, 256, 256))           # 80 MB: streamed in row chunks
    xp = W.pinned_empty(x.shape)
    xp[...] = x
    assert W.is_pinned_array(xp) and not W.is_pinned_array(x)
    assert not W.is_pinned_array(xp[:, ::2]) and not W.is_pinned_array(xp.astype(np.float32))
    y = W.sp_w_svd(x, 12, 3)
    for _ in range(2):
        assert np.array_equal(W.sp_w_svd(xp, 12, 3), y)
    assert np.array_equal(xp, x)
    pa, pb = W.forward_w(x, 4), W.forward_w(xp, 4)
    assert np.array_equal(pa.smooth, pb.smooth) and all(np.array_equal(u, v) for u, v in zip(pa.details, pb.details))
    assert np.array_equal(W.inverse_w(pb), W.inverse_w(pa))
    # a pinned view with an offset (rows 8..) is still DMA'd in place
    assert np.array_equal(W.sp_w_svd(xp[8:], 12, 3), W.sp_w_svd(np.ascontiguousarray(x[8:]), 12, 3))


def test_sp_w_svd_many_pipeline_equals_single_calls():
    """Two calls in flight on their own host threads and streams (upload of the next cube under the
    K4 / download of the current one): the results, in order, are the single calls' bit for bit."""
    import paper_2601_08228_b200 as W

    rng = np.random.default_rng(29)
    cubes = [rng.standard_normal((160, 256, 256)) for _ in range(3)]    # 80 MB each: streamed
    pinned = W.pinned_empty(cubes[0].shape)
    pinned[...] = cubes[0]
    seq = [pinned, cubes[1], cubes[2], pinned, cubes[1]]
    want = [W.sp_w_svd(c, 10, 3) for c in cubes]
    order = [0, 1, 2, 0, 1]
    for depth in (1, 2, 3):
        got = list(W.sp_w_svd_many(iter(seq), 10, 3, depth=depth))
        assert len(got) == len(seq)
        for g, k in zip(got, order):
            assert np.array_equal(g, want[k])
    small = [rng.standard_normal((8, 6, 8)) for _ in range(4)]          # device path (below the streaming size)
    for g, c in zip(W.sp_w_svd_many(small, 2, 1), small):
        assert np.array_equal(g, W.sp_w_svd(c, 2, 1))
    assert list(W.sp_w_svd_many([], 2, 1)) == []
    with pytest.raises(ValueError):
        list(W.sp_w_svd_many(small, 2, 1, depth=0))


def test_status_readback_bypasses_the_copy_engine_and_matches():
    """wt_readback_i32 (K4's info vector into page-locked memory by a kernel, not a copy-engine
    copy): values, counts on both sides of the block size, and the LinAlgError mapping of
    raise_if_failed (decomposition.py:66) while another stream keeps the D2H engine busy."""
    from paper_2601_08228_b200 import _native as N

    lib = N.require_gpu()
    for n in (1, 2, 31, 32, 255, 256, 257, 5000):
        src = torch.arange(n, dtype=torch.int32, device="cuda") * 3 - 7
        dst = torch.full((n + 3,), -99, dtype=torch.int32).pin_memory()
        N.check(lib.wt_readback_i32(src.data_ptr(), dst.data_ptr(), n, torch.cuda.current_stream().cuda_stream), "readback")
        assert torch.equal(dst[:n], src.cpu()) and bool((dst[n:] == -99).all())
    N.check(lib.wt_readback_i32(0, 0, 0, torch.cuda.current_stream().cuda_stream), "readback")
    big_d = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    big_h = torch.empty(64 << 20, dtype=torch.float64).pin_memory()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(4):
            big_h.copy_(big_d, non_blocking=True)
    ok = torch.zeros(40, dtype=torch.int32, device="cuda")
    E.raise_if_failed(ok)
    bad = ok.clone()
    bad[17] = 2
    with pytest.raises(np.linalg.LinAlgError, match="SVD did not converge"):
        E.raise_if_failed(bad)
    side.synchronize()
