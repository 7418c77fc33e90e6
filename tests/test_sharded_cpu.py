"""Multi-process (gloo, CPU) tests of the sharded rows -> slices -> rows pipelines.

The exchange logic of paper_2601_08228_b200/sharded.py (all-to-all split
sizes, row/slice permutations, uneven splits) runs exactly as on the GPUs; the
per-shard compute is the CPU oracle, so each sharded result must equal the
oracle applied to the gathered cube.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import wten_oracle as O


class OracleOps:
    """CPU stand-in for sharded.CudaOps (test infrastructure only)."""

    def empty(self, shape):
        return torch.empty(shape, dtype=torch.float64)

    def forward(self, x, levels, mask, base):
        s, d = O.lift_forward(x.numpy(), levels)
        return torch.from_numpy(O.packed_slices(s, d)[base:].copy())

    def inverse(self, buf, n1, n2, p, levels, mask, base):
        full = np.zeros((p, n1, n2))
        full[base:] = buf.numpy()
        blocks, off = [], 0
        for j in range(1, levels + 1):
            cnt = p >> j
            blocks.append(np.moveaxis(full[off:off + cnt], 0, 2))
            off += cnt
        smooth = np.moveaxis(full[off:], 0, 2)
        return torch.from_numpy(O.lift_inverse(smooth, blocks))

    def copy_rows(self, src, dst):
        dst.copy_(src)

    def truncated(self, slices, r):
        if slices.shape[0] == 0:
            return slices.clone()
        st = np.moveaxis(slices.numpy(), 0, 2)
        return torch.from_numpy(np.ascontiguousarray(np.moveaxis(O.truncated(*O.stack_svd(st), r), 2, 0)))

    def gemm(self, a, b):
        return torch.from_numpy(np.matmul(a.numpy(), b.numpy()))

    def pinv(self, slices, tol):
        k, n1, n2 = slices.shape
        if k == 0:
            return torch.empty((0, n2, n1), dtype=torch.float64)
        st = np.moveaxis(slices.numpy(), 0, 2)
        return torch.from_numpy(np.ascontiguousarray(np.moveaxis(O.pinv_stack(st, tol), 2, 0)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, outdir, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2601_08228_b200 import sharded

    n1, n2, p, r, L = case
    x = np.random.default_rng(7).standard_normal((n1, n2, p))
    rows = sharded.splits(n1, ws)
    r0 = sum(rows[:rank])
    xl = torch.from_numpy(x[r0:r0 + rows[rank]].copy())
    ops = OracleOps()
    sp = sharded.sp_w_svd_sharded(xl, r, L, n1, ops=ops)
    ws_rec = sharded.w_svd_recon_sharded(xl, r, L, n1, ops=ops)
    pv = sharded.pinv_w_sharded(xl, L, n1, tol=1e-12, ops=ops)
    b = np.random.default_rng(8).standard_normal((n2, 5, p))
    brows = sharded.splits(n2, ws)
    b0 = sum(brows[:rank])
    wp = sharded.w_product_sharded(xl, torch.from_numpy(b[b0:b0 + brows[rank]].copy()), L, n1, ops=ops)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), sp=sp.numpy(), ws=ws_rec.numpy(), pv=pv.numpy(),
             wp=wp.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,case", [(2, (12, 10, 16, 3, 3)), (3, (10, 7, 8, 2, 2)),
                                     (4, (9, 9, 8, 4, 3))])
def test_sharded_pipelines_match_oracle(ws, case):
    n1, n2, p, r, L = case
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(ws, _free_port(), d, case), nprocs=ws, join=True)
        parts = [np.load(os.path.join(d, f"r{g}.npz")) for g in range(ws)]
        sp = np.concatenate([q["sp"] for q in parts], axis=0)
        wsr = np.concatenate([q["ws"] for q in parts], axis=0)
        pv = np.concatenate([q["pv"] for q in parts], axis=0)
        wp = np.concatenate([q["wp"] for q in parts], axis=0)
    x = np.random.default_rng(7).standard_normal((n1, n2, p))
    b = np.random.default_rng(8).standard_normal((n2, 5, p))
    np.testing.assert_allclose(wp, O.w_product(x, b, L), rtol=0, atol=1e-12)
    np.testing.assert_allclose(sp, O.sp_w_svd(x, r, L), rtol=0, atol=1e-12)
    np.testing.assert_allclose(wsr, O.w_svd(x, r, L)["recon"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(pv, O.pinv_w(x, L), rtol=0, atol=1e-10)


@pytest.mark.parametrize("G,n1,n2,p,L", [(2, 12, 10, 16, 3), (3, 10, 7, 8, 2), (4, 9, 6, 8, 3),
                                         (8, 16, 4, 32, 4)])
def test_fused_peer_tables_assemble_full_slices(G, n1, n2, p, L):
    """Simulate G ranks' fused K1 stores / K2 loads through sharded.peer_slice_table
    with fake per-rank base addresses: every owner must end up holding full
    coarse slices, and every rank must read back exactly its rows."""
    from paper_2601_08228_b200 import sharded

    x = np.random.default_rng(5).standard_normal((n1, n2, p))
    m = p >> L
    K, base = 2 * m, p - 2 * m
    ks = sharded.splits(K, G)
    rows = sharded.splits(n1, G)
    span = 1 << 40
    ptrs = [(g + 1) * span for g in range(G)]
    bufs = [np.full(max(ks) * n1 * n2, np.nan) for _ in range(G)]

    def locate(addr):
        g = addr // span - 1
        off = addr - ptrs[g]
        assert off % 8 == 0
        return g, off // 8

    r0 = 0
    for me in range(G):                      # K1 of every rank: stores via its table
        tab = sharded.peer_slice_table(ptrs, ks, r0, n1, n2)
        assert len(tab) == K
        s, d = O.lift_forward(x[r0:r0 + rows[me]], L)
        coarse = O.packed_slices(s, d)[base:]            # (K, R, n2) of my rows
        for k in range(K):
            g, off = locate(tab[k])
            bufs[g][off:off + rows[me] * n2] = coarse[k].ravel()
        r0 += rows[me]
    s, d = O.lift_forward(x, L)
    full = O.packed_slices(s, d)[base:]
    for g, st in enumerate(sharded.offsets(ks)):          # owners hold full slices
        got = bufs[g][:ks[g] * n1 * n2].reshape(ks[g], n1, n2)
        assert np.array_equal(got, full[st:st + ks[g]])
    r0 = 0
    for me in range(G):                      # K2 of every rank: loads via its table
        tab = sharded.peer_slice_table(ptrs, ks, r0, n1, n2)
        for k in range(K):
            g, off = locate(tab[k])
            assert np.array_equal(bufs[g][off:off + rows[me] * n2].reshape(rows[me], n2),
                                  full[k, r0:r0 + rows[me]])
        r0 += rows[me]


@pytest.mark.parametrize("G,n1,n2,p,L", [(2, 12, 10, 16, 3), (3, 10, 7, 8, 2), (8, 9, 20, 16, 1)])
def test_fused_pinv_tables_transposed_results(G, n1, n2, p, L):
    """w-pinv fused exchange: owners hold (n2, n1) result slices; rank g reads back
    its splits(n2, G) rows of every slice through the K2 table (all p slices)."""
    from paper_2601_08228_b200 import sharded

    ks = sharded.splits(p, G)
    orows = sharded.splits(n2, G)
    span = 1 << 40
    ptrs = [(g + 1) * span for g in range(G)]
    res = np.random.default_rng(7).standard_normal((p, n2, n1))     # the owners' pinv slices
    bufs = [np.zeros(max(ks) * n1 * n2) for _ in range(G)]
    for g, st in enumerate(sharded.offsets(ks)):
        bufs[g][:ks[g] * n1 * n2] = res[st:st + ks[g]].ravel()
    r0 = 0
    for me in range(G):
        tab = sharded.peer_slice_table(ptrs, ks, r0, n2, n1)
        assert len(tab) == p
        for k in range(p):
            g, off = tab[k] // span - 1, (tab[k] % span) // 8
            got = bufs[g][off:off + orows[me] * n1].reshape(orows[me], n1)
            assert np.array_equal(got, res[k, r0:r0 + orows[me]])
        r0 += orows[me]


def test_splits():
    from paper_2601_08228_b200 import sharded

    assert sharded.splits(10, 3) == [4, 3, 3]
    assert sharded.splits(32, 8) == [4] * 8
    assert sharded.splits(2, 4) == [1, 1, 0, 0]
    assert sharded.offsets([4, 3, 3]) == [0, 4, 7]
