"""Multi-process sharded pipelines with the PRODUCT compute (sharded.CudaOps: K1, K2,
K3, K4, K5, K7 on cuda:0) and a gloo group at world sizes 2-4 (host-staged
exchanges; only one GPU is available here, so every rank shares it).  The CUDA
kernels see real uneven row shards, ranks owning zero coarse slices and slice
shards of different sizes; every gathered result must equal the single-call
product path and the CPU oracle on the same cube (multi-GPU
readiness).  The NCCL / symmetric-memory transport is covered on one GPU by
tests/test_gpu_sharded.py."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, outdir, case):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2601_08228_b200 import sharded

    n1, n2, p, r, L = case
    x = np.random.default_rng(7).standard_normal((n1, n2, p))
    rows = sharded.splits(n1, ws)
    r0 = sum(rows[:rank])
    xl = torch.from_numpy(x[r0:r0 + rows[rank]].copy()).cuda()
    ops = sharded.CudaOps(torch.device("cuda", 0))
    sp = sharded.sp_w_svd_sharded(xl, r, L, n1, ops=ops)
    wr = sharded.w_svd_recon_sharded(xl, r, L, n1, ops=ops)
    pv = sharded.pinv_w_sharded(xl, L, n1, tol=1e-12, ops=ops)
    b = np.random.default_rng(8).standard_normal((n2, 5, p))
    brows = sharded.splits(n2, ws)
    b0 = sum(brows[:rank])
    wp = sharded.w_product_sharded(xl, torch.from_numpy(b[b0:b0 + brows[rank]].copy()).cuda(), L, n1, ops=ops)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), sp=sp.cpu().numpy(), ws=wr.cpu().numpy(),
             pv=pv.cpu().numpy(), wp=wp.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,case", [
    (2, (130, 96, 32, 5, 3)),     # rows 65 / 65; 8 coarse slices
    (3, (100, 136, 16, 4, 3)),    # uneven rows 34 / 33 / 33; preconditioned slices (n >= 128 side)
    (4, (41, 30, 8, 3, 3)),       # 2 coarse slices over 4 ranks: two ranks own none
])
def test_sharded_cuda_ops_match_single_gpu(ws, case):
    import paper_2601_08228_b200 as W

    n1, n2, p, r, L = case
    ctx = mp.get_context("spawn")
    with tempfile.TemporaryDirectory() as d:
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(k, ws, port, d, case)) for k in range(ws)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(timeout=600)
            assert pr.exitcode == 0, f"rank exited with {pr.exitcode}"
        parts = [np.load(os.path.join(d, f"r{k}.npz")) for k in range(ws)]
        x = np.random.default_rng(7).standard_normal((n1, n2, p))
        b = np.random.default_rng(8).standard_normal((n2, 5, p))
        sp = np.concatenate([q["sp"] for q in parts])
        wr = np.concatenate([q["ws"] for q in parts])
        pv = np.concatenate([q["pv"] for q in parts])
        wp = np.concatenate([q["wp"] for q in parts])
        assert relerr(sp, W.sp_w_svd(x, r, L)) < 1e-10 and relerr(sp, O.sp_w_svd(x, r, L)) < 1e-8
        assert relerr(wr, W.w_svd(x, r, L)[1]) < 1e-10 and relerr(wr, O.w_svd(x, r, L)["recon"]) < 1e-8
        assert relerr(pv, W.pinv_w(x, L)) < 1e-9 and relerr(pv, O.pinv_w(x, L)) < 1e-8
        assert relerr(wp, W.w_product(x, b, L)) < 1e-12 and relerr(wp, O.w_product(x, b, L)) < 1e-10
