"""The sharded pipelines with the product ops (CUDA kernels + NCCL) on one GPU
(world size 1: the all-to-alls are local copies).  The multi-rank exchange is
covered by tests/test_sharded_cpu.py over gloo."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import sharded
from oracle import wten_oracle as O
from wt_helpers import relerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl1():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_sharded_equals_single_gpu(nccl1):
    x = np.random.default_rng(31).standard_normal((64, 48, 32))
    xd = torch.from_numpy(x).cuda()
    sp = sharded.sp_w_svd_sharded(xd, 6, 3, 64)
    assert torch.equal(sp, W.sp_w_svd(xd, 6, 3))
    assert relerr(sp.cpu().numpy(), O.sp_w_svd(x, 6, 3)) < 1e-10
    ws = sharded.w_svd_recon_sharded(xd, 6, 2, 64)
    assert relerr(ws.cpu().numpy(), O.w_svd(x, 6, 2)["recon"]) < 1e-10
    pv = sharded.pinv_w_sharded(xd, 2, 64)
    assert relerr(pv.cpu().numpy(), O.pinv_w(x, 2)) < 1e-9


def test_fused_exchange_equals_nccl_path(nccl1):
    """K1/K2 with the exchange fused in (peer-pointer tables over symmetric memory)."""
    x = np.random.default_rng(32).standard_normal((64, 48, 32))
    xd = torch.from_numpy(x).cuda()
    for _ in range(2):  # second call reuses the cached symmetric buffers
        fz = sharded.sp_w_svd_fused(xd, 6, 3, 64)
        assert torch.equal(fz, sharded.sp_w_svd_sharded(xd, 6, 3, 64))
    assert relerr(fz.cpu().numpy(), O.sp_w_svd(x, 6, 3)) < 1e-10


def test_fused_w_svd_and_pinv_equal_nccl_path(nccl1):
    """Full-pyramid exchanges (all p slices) fused into K1/K2: w-svd recon and w-pinv
    (the pinv's result slices are n2 x n1, its rows split over n2)."""
    x = np.random.default_rng(33).standard_normal((40, 56, 16))
    xd = torch.from_numpy(x).cuda()
    ws = sharded.w_svd_recon_fused(xd, 5, 2, 40)
    assert torch.equal(ws, sharded.w_svd_recon_sharded(xd, 5, 2, 40))
    assert relerr(ws.cpu().numpy(), O.w_svd(x, 5, 2)["recon"]) < 1e-10
    pv = sharded.pinv_w_fused(xd, 2, 40)
    assert pv.shape == (56, 40, 16)
    assert torch.equal(pv, sharded.pinv_w_sharded(xd, 2, 40))
    assert relerr(pv.cpu().numpy(), O.pinv_w(x, 2)) < 1e-9


def test_w_product_sharded_equals_single_gpu(nccl1):
    """Row-sharded w-product (A's rows local, B all-gathered) with the product ops."""
    rng = np.random.default_rng(34)
    a = rng.standard_normal((64, 48, 32))
    b = rng.standard_normal((48, 40, 32))
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c = sharded.w_product_sharded(ad, bd, 3, 64)
    assert torch.equal(c, W.w_product(ad, bd, 3))
    assert relerr(c.cpu().numpy(), O.w_product(a, b, 3)) < 1e-10
