"""Multi-GPU w-svd / sp-w-svd / w-pinv: rows -> wavelet slices -> rows.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The cube
is sharded by spatial rows i (complete tubes), so the lifting transform needs
no communication (every 2^L-band chunk of a tube is independent, SURVEY.md
finding 3).  The facewise SVD is independent per wavelet slice, so one
all-to-all redistributes the packed slices from row shards to slice shards, the
slices are decomposed locally, and a second all-to-all brings the results back
to row shards for the inverse transform.  sp-w-svd
only exchanges the 2m coarsest slices [dL | sL] (1/2^(L-1) of the data).

The compute behind the exchange is pluggable (``ops``): :class:`CudaOps` is the
product (K1/K2/K4/K5 kernels + NCCL); the CPU tests drive the same exchange
logic over gloo with an oracle-backed ops object.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native as N
from . import engine as E
from .decomposition import _check_levels, _check_rank


def splits(n: int, parts: int):
    """Balanced contiguous split sizes (first n % parts parts get one extra)."""
    base, extra = divmod(n, parts)
    return [base + (1 if g < extra else 0) for g in range(parts)]


def offsets(sizes):
    out, acc = [], 0
    for s in sizes:
        out.append(acc)
        acc += s
    return out


class CudaOps:
    """Product compute for the sharded pipelines (hand-written sm_100a kernels)."""

    def __init__(self, device=None):
        self.device = device or torch.device("cuda", torch.cuda.current_device())

    def empty(self, shape):
        return torch.empty(shape, dtype=torch.float64, device=self.device)

    def forward(self, x, levels, mask, slice_base):
        return E.lift_forward(x, levels, mask=mask, slice_base=slice_base)

    def inverse(self, buf, n1, n2, p, levels, mask, slice_base):
        return E.lift_inverse(buf, n1, n2, p, levels, mask=mask, slice_base=slice_base)

    def copy_rows(self, src, dst):
        E.copy2d(src, trans=False, out=dst)

    def truncated(self, slices, r):
        if slices.shape[0] == 0:
            return self.empty(slices.shape)
        return E.svd_truncated_recon(slices, r)

    def pinv(self, slices, tol):
        k, n1, n2 = slices.shape
        if k == 0:
            return self.empty((0, n2, n1))
        sigma, vec, info = E.svd(slices, min(n1, n2))
        E.raise_if_failed(info)
        return E.pinv_blocks(slices, sigma, vec, tol)

    def gemm(self, a, b):
        if a.shape[1] == 0:
            return self.empty((a.shape[0], 0, b.shape[2]))
        return E.gemm(a, b)


def _host_staged(t, group) -> bool:
    """CUDA tensors over a gloo group (the multi-process tests on one GPU) go through
    host buffers; NCCL exchanges device memory directly."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def _a2a(out, inp, out_splits, in_splits, group):
    if _host_staged(out, group):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(o)
        return
    dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def rows_to_slices(ops, local, rows, group):
    """(K, R_me, c) packed slices of my rows -> (K_me, n, c) full slices I own.

    ``rows`` = row split sizes of every rank (sum n); slices are split with
    :func:`splits` (K_me for rank me).
    """
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    K, R_me, c = local.shape
    ks = splits(K, G)
    n = sum(rows)
    in_splits = [ks[h] * R_me * c for h in range(G)]
    out_splits = [ks[me] * rows[g] * c for g in range(G)]
    recv = ops.empty((sum(out_splits),))
    _a2a(recv, local.reshape(-1), out_splits, in_splits, group)
    full = ops.empty((ks[me], n, c))
    off, r0 = 0, 0
    for g in range(G):
        cnt = out_splits[g]
        if cnt:
            ops.copy_rows(recv[off:off + cnt].view(ks[me], rows[g], c), full[:, r0:r0 + rows[g], :])
        off += cnt
        r0 += rows[g]
    return full, ks


def slices_to_rows(ops, full, ks, rows, group):
    """Inverse of :func:`rows_to_slices` for (K_me, n, c) results with output row splits ``rows``."""
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    k_me, n, c = full.shape
    K = sum(ks)
    in_splits = [k_me * rows[g] * c for g in range(G)]
    send = ops.empty((sum(in_splits),))
    off, r0 = 0, 0
    for g in range(G):
        cnt = in_splits[g]
        if cnt:
            ops.copy_rows(full[:, r0:r0 + rows[g], :], send[off:off + cnt].view(k_me, rows[g], c))
        off += cnt
        r0 += rows[g]
    out_splits = [ks[h] * rows[me] * c for h in range(G)]
    recv = ops.empty((sum(out_splits),))
    _a2a(recv, send, out_splits, in_splits, group)
    return recv.view(K, rows[me], c)  # rank-major order == slice order


def sp_w_svd_sharded(x_local, r, levels, n1, group=None, ops=None):
    """sp-w-svd of an (n1, n2, p) cube whose rows are sharded over the group.

    ``x_local`` holds this rank's rows (split by :func:`splits`); returns this
    rank's rows of the reconstruction.  Equal (up to the per-slice SVD) to
    ``decomposition.sp_w_svd`` on the gathered cube.
    """
    ops = ops or CudaOps()
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    R, n2, p = x_local.shape
    rows = splits(n1, G)
    assert R == rows[me], f"rank {me} holds {R} rows, expected {rows[me]}"
    _check_rank(r, n1, n2)
    _check_levels(p, levels)
    m = p >> levels
    base = p - 2 * m
    mask = E.level_mask(levels, smooth=True, details=[levels])
    coarse = ops.forward(x_local, levels, mask, base)          # (2m, R, n2)
    full, ks = rows_to_slices(ops, coarse, rows, group)         # (k_me, n1, n2)
    rec = ops.truncated(full, r)
    back = slices_to_rows(ops, rec, ks, rows, group)            # (2m, R, n2)
    return ops.inverse(back, R, n2, p, levels, mask, base)


def w_svd_recon_sharded(x_local, r, levels, n1, group=None, ops=None):
    """Rank-r w-svd reconstruction (all p wavelet slices) of a row-sharded cube."""
    ops = ops or CudaOps()
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    R, n2, p = x_local.shape
    rows = splits(n1, G)
    assert R == rows[me]
    _check_rank(r, n1, n2)
    _check_levels(p, levels)
    pyr = ops.forward(x_local, levels, N.MASK_ALL, 0)           # (p, R, n2)
    full, ks = rows_to_slices(ops, pyr, rows, group)
    rec = ops.truncated(full, r)
    back = slices_to_rows(ops, rec, ks, rows, group)
    return ops.inverse(back, R, n2, p, levels, N.MASK_ALL, 0)


def pinv_w_sharded(x_local, levels, n1, tol=1e-12, group=None, ops=None):
    """w-pinv of a row-sharded (n1, n2, p) cube; returns this rank's rows of the
    (n2, n1, p) pseudo-inverse (its rows split over n2 with :func:`splits`)."""
    ops = ops or CudaOps()
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    R, n2, p = x_local.shape
    rows = splits(n1, G)
    assert R == rows[me]
    _check_levels(p, levels)
    pyr = ops.forward(x_local, levels, N.MASK_ALL, 0)
    full, ks = rows_to_slices(ops, pyr, rows, group)            # (k_me, n1, n2)
    inv = ops.pinv(full, tol)                                   # (k_me, n2, n1)
    out_rows = splits(n2, G)
    back = slices_to_rows(ops, inv, ks, out_rows, group)        # (p, n2_me, n1)
    return ops.inverse(back, out_rows[me], n1, p, levels, N.MASK_ALL, 0)


def gather_rows(ops, local, rows, group):
    """All ranks' row blocks (rank order) of a row-sharded (R_me, ...) tensor ->
    the full (sum rows, ...) tensor on every rank (NCCL all-gather; uneven
    splits are padded to the largest block)."""
    G = dist.get_world_size(group)
    R = max(rows)
    tail = tuple(local.shape[1:])
    pad = ops.empty((R,) + tail)
    if local.shape[0]:
        pad[:local.shape[0]].copy_(local)
    allb = ops.empty((G * R,) + tail)
    if _host_staged(allb, group):
        h = torch.empty(allb.shape, dtype=allb.dtype)
        dist.all_gather_into_tensor(h, pad.cpu(), group=group)
        allb.copy_(h)
    else:
        dist.all_gather_into_tensor(allb, pad, group=group)
    full = ops.empty((sum(rows),) + tail)
    r0 = 0
    for g in range(G):
        full[r0:r0 + rows[g]].copy_(allb[g * R:g * R + rows[g]])
        r0 += rows[g]
    return full


def w_product_sharded(a_local, b_local, levels, n1, group=None, ops=None):
    """w-product C = A *_w B with A (n1, n2, p) and B (n2, n3, p) both sharded by
    rows (algebra.py:43-51).  The facewise product is row-separable in A, so C's
    rows follow A's: every rank transforms its rows of A locally (no exchange),
    all-gathers B (the small-right-operand layout of SURVEY.md section 8(e)),
    runs K3 on its rows of every wavelet slice and inverts them locally.
    Returns this rank's rows of C (the split of A's rows)."""
    ops = ops or CudaOps()
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    R, n2, p = a_local.shape
    rows = splits(n1, G)
    assert R == rows[me], f"rank {me} holds {R} rows of A, expected {rows[me]}"
    brows = splits(n2, G)
    assert b_local.shape[0] == brows[me] and b_local.shape[2] == p
    _check_levels(p, levels)
    n3 = b_local.shape[1]
    b = gather_rows(ops, b_local, brows, group)                     # (n2, n3, p)
    pa = ops.forward(a_local, levels, N.MASK_ALL, 0)                 # (p, R, n2)
    pb = ops.forward(b, levels, N.MASK_ALL, 0)                       # (p, n2, n3)
    pc = ops.gemm(pa, pb)                                            # (p, R, n3)
    return ops.inverse(pc, R, n3, p, levels, N.MASK_ALL, 0)


def peer_slice_table(ptrs, ks, row0, n1, n2, elem=8):
    """Address of this rank's row block in the owner's slice buffer, per coarse slice.

    Slice s (0 <= s < sum(ks)) is owned by the rank g with offsets(ks)[g] <= s <
    offsets(ks)[g] + ks[g]; the owner's buffer holds its slices as full
    (n1, n2) row-major matrices, and this rank's rows start at row ``row0``.
    Pure integer math (tested on CPU); ``ptrs`` are the symmetric buffers' base
    addresses on every rank.
    """
    starts = offsets(ks)
    tab = []
    for g, (st, k) in enumerate(zip(starts, ks)):
        for j in range(k):
            tab.append(int(ptrs[g]) + ((j * n1 + row0) * n2) * elem)
    return tab


_SYMM = {}


def _symm_pair(numel, device, group):
    """Two cached symmetric-memory buffers (+ handles) of `numel` doubles."""
    import torch.distributed._symmetric_memory as symm_mem

    gname = (group or dist.group.WORLD).group_name
    key = (numel, str(device), gname)
    if key not in _SYMM:
        bufs = []
        for _ in range(2):
            t = symm_mem.empty(numel, dtype=torch.float64, device=device)
            bufs.append((t, symm_mem.rendezvous(t, gname)))
        _SYMM[key] = bufs
    return _SYMM[key]


def _fused_exchange(x_local, levels, n1, mask, base, decompose, out_rows, out_cols, group, phases=None):
    """rows -> owners' slices (peer stores in K1), ``decompose`` in place on the owner,
    owners' result slices -> rows (peer loads in K2).

    Packed slices ``base .. p-1`` (as selected by ``mask``) are dealt to the ranks
    in contiguous runs; ``decompose(full, out)`` maps the owner's (k, n1, n2)
    slices to (k, out_rows, out_cols) result slices; this rank gets back its
    ``splits(out_rows, G)`` share of the result rows as an (rows, out_cols, p) tensor.
    """
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    R, n2, p = x_local.shape
    rows = splits(n1, G)
    assert R == rows[me], f"rank {me} holds {R} rows, expected {rows[me]}"
    K = p - base
    ks = splits(K, G)
    orows = splits(out_rows, G)
    dev = x_local.device
    (recv, h_recv), (recb, h_rec) = _symm_pair(max(ks) * n1 * n2, dev, group)
    tab_f = torch.tensor(peer_slice_table(h_recv.buffer_ptrs, ks, sum(rows[:me]), n1, n2),
                         dtype=torch.int64, device=dev)
    tab_i = torch.tensor(peer_slice_table(h_rec.buffer_ptrs, ks, sum(orows[:me]), out_rows, out_cols),
                         dtype=torch.int64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if phases is not None else None
    mark = (lambda i: ev[i].record()) if ev else (lambda i: None)
    mark(0)
    # Memory ordering: K1's peer stores are followed (stream order) by the
    # symmetric-memory barrier kernel, whose signal is a system-scope release and
    # whose wait is a system-scope acquire; K1 also ends every CTA with a
    # system-scope fence after its last peer store (lift_fast.cu, peer variant).
    E.lift_forward_peer(x_local.contiguous(), levels, tab_f, mask, base)
    mark(1)
    h_recv.barrier(channel=0)                   # every rank's peer stores have landed
    mark(2)
    k_me = ks[me]
    if k_me:
        decompose(recv[:k_me * n1 * n2].view(k_me, n1, n2),
                  recb[:k_me * out_rows * out_cols].view(k_me, out_rows, out_cols))
    mark(3)
    h_rec.barrier(channel=0)                    # every owner's result is ready
    mark(4)
    y = E.lift_inverse_peer(tab_i, orows[me], out_cols, p, levels, mask, base)
    h_rec.barrier(channel=1)                    # all peer loads done before buffers are reused
    mark(5)
    if ev:
        ev[5].synchronize()
        phases.update({"k1_peer_store_ms": ev[0].elapsed_time(ev[1]),
                       "exchange_barrier_ms": ev[1].elapsed_time(ev[2]),
                       "k4_ms": ev[2].elapsed_time(ev[3]),
                       "owners_barrier_ms": ev[3].elapsed_time(ev[4]),
                       "k2_peer_load_ms": ev[4].elapsed_time(ev[5]),
                       "slices_owned": k_me, "rows_owned": R})
    return y


def sp_w_svd_fused(x_local, r, levels, n1, group=None, phase_times=False):
    """sp-w-svd of a row-sharded cube with the exchange fused into K1 / K2.

    K1 stores each coarse slice row block straight into the owning GPU's
    symmetric-memory buffer (peer stores over NVLink), so the owner holds full
    (n1, n2) slices without an all-to-all or a permute; after a device-side
    barrier every rank decomposes its slices in place into a second symmetric
    buffer, and K2 loads its rows of every reconstructed slice from the owners
    (peer loads).  Same result as :func:`sp_w_svd_sharded`.
    """
    R, n2, p = x_local.shape
    _check_rank(r, n1, n2)
    _check_levels(p, levels)
    m = p >> levels

    def decompose(full, out):
        E.svd_truncated_recon(full, r, out=out)

    mask = E.level_mask(levels, smooth=True, details=[levels])
    phases = {} if phase_times else None
    y = _fused_exchange(x_local, levels, n1, mask, p - 2 * m, decompose, n1, n2, group, phases)
    return (y, phases) if phase_times else y


def w_svd_recon_fused(x_local, r, levels, n1, group=None):
    """Rank-r w-svd reconstruction of a row-sharded cube, all p wavelet slices
    exchanged by the peer stores / loads of K1 / K2 (see :func:`sp_w_svd_fused`)."""
    R, n2, p = x_local.shape
    _check_rank(r, n1, n2)
    _check_levels(p, levels)

    def decompose(full, out):
        sigma, vec, info = E.svd(full, r)
        E.raise_if_failed(info)
        E.truncated_recon(full, sigma, vec, r, out=out)

    return _fused_exchange(x_local, levels, n1, N.MASK_ALL, 0, decompose, n1, n2, group)


def pinv_w_fused(x_local, levels, n1, tol=1e-12, group=None):
    """w-pinv of a row-sharded cube with the fused exchange; returns this rank's
    ``splits(n2, G)`` rows of the (n2, n1, p) pseudo-inverse."""
    R, n2, p = x_local.shape
    _check_levels(p, levels)

    def decompose(full, out):
        sigma, vec, info = E.svd(full, min(n1, n2))
        E.raise_if_failed(info)
        E.pinv_blocks(full, sigma, vec, tol, out=out)

    return _fused_exchange(x_local, levels, n1, N.MASK_ALL, 0, decompose, n2, n1, group)


def bench_w_product(dist_mod, timed_region, steps=3, warmup=1, n=512, p=128, levels=3):
    """Config-5-sized w-product (A, B: n x n x p) with both operands row-sharded
    over the group (strong scaling; B all-gathered, no all-to-all)."""
    G = dist_mod.get_world_size()
    me = dist_mod.get_rank()
    rows = splits(n, G)
    r0 = sum(rows[:me])
    gen = torch.Generator(device="cuda").manual_seed(5)
    a = torch.rand((rows[me], n, p), dtype=torch.float64, device="cuda", generator=gen)
    b = torch.rand((rows[me], n, p), dtype=torch.float64, device="cuda", generator=gen)
    out = {}

    def step(record):
        out["c"] = w_product_sharded(a, b, levels, n)

    ms = timed_region(step, steps, warmup, dist_mod)
    flops = 2.0 * n * n * n * p
    return {"config": f"w_product {n}x{n}x{p} * {n}x{n}x{p} L={levels}, rows of A and B sharded over "
                      f"{G} GPUs, B all-gathered (NCCL)",
            "metric": "TFLOP/s (facewise products)", "value": flops * steps / (ms * 1e-3) / 1e12,
            "ms_per_call": ms / steps, "scaling": "strong", "row0": r0}


def bench_sp_w_svd(dist_mod, timed_region, steps=3, warmup=1, shape=(1024, 1024, 256), r=30,
                   levels=4, fused=False, full=False):
    """Config 4 sp-w-svd (or, with ``full``, config 3 w-svd reconstruction over all
    p wavelet slices) strong-scaled over the group (rows sharded; see bench.py)."""
    from . import synth

    G = dist_mod.get_world_size()
    me = dist_mod.get_rank()
    n1, n2, p = shape
    rows = splits(n1, G)
    r0 = sum(rows[:me])
    # rank 0 generates the cube once and broadcasts it (NVLink); each rank keeps its rows
    if me == 0:
        cube = torch.from_numpy(synth.hyperspectral_cube(n1, n2, p, seed=0)).cuda()
    else:
        cube = torch.empty((n1, n2, p), dtype=torch.float64, device="cuda")
    dist_mod.broadcast(cube, src=0)
    x = cube[r0:r0 + rows[me]].contiguous()
    del cube
    out = {}

    if full:
        fn = w_svd_recon_fused if fused else w_svd_recon_sharded
    else:
        fn = sp_w_svd_fused if fused else sp_w_svd_sharded

    def step(record):
        out["y"] = fn(x, r, levels, n1)

    ms = timed_region(step, steps, warmup, dist_mod)
    total = n1 * n2 * p
    k = p if full else 2 * (p >> levels)
    how = ("peer stores/loads fused into K1/K2 (symmetric memory)" if fused
           else "NCCL all-to-all")
    what = "w_svd recon" if full else "sp_w_svd"
    return {"config": f"{what} {n1}x{n2}x{p} rank {r} L={levels}, rows sharded over {G} GPUs, "
                      f"{k} wavelet slices exchanged by {how}",
            "metric": "tensor-elems/s", "value": total * steps / (ms * 1e-3), "ms_per_call": ms / steps,
            "scaling": "strong", "exchange_bytes_per_rank": 2 * 8 * k * rows[me] * n2}
