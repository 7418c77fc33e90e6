"""Device-resident engine: thin wrappers over the C ABI on torch CUDA tensors.

Every function takes and returns float64 CUDA tensors and runs on torch's
current stream, so it composes with torch.distributed / CUDA graphs.  The
public, reference-shaped API (``lifting``, ``algebra``, ``decomposition``) is
built on these.  Packed pyramids are slice-major ``(slices, n1, n2)`` buffers in
block order ``[d1 | ... | dL | sL]`` (include/wten_b200.h).
"""

from __future__ import annotations

import contextlib
import threading
import weakref

import numpy as np
import torch

from . import _native as N

F64 = torch.float64


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int:
    return 0 if t is None else t.data_ptr()


def detail_offset(p: int, j: int) -> int:
    """First packed slice of detail level j (1-based)."""
    return p - (p >> (j - 1))


def smooth_offset(p: int, levels: int) -> int:
    return p - (p >> levels)


def block_slices(p: int, levels: int):
    """[(tag, first_slice, count)] in packed order d1..dL, s (decomposition.py:98-99 order)."""
    out = [(f"d{j}", detail_offset(p, j), p >> j) for j in range(1, levels + 1)]
    out.append(("s", smooth_offset(p, levels), p >> levels))
    return out


def level_mask(levels: int, smooth: bool = True, details=None) -> int:
    """Bit 0 = smooth, bit j = detail level j."""
    m = 1 if smooth else 0
    for j in (range(1, levels + 1) if details is None else details):
        m |= 1 << j
    return m


_STAGE_ELEMS = 4 << 20   # 32 MB pinned staging chunks
_STAGE_SLOTS = 3
_stage_ring: list = []
_stage_lock = threading.Lock()  # the ring is shared: one uploader at a time


def _upload(host: torch.Tensor, device) -> torch.Tensor:
    """H2D of a contiguous host f64 tensor through a ring of pinned chunks: the
    (multi-threaded) host copy of chunk i+1 overlaps the DMA of chunk i.  A
    pageable tensor.to("cuda") runs at ~9 GB/s on the B200 boxes; this at the
    PCIe rate (tools/h2d_probe.py)."""
    with _stage_lock:
        return _upload_locked(host, device)


def _upload_locked(host: torch.Tensor, device) -> torch.Tensor:
    global _stage_ring
    if not _stage_ring:
        _stage_ring = [(torch.empty(_STAGE_ELEMS, dtype=F64, pin_memory=True), torch.cuda.Event())
                       for _ in range(_STAGE_SLOTS)]
    out = torch.empty(host.shape, dtype=F64, device=device)
    src, dst = host.reshape(-1), out.view(-1)
    # the copies run on (and the slot events record) the DESTINATION device's
    # stream, so an event tracks its DMA even when `device` is not the current one
    with torch.cuda.device(out.device):
        stream = torch.cuda.current_stream()
        for i, s0 in enumerate(range(0, src.numel(), _STAGE_ELEMS)):
            buf, ev = _stage_ring[i % _STAGE_SLOTS]
            ev.synchronize()                     # the slot's previous DMA has drained
            m = min(_STAGE_ELEMS, src.numel() - s0)
            buf[:m].copy_(src[s0:s0 + m])
            dst[s0:s0 + m].copy_(buf[:m], non_blocking=True)
            ev.record(stream)
    return out


def as_device(x, device=None) -> torch.Tensor:
    """float64, C-contiguous CUDA tensor (H2D copy for host inputs)."""
    N.require_gpu()
    if isinstance(x, torch.Tensor):
        t = x
        if t.is_cuda:
            return (t if t.dtype == F64 else t.to(F64)).contiguous()
        t = t.to(F64).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))
    if t.numel() >= 2 * _STAGE_ELEMS and not t.is_pinned():
        return _upload(t, device or "cuda")
    return t.to(device or "cuda").contiguous()


def is_pinned_array(a) -> bool:
    """True for a C-contiguous float64 numpy array in page-locked (CUDA-registered) memory:
    the streamed host paths DMA such inputs in place instead of staging them."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.size):
        return False
    try:
        return bool(torch.from_numpy(a).is_pinned())
    except (RuntimeError, ValueError, TypeError):  # read-only or exotic buffers
        return False


def pinned_empty(shape) -> np.ndarray:
    """An uninitialised float64 numpy array in page-locked memory (kept alive by the array).
    Cubes built in such arrays are uploaded by DMA straight from the array (no staging copy):
    the config-4 sp_w_svd call takes ~41 instead of ~59 ms to get its 2 GiB input on the GPU."""
    N.require_gpu()
    return torch.empty(tuple(int(d) for d in np.atleast_1d(shape)), dtype=F64, pin_memory=True).numpy()


# ----------------------------------------------------------- host results ----
# Large results handed to numpy callers live in pinned memory only while that is
# cheap: a pool of at most two pinned buffers per size (and _POOL_BYTES in all)
# that no handed-out array still references.  A caller who keeps every result
# would otherwise make each call page-lock a fresh multi-GB block (~0.9 s for
# 2 GiB, more than the whole computation); beyond the pool the result goes to
# pageable memory through the pinned download ring instead (~2x the DMA time).
_POOL_MIN_ELEMS = 8 << 20   # 64 MB: smaller results use torch's caching host allocator
_POOL_PER_SIZE = 4          # (a depth-3 pipeline of calls plus the result the caller still holds)
_POOL_BYTES = 8 << 30
_pool: dict = {}            # numel -> [[pinned tensor, state]]; state: None free, _BUSY, weakref to the ndarray
_BUSY = object()
_pool_lock = threading.Lock()
_dl_ring: list = []         # pinned download staging slots (for pageable results)
_dl_lock = threading.Lock()


def host_buffer(numel: int) -> torch.Tensor:
    """1-D CPU f64 buffer for a host result (pinned when the pool has one to spare)."""
    if numel < _POOL_MIN_ELEMS:
        return torch.empty(numel, dtype=F64, pin_memory=True)
    with _pool_lock:
        lst = _pool.setdefault(numel, [])
        for ent in lst:
            st = ent[1]
            if st is None or (st is not _BUSY and st() is None):
                ent[1] = _BUSY
                return ent[0]
        pooled = sum(len(v) * k for k, v in _pool.items()) * 8
        if len(lst) < _POOL_PER_SIZE and pooled + numel * 8 > _POOL_BYTES:
            # over the cap: give up unreferenced buffers of other sizes (a workload of another shape
            # came before; its buffers go back to torch's caching host allocator)
            for k in list(_pool):
                if k == numel:
                    continue
                keep = [e for e in _pool[k] if not (e[1] is None or (e[1] is not _BUSY and e[1]() is None))]
                pooled -= (len(_pool[k]) - len(keep)) * k * 8
                _pool[k] = keep
                if pooled + numel * 8 <= _POOL_BYTES:
                    break
        if len(lst) < _POOL_PER_SIZE and pooled + numel * 8 <= _POOL_BYTES:
            t = torch.empty(numel, dtype=F64, pin_memory=True)
            lst.append([t, _BUSY])
            return t
    return torch.empty(numel, dtype=F64)


def hand_out(t: torch.Tensor) -> np.ndarray:
    """The numpy array of a host_buffer() result for the caller; a pooled buffer
    returns to the pool once that array and every view of it are gone."""
    arr = t.numpy()
    with _pool_lock:
        for ent in _pool.get(t.numel(), []):
            if ent[0].data_ptr() == t.data_ptr():
                ent[1] = weakref.ref(arr)
    return arr


def release(t: torch.Tensor) -> None:
    """Return a host_buffer() result that is not handed out (error paths)."""
    with _pool_lock:
        for ent in _pool.get(t.numel(), []):
            if ent[0].data_ptr() == t.data_ptr():
                ent[1] = None


class Download:
    """D2H of device pieces into a 1-D host buffer on the current stream: direct
    DMA into pinned memory, else through the pinned download ring (each slot's
    host copy runs when the slot is reused, overlapping the other slots' DMA)."""

    def __init__(self, host: torch.Tensor):
        self.host = host
        self.direct = host.is_pinned()
        self.pending = []
        self.i = 0
        if not self.direct:
            _dl_lock.acquire()
            if not _dl_ring:
                _dl_ring.extend((torch.empty(_STAGE_ELEMS, dtype=F64, pin_memory=True), torch.cuda.Event())
                                for _ in range(_STAGE_SLOTS + 1))

    def put(self, lo: int, src: torch.Tensor) -> None:
        src = src.reshape(-1)
        n = src.numel()
        if self.direct:
            self.host[lo:lo + n].copy_(src, non_blocking=True)
            return
        stream = torch.cuda.current_stream()
        for c0 in range(0, n, _STAGE_ELEMS):
            m = min(_STAGE_ELEMS, n - c0)
            slot = self.i % len(_dl_ring)
            self.i += 1
            self._drain(slot)
            buf, ev = _dl_ring[slot]
            buf[:m].copy_(src[c0:c0 + m], non_blocking=True)
            ev.record(stream)
            self.pending.append((slot, lo + c0, m))

    def _drain(self, slot=None) -> None:
        keep = []
        for ent in self.pending:
            s, lo, m = ent
            if slot is None or s == slot:
                buf, ev = _dl_ring[s]
                ev.synchronize()
                self.host[lo:lo + m].copy_(buf[:m])
            else:
                keep.append(ent)
        self.pending = keep

    def finish(self) -> None:
        """Wait for every piece (host copies done; pinned: the caller synchronizes)."""
        if not self.direct:
            try:
                self._drain()
            finally:
                _dl_lock.release()


def to_host(t: torch.Tensor) -> np.ndarray:
    """D2H of a result into host memory (pinned when cheap: host_buffer)."""
    t = t.contiguous()
    h = host_buffer(t.numel())
    dl = Download(h)
    try:
        dl.put(0, t)
    finally:
        dl.finish()
    if dl.direct:
        torch.cuda.current_stream().synchronize()
    return hand_out(h).reshape(t.shape)


# ------------------------------------------------- host-streamed transform ----

_PIPE_STREAMS: dict = {}
_CHUNK_BYTES = 32 << 20


def _pipe_streams():
    dev = torch.cuda.current_device()
    key = (dev, threading.get_ident())  # per host thread: concurrent calls must not queue behind each other
    if key not in _PIPE_STREAMS:
        _PIPE_STREAMS[key] = tuple(torch.cuda.Stream() for _ in range(3))
    return _PIPE_STREAMS[key]


def _row_chunks(n1: int, row_elems: int):
    rows = max(1, min(n1, _CHUNK_BYTES // max(1, 8 * row_elems)))
    return rows, [(r0, min(n1, r0 + rows)) for r0 in range(0, n1, rows)]


def host_lift(src, n1: int, n2: int, p: int, levels: int, forward: bool) -> torch.Tensor:
    """The numpy drop-in transform, streamed through the GPU in row chunks.

    forward: ``src`` is the (n1, n2, p) host cube; returns the tube-major packed
    pyramid (the reference's per-level arrays back to back) in pinned memory.
    inverse: ``src`` is that pinned packed pyramid; returns the pinned cube.
    Per chunk of rows: host -> pinned staging (forward only), H2D, K1 / K2, and
    D2H straight into the pinned result run on three streams, so the staging
    copy, both PCIe directions and the kernels overlap (the transform is
    row-separable: a chunk's rows are contiguous in every tube-major block).
    """
    lib = N.require_gpu()  # noqa: F841  (fail loudly without the library / a GPU)
    nt = n1 * n2
    rows, chunks = _row_chunks(n1, n2 * p)
    blocks = [(off, cnt) for _, off, cnt in block_slices(p, levels)]
    out = host_buffer(nt * p)
    s_in, s_cmp, s_out = _pipe_streams()
    main = torch.cuda.current_stream()
    for st in (s_in, s_cmp, s_out):
        st.wait_stream(main)
    if not forward and not src.is_pinned():  # a pageable pyramid (host_buffer fallback): stage it up whole
        src = _upload(src, "cuda")
        for st in (s_in, s_cmp, s_out):
            st.wait_stream(main)
    cap = rows * n2 * p
    direct = forward and is_pinned_array(src)
    with _stage_lock:
        if forward and not _stage_ring:
            _upload_locked(torch.empty(0, dtype=F64), "cuda")  # allocate the pinned ring
        dx = [torch.empty(cap, dtype=F64, device="cuda") for _ in range(2)]
        dy = [torch.empty(cap, dtype=F64, device="cuda") for _ in range(2)]
        free_in = [None, None]   # dx[b] consumed by the kernel
        free_out = [None, None]  # dy[b] drained by the D2H
        dl = Download(out)
        for i, (r0, r1) in enumerate(chunks):
            b = i % 2
            rn = (r1 - r0) * n2
            n = rn * p
            with torch.cuda.stream(s_in):
                if free_in[b] is not None:
                    s_in.wait_event(free_in[b])
                if forward and direct:  # page-locked cube: DMA in place
                    dx[b][:n].copy_(torch.from_numpy(src[r0:r1]).reshape(-1), non_blocking=True)
                elif forward:
                    stage, ev = _stage_ring[i % _STAGE_SLOTS]
                    ev.synchronize()
                    part = torch.from_numpy(src[r0:r1]).reshape(-1)
                    for c0 in range(0, n, _STAGE_ELEMS):    # chunks above the ring slot size
                        m = min(_STAGE_ELEMS, n - c0)
                        if c0:
                            ev.record(s_in)
                            ev.synchronize()
                        stage[:m].copy_(part[c0:c0 + m])
                        dx[b][c0:c0 + m].copy_(stage[:m], non_blocking=True)
                    ev.record(s_in)
                else:
                    for off, cnt in blocks:  # this chunk's rows of every block
                        dx[b][off * rn:(off + cnt) * rn].copy_(
                            src[off * nt + r0 * n2 * cnt:off * nt + r1 * n2 * cnt], non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(loaded)
                if free_out[b] is not None:
                    s_cmp.wait_event(free_out[b])
                if forward:
                    lift_forward(dx[b][:n].view(r1 - r0, n2, p), levels, layout=N.LAYOUT_TUBE,
                                 out=dy[b][:n].view(p, r1 - r0, n2))
                else:
                    lift_inverse(dx[b][:n], r1 - r0, n2, p, levels, layout=N.LAYOUT_TUBE,
                                 out=dy[b][:n].view(r1 - r0, n2, p))
                free_in[b] = torch.cuda.Event()
                free_in[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(free_in[b])
                if forward:
                    for off, cnt in blocks:
                        dl.put(off * nt + r0 * n2 * cnt, dy[b][off * rn:(off + cnt) * rn])
                else:
                    dl.put(r0 * n2 * p, dy[b][:n])
                free_out[b] = torch.cuda.Event()
                free_out[b].record(s_out)
        s_out.synchronize()
        dl.finish()
        main.wait_stream(s_out)
    return out


_download_lock = threading.Lock()


def host_slices_pipeline(src: np.ndarray, levels: int, mask: int, base: int, decompose,
                         out_rows: int, out_cols: int) -> np.ndarray:
    """Host cube in, host cube out, with the PCIe traffic overlapped with K1 / K2.

    ``src`` is the (n1, n2, p) host array.  Row chunks of it are staged through
    the pinned ring, copied H2D and lifted by K1, which stores each chunk's rows
    of packed slices ``base .. p-1`` (as selected by ``mask``) straight into the
    device slice buffer (p - base, n1, n2) through a per-chunk table of row-block
    addresses (wt_lift_fwd_f64_peer), so H2D of chunk i+1 overlaps K1 of chunk i.
    ``decompose(slices)`` returns the (p - base, out_rows, out_cols) result slices;
    K2 then loads them back chunk by chunk of result rows (wt_lift_inv_f64_peer)
    while the D2H of the previous chunk drains into the pinned result.  Returns
    the (out_rows, out_cols, p) result as a numpy array (pinned memory from
    host_buffer's pool when one is free, else pageable).
    """
    lib = N.require_gpu()  # noqa: F841  (fail loudly without the library / a GPU)
    n1, n2, p = src.shape
    K = p - base
    dev = torch.device("cuda", torch.cuda.current_device())
    slices = torch.empty((K, n1, n2), dtype=F64, device=dev)
    s_in, s_cmp, s_out = _pipe_streams()
    main = torch.cuda.current_stream()
    for st in (s_in, s_cmp, s_out):
        st.wait_stream(main)

    def tables(buf, rows_total, cols, rows_per_chunk, chunks):
        # (len(chunks), K) row-block addresses, computed ON the device (chunk c starts at row
        # c * rows_per_chunk): a pageable H2D copy of the table would queue on the upload copy
        # engine behind the bulk chunks of other calls in flight (sp_w_svd_many) -- up to a whole
        # cube, ~39 ms -- and stall this call's K2 / download.  The consumer stream waits for it.
        ks = torch.arange(K, dtype=torch.int64, device=dev)[None, :] * rows_total
        r0s = torch.arange(len(chunks), dtype=torch.int64, device=dev)[:, None] * rows_per_chunk
        t = (ks + r0s) * (cols * 8) + buf.data_ptr()
        s_cmp.wait_stream(torch.cuda.current_stream())
        return t

    rows, chunks = _row_chunks(n1, n2 * p)
    tab_f = tables(slices, n1, n2, rows, chunks)
    direct = is_pinned_array(src)
    cap = rows * n2 * p
    with _stage_lock:
        if not _stage_ring:
            _upload_locked(torch.empty(0, dtype=F64), dev)  # allocate the pinned ring
        dx = [torch.empty(cap, dtype=F64, device=dev) for _ in range(2)]
        free_in = [None, None]
        for i, (r0, r1) in enumerate(chunks):
            b = i % 2
            n = (r1 - r0) * n2 * p
            with torch.cuda.stream(s_in):
                if free_in[b] is not None:
                    s_in.wait_event(free_in[b])
                part = torch.from_numpy(src[r0:r1]).reshape(-1)
                if direct:  # page-locked source: DMA in place
                    dx[b][:n].copy_(part, non_blocking=True)
                for c0 in range(0, 0 if direct else n, _STAGE_ELEMS):
                    stage, ev = _stage_ring[(i + c0 // _STAGE_ELEMS) % _STAGE_SLOTS]
                    ev.synchronize()
                    m = min(_STAGE_ELEMS, n - c0)
                    stage[:m].copy_(part[c0:c0 + m])
                    dx[b][c0:c0 + m].copy_(stage[:m], non_blocking=True)
                    ev.record(s_in)
                loaded = torch.cuda.Event()
                loaded.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(loaded)
                lift_forward_peer(dx[b][:n].view(r1 - r0, n2, p), levels, tab_f[i], mask, base)
                free_in[b] = torch.cuda.Event()
                free_in[b].record(s_cmp)
        # The lock is kept until this cube has ARRIVED: concurrent calls (sp_w_svd_many) then upload
        # one after the other at the full PCIe rate instead of chunk by chunk side by side, so the
        # next call's upload runs under this call's K4 and download (two interleaved uploads end
        # together, and so do their K4s and downloads: ~61 instead of ~41 ms per config-4 cube).
        loaded.synchronize()
    main.wait_stream(s_cmp)
    result = decompose(slices)                                  # (K, out_rows, out_cols)
    for st in (s_cmp, s_out):
        st.wait_stream(main)
    orows, ochunks = _row_chunks(out_rows, out_cols * p)
    tab_i = tables(result, out_rows, out_cols, orows, ochunks)
    out = host_buffer(out_rows * out_cols * p)
    ocap = orows * out_cols * p
    dy = [torch.empty(ocap, dtype=F64, device=dev) for _ in range(2)]
    free_out = [None, None]
    dl = Download(out)
    with _download_lock:  # (one result at a time on the D2H engine, for the same reason)
        for i, (r0, r1) in enumerate(ochunks):
            b = i % 2
            n = (r1 - r0) * out_cols * p
            with torch.cuda.stream(s_cmp):
                if free_out[b] is not None:
                    s_cmp.wait_event(free_out[b])
                lift_inverse_peer(tab_i[i], r1 - r0, out_cols, p, levels, mask, base,
                                  out=dy[b][:n].view(r1 - r0, out_cols, p))
                done = torch.cuda.Event()
                done.record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done)
                dl.put(r0 * out_cols * p, dy[b][:n])
                free_out[b] = torch.cuda.Event()
                free_out[b].record(s_out)
        s_out.synchronize()
        dl.finish()
    main.wait_stream(s_out)
    result.record_stream(s_cmp)
    return hand_out(out).reshape(out_rows, out_cols, p)


# --------------------------------------------------------------- lifting ----

def lift_forward(x: torch.Tensor, levels: int, layout: int = N.LAYOUT_SLICE,
                 mask: int = N.MASK_ALL, slice_base: int = 0,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """K1 on a contiguous (n1, n2, p) tensor -> packed buffer (slices-slice_base, n1, n2)."""
    lib = N.require_gpu()
    n1, n2, p = x.shape
    if out is None:
        out = torch.empty((p - slice_base, n1, n2), dtype=F64, device=x.device)
    N.check(lib.wt_lift_fwd_f64(_ptr(x), n1, n2, p, levels, _ptr(out), layout, slice_base,
                                mask & N.MASK_ALL, _stream()), "wt_lift_fwd_f64")
    return out


def lift_inverse(buf: torch.Tensor, n1: int, n2: int, p: int, levels: int,
                 layout: int = N.LAYOUT_SLICE, mask: int = N.MASK_ALL, slice_base: int = 0,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """K2: packed buffer -> contiguous (n1, n2, p) tensor."""
    lib = N.require_gpu()
    if out is None:
        out = torch.empty((n1, n2, p), dtype=F64, device=buf.device)
    N.check(lib.wt_lift_inv_f64(_ptr(buf), n1, n2, p, levels, layout, slice_base,
                                mask & N.MASK_ALL, _ptr(out), _stream()), "wt_lift_inv_f64")
    return out


def lift_forward_peer(x: torch.Tensor, levels: int, table: torch.Tensor, mask: int = N.MASK_ALL,
                      slice_base: int = 0) -> None:
    """K1 storing packed slice s of x's tubes at table[s - slice_base] (device int64 addresses,
    possibly on peer GPUs): the fused rows -> slices exchange."""
    lib = N.require_gpu()
    n1, n2, p = x.shape
    assert table.dtype == torch.int64 and table.is_cuda and table.numel() == p - slice_base
    N.check(lib.wt_lift_fwd_f64_peer(_ptr(x), n1, n2, p, levels, _ptr(table), slice_base,
                                     mask & N.MASK_ALL, _stream()), "wt_lift_fwd_f64_peer")


def lift_inverse_peer(table: torch.Tensor, n1: int, n2: int, p: int, levels: int,
                      mask: int = N.MASK_ALL, slice_base: int = 0,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """K2 loading packed slice s of this rank's tubes from table[s - slice_base]."""
    lib = N.require_gpu()
    if out is None:
        out = torch.empty((n1, n2, p), dtype=F64, device=table.device)
    N.check(lib.wt_lift_inv_f64_peer(_ptr(table), n1, n2, p, levels, slice_base, mask & N.MASK_ALL,
                                     _ptr(out), _stream()), "wt_lift_inv_f64_peer")
    return out


_WP_WS: dict = {}  # (device, stream) -> cached workspace of the one-call w-product


def w_product(a: torch.Tensor, b: torch.Tensor, levels: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """K1, K1, K3, K2 of a w-product in ONE C-ABI call (wt_w_product_f64); a, b
    C-contiguous CUDA f64.  The pyramid workspace is cached per device and stream
    (repeated calls on resident tensors replay a CUDA graph of the four launches)."""
    lib = N.require_gpu()
    n1, n2, p = a.shape
    n3 = b.shape[1]
    if out is None:
        out = torch.empty((n1, n3, p), dtype=F64, device=a.device)
    need = int(lib.wt_w_product_workspace_bytes(n1, n2, n3, p))
    key = (a.device.index, _stream())
    ws = _WP_WS.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.empty((max(need, 1),), dtype=torch.uint8, device=a.device)
        _WP_WS[key] = ws
    N.check(lib.wt_w_product_f64(_ptr(a), _ptr(b), n1, n2, n3, p, levels, _ptr(out), _ptr(ws), ws.numel(),
                                 _stream()), "wt_w_product_f64")
    return out


# ------------------------------------------------------------------ GEMM ----

def gemm(a: torch.Tensor, b: torch.Tensor, trans_a: bool = False, trans_b: bool = False,
         alpha: float = 1.0, beta: float = 0.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """K3: batched C[k] = alpha op(A[k]) op(B[k]) + beta C[k] for (batch, rows, cols) tensors.

    Operands may be any 3-D views whose last dimension is contiguous.
    """
    lib = N.require_gpu()
    assert a.dim() == 3 and b.dim() == 3 and a.shape[0] == b.shape[0]
    assert a.stride(2) == 1 and b.stride(2) == 1
    batch = a.shape[0]
    M, K = (a.shape[2], a.shape[1]) if trans_a else (a.shape[1], a.shape[2])
    K2, Nn = (b.shape[2], b.shape[1]) if trans_b else (b.shape[1], b.shape[2])
    assert K == K2, f"inner dimensions differ: {K} vs {K2}"
    if out is None:
        out = torch.empty((batch, M, Nn), dtype=F64, device=a.device)
    assert out.stride(2) == 1
    N.check(lib.wt_gemm_f64(int(trans_a), int(trans_b), M, Nn, K, float(alpha), _ptr(a),
                            a.stride(1), a.stride(0), _ptr(b), b.stride(1), b.stride(0),
                            float(beta), _ptr(out), out.stride(1), out.stride(0), batch,
                            _stream()), "wt_gemm_f64")
    return out


def copy2d(src: torch.Tensor, trans: bool, out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched (transposing) copy of (batch, r, c) views."""
    lib = N.require_gpu()
    batch, r, c = src.shape
    assert src.stride(2) == 1
    shape = (batch, c, r) if trans else (batch, r, c)
    if out is None:
        out = torch.empty(shape, dtype=F64, device=src.device)
    assert out.stride(2) == 1
    N.check(lib.wt_copy2d_f64(_ptr(src), src.stride(1), src.stride(0), _ptr(out), out.stride(1),
                              out.stride(0), shape[1], shape[2], batch, int(trans), _stream()),
            "wt_copy2d_f64")
    return out


def scale_cols(m: torch.Tensor, s: torch.Tensor, mode: int, tol: float = 0.0,
               ncols: int | None = None) -> torch.Tensor:
    """In place: m[k][:, j] *= f(s[k][j]) (see WT_SCALE_*)."""
    lib = N.require_gpu()
    batch, rows, cols = m.shape
    ncols = cols if ncols is None else ncols
    assert m.stride(2) == 1 and s.is_contiguous()
    N.check(lib.wt_scale_cols_f64(_ptr(m), rows, ncols, m.stride(1), m.stride(0), _ptr(s),
                                  s.shape[-1], batch, mode, float(tol), _stream()),
            "wt_scale_cols_f64")
    return m


# ------------------------------------------------------------------- SVD ----

def orthonormal_fixup(m: torch.Tensor, s: torch.Tensor, tau: float) -> torch.Tensor:
    """In place: re-orthonormalise the columns j of m[k] (rows x r) with s[k][j] <= tau * s[k][0]
    (wt_orthonormal_fixup_f64); m's column order is s's (descending)."""
    lib = N.require_gpu()
    batch, rows, r = m.shape
    assert m.stride(2) == 1 and s.is_contiguous()
    N.check(lib.wt_orthonormal_fixup_f64(_ptr(m), rows, r, m.stride(1), m.stride(0), _ptr(s), s.shape[-1], batch,
                                         float(tau), _stream()), "wt_orthonormal_fixup_f64")
    return m


def diag_blocks(sigma: torch.Tensor, r: int) -> torch.Tensor:
    """(batch, q) singular values -> (batch, r, r) diagonal S blocks (wt_diag_blocks_f64)."""
    lib = N.require_gpu()
    batch, q = sigma.shape
    out = torch.empty((batch, r, r), dtype=F64, device=sigma.device)
    N.check(lib.wt_diag_blocks_f64(_ptr(sigma), q, r, batch, _ptr(out), _stream()), "wt_diag_blocks_f64")
    return out


def lu_zero_pivot(a: torch.Tensor) -> torch.Tensor:
    """(batch, n, n) -> int32 (batch,): 1 + first exactly-zero pivot of partial-pivoting LU, else 0."""
    lib = N.require_gpu()
    w = a.contiguous().clone()
    batch, n, _ = w.shape
    info = torch.empty((batch,), dtype=torch.int32, device=a.device)
    N.check(lib.wt_lu_pivot_check_f64(_ptr(w), n, batch, _ptr(info), _stream()), "wt_lu_pivot_check_f64")
    return info


# Test / diagnostic switches of the library (wt_set_option; include/wten_b200.h).
OPTIONS = {"svd_split": 0, "svd_ctas_per_sm": 1, "svd_pair_skip": 2, "svd_persist": 3, "svd_precond": 4,
           "svd_profile": 5, "svd_trace": 6, "eig_profile": 7, "eig_twostage": 8, "gemm_tma": 9, "eig_split": 10}


def set_option(name: str, value: int) -> int:
    """Set a library switch (tests / diagnostics only); returns the previous value."""
    return int(N.load().wt_set_option(OPTIONS[name], int(value)))


def options_from_env() -> None:
    """Diagnostics tools (tools/*.py): WT_OPT_<NAME>=value environment variables set the
    switches above (the library itself reads no environment)."""
    import os

    for name in OPTIONS:
        v = os.environ.get("WT_OPT_" + name.upper())
        if v is not None:
            set_option(name, int(v))


@contextlib.contextmanager
def option(name: str, value: int):
    """``with option("svd_split", 4): ...`` -- the switch is restored afterwards."""
    old = set_option(name, value)
    try:
        yield
    finally:
        set_option(name, old)


class SvdNotConverged(RuntimeError):
    pass


def svd(a: torch.Tensor, nvec: int, tol: float = 0.0, max_sweeps: int = 0):
    """K4 over a batch of row-major matrices a (batch, n1, n2) (last dim contiguous).

    Returns (sigma (batch, q) descending, vec (batch, nvec, max(n1, n2)), info (batch,) int32):
    vec rows are the long-side singular vectors (right if n1 <= n2, else left).
    """
    lib = N.require_gpu()
    batch, n1, n2 = a.shape
    assert a.stride(2) == 1
    q, ln = min(n1, n2), max(n1, n2)
    sigma = torch.empty((batch, q), dtype=F64, device=a.device)
    vec = torch.empty((batch, nvec, ln), dtype=F64, device=a.device)
    info = torch.empty((batch,), dtype=torch.int32, device=a.device)
    if batch == 0:
        return sigma, vec, info
    # (K4 runs batches above 65535 matrices in chunks through a workspace prefix)
    wsb = int(lib.wt_svd_workspace_bytes(n1, n2, min(batch, 65535)))
    ws = torch.empty((wsb,), dtype=torch.uint8, device=a.device)
    N.check(lib.wt_svd_jacobi_f64(_ptr(a), a.stride(1), a.stride(0), n1, n2, batch, _ptr(sigma),
                                  _ptr(vec), nvec, _ptr(info), float(tol), int(max_sweeps),
                                  _ptr(ws), wsb, _stream()), "wt_svd_jacobi_f64")
    return sigma, vec, info


def svd_topk(a: torch.Tensor, k: int, nvec: int, tol: float = 0.0, max_sweeps: int = 0):
    """K4, the k leading singular triplets of every (n1, n2) slice (wt_svd_topk_f64):
    (sigma (batch, k) descending, vec (batch, nvec, max(n1, n2)), info)."""
    lib = N.require_gpu()
    batch, n1, n2 = a.shape
    assert a.stride(2) == 1 and 1 <= nvec <= k
    ln = max(n1, n2)
    sigma = torch.empty((batch, k), dtype=F64, device=a.device)
    vec = torch.empty((batch, nvec, ln), dtype=F64, device=a.device)
    info = torch.empty((batch,), dtype=torch.int32, device=a.device)
    if batch == 0:
        return sigma, vec, info
    wsb = int(lib.wt_svd_topk_workspace_bytes(n1, n2, batch, k))
    ws = torch.empty((wsb,), dtype=torch.uint8, device=a.device)
    N.check(lib.wt_svd_topk_f64(_ptr(a), a.stride(1), a.stride(0), n1, n2, batch, k, _ptr(sigma), _ptr(vec), nvec,
                                _ptr(info), float(tol), int(max_sweeps), _ptr(ws), wsb, _stream()),
            "wt_svd_topk_f64")
    return sigma, vec, info


def topk_width(q: int, r: int) -> int:
    """Leading triplets computed for a rank-r truncation of slices with q = min(n1, n2):
    k = max(64, 2r) rounded up to 32 when that is at most q / 2 (else 0: full SVD)."""
    k = max(64, (2 * r + 31) // 32 * 32)
    return k if q >= 256 and k <= q // 2 else 0


def svd_truncated_recon(a: torch.Tensor, r: int, out: torch.Tensor | None = None, tol: float = 0.0) -> torch.Tensor:
    """Rank-r reconstruction of every slice (_stack_svd + _truncated_blocks,
    decomposition.py:64-72): K4 on the k leading triplets when k = topk_width(q, r)
    applies, the full K4 otherwise, then K5."""
    batch, n1, n2 = a.shape
    k = topk_width(min(n1, n2), r)
    if k:
        sigma, vec, info = svd_topk(a, k, r, tol=tol)
    else:
        sigma, vec, info = svd(a, r, tol=tol)
    raise_if_failed(info)
    return truncated_recon(a, sigma, vec, r, out=out)


def last_sweeps() -> int:
    return int(N.load().wt_svd_last_sweeps())


def last_jacobi_flops() -> float:
    """FP64 flops executed by the last K4 call's Jacobi iteration (this thread)."""
    return float(N.load().wt_svd_last_jacobi_flops())


_readback_tls = threading.local()


def raise_if_failed(info: torch.Tensor):
    """Map K4 status to the reference's LAPACK error (numpy.linalg.LinAlgError).

    info 1 (non-finite data) and info 2 (sweep limit reached before the
    convergence test passed) both raise ``LinAlgError("SVD did not converge")``,
    as dgesdd does when its iteration fails (decomposition.py:66 via
    np.linalg.svd).  One small readback of the status vector, no torch kernels."""
    if info.numel() == 0:
        return
    if info.is_cuda and info.dtype == torch.int32 and info.is_contiguous():
        # wt_readback_i32: a one-warp kernel writes the status words into page-locked host memory
        # (per host thread) and the stream is synchronised -- no copy-engine copy, which would
        # queue behind the bulk transfers of other calls in flight (sp_w_svd_many)
        n = info.numel()
        buf = getattr(_readback_tls, "buf", None)
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(n, 1024), dtype=torch.int32, pin_memory=True)
            _readback_tls.buf = buf
        with torch.cuda.device(info.device):
            N.check(N.require_gpu().wt_readback_i32(_ptr(info), buf.data_ptr(), n, _stream()), "wt_readback_i32")
        failed = bool((buf[:n] != 0).any())
    else:
        failed = bool((info.cpu() != 0).any())
    if failed:
        raise np.linalg.LinAlgError("SVD did not converge")


def truncated_recon(a: torch.Tensor, sigma: torch.Tensor, vec: torch.Tensor, r: int,
                    out: torch.Tensor | None = None, keep_t: bool = False):
    """K5 (wt_svd_truncate_f64): rank-r reconstruction of every slice from the long-side vectors.

    Right side (n1 <= n2): T = A V_r (n1 x r) and recon = T V_r^T.
    Left side  (n1 >  n2): T = A^T U_r (n2 x r) and recon = U_r T^T.
    Equal to U_r diag(s_r) V_r^T of decomposition.py:70-72.
    """
    lib = N.require_gpu()
    batch, n1, n2 = a.shape
    assert a.stride(2) == 1 and vec.is_contiguous()
    t = torch.empty((batch, min(n1, n2), r), dtype=F64, device=a.device)
    if out is None:
        out = torch.empty((batch, n1, n2), dtype=F64, device=a.device)
    assert out.stride(2) == 1
    N.check(lib.wt_svd_truncate_f64(_ptr(a), a.stride(1), a.stride(0), n1, n2, batch, _ptr(vec),
                                    vec.shape[1], r, _ptr(out), out.stride(1), out.stride(0), _ptr(t),
                                    _stream()), "wt_svd_truncate_f64")
    return (out, t) if keep_t else out


def svd_factors(t: torch.Tensor, vec: torch.Tensor, sigma: torch.Tensor, n1: int, n2: int, r: int):
    """K6 (wt_svd_factors_f64): U (batch, n1, r), V (batch, n2, r) from K5's T (decomposition.py:75-82)."""
    lib = N.require_gpu()
    batch = t.shape[0]
    assert t.is_contiguous() and vec.is_contiguous() and sigma.is_contiguous()
    u = torch.empty((batch, n1, r), dtype=F64, device=t.device)
    v = torch.empty((batch, n2, r), dtype=F64, device=t.device)
    N.check(lib.wt_svd_factors_f64(_ptr(t), _ptr(vec), vec.shape[1], _ptr(sigma), n1, n2, batch, r,
                                   _ptr(u), _ptr(v), _stream()), "wt_svd_factors_f64")
    return u, v


def pinv_blocks(a: torch.Tensor, sigma: torch.Tensor, vec: torch.Tensor, tol: float,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """K7 (wt_pinv_from_svd_f64): per-slice Moore-Penrose inverse (n2 x n1), cutoff tol*sigma_max.

    decomposition.py:157-163: A+ = V diag(s+) U^T, s+ = 1/s for s > tol*s_max.
    Right side: A+ = V (A V)^T weighted by s+^2; left side: A+ = (A^T U) s+^2 U^T.
    """
    lib = N.require_gpu()
    batch, n1, n2 = a.shape
    q = min(n1, n2)
    assert a.stride(2) == 1 and vec.is_contiguous() and vec.shape[1] == q and sigma.is_contiguous()
    t = torch.empty((batch, q, q), dtype=F64, device=a.device)
    if out is None:
        out = torch.empty((batch, n2, n1), dtype=F64, device=a.device)
    assert out.stride(2) == 1
    rank = torch.empty((batch,), dtype=torch.int32, device=a.device)
    # GEMMs limited per slice to the kept singular values (zero slices cost nothing)
    N.check(lib.wt_pinv_from_svd_ranked_f64(_ptr(a), a.stride(1), a.stride(0), n1, n2, batch,
                                            _ptr(sigma), _ptr(vec), float(tol), _ptr(out), out.stride(1),
                                            out.stride(0), _ptr(t), _ptr(rank), _stream()),
            "wt_pinv_from_svd_ranked_f64")
    return out


def tube_transpose(x: torch.Tensor) -> torch.Tensor:
    """(n1, n2, p) -> (n2, n1, p) slicewise transpose (wt_tube_transpose_f64)."""
    lib = N.require_gpu()
    x = x.contiguous()
    n1, n2, p = x.shape
    out = torch.empty((n2, n1, p), dtype=F64, device=x.device)
    N.check(lib.wt_tube_transpose_f64(_ptr(x), n1, n2, p, _ptr(out), _stream()), "wt_tube_transpose_f64")
    return out


def tube_delta(x: torch.Tensor) -> torch.Tensor:
    """(n1, n2, p) -> x[..., k] - x[..., 0] per tube (wt_tube_delta_f64)."""
    lib = N.require_gpu()
    assert x.is_contiguous()
    out = torch.empty_like(x)
    N.check(lib.wt_tube_delta_f64(_ptr(x), x.numel() // max(1, x.shape[-1]), x.shape[-1], _ptr(out),
                                  _stream()), "wt_tube_delta_f64")
    return out


# ------------------------------------------------------------ reductions ----

def band_sums(x: torch.Tensor, y: torch.Tensor | None, mode: int) -> torch.Tensor:
    """Per-band sums over a spatial (n1, n2, p) tensor (deterministic)."""
    lib = N.require_gpu()
    n1, n2, p = x.shape
    nt = n1 * n2
    scratch = int(lib.wt_slice_reduce_scratch(nt, p)) // 8
    out = torch.empty((scratch,), dtype=F64, device=x.device)
    N.check(lib.wt_slice_reduce_f64(_ptr(x), _ptr(y), nt, p, mode, _ptr(out), _stream()),
            "wt_slice_reduce_f64")
    return out[:p]


# --------------------------------------------------------- imaging helpers ----

def toeplitz_tensor(c: torch.Tensor, n: int, p: int) -> torch.Tensor:
    """(n, n, p) slice-constant symmetric Toeplitz operator c[|i - j|] (wt_toeplitz_tensor_f64)."""
    lib = N.require_gpu()
    c = c.contiguous()
    out = torch.empty((n, n, p), dtype=F64, device=c.device)
    N.check(lib.wt_toeplitz_tensor_f64(_ptr(c), c.numel(), n, p, _ptr(out), _stream()), "wt_toeplitz_tensor_f64")
    return out


def gauss_smooth2d(x: torch.Tensor, half_kernel: torch.Tensor) -> torch.Tensor:
    """Reflect-mode separable Gaussian filter over axes 0, 1 of (n1, n2, e) (wt_gauss_smooth2d_f64)."""
    lib = N.require_gpu()
    x = x.contiguous()
    n1, n2, e = x.shape
    tmp = torch.empty_like(x)
    out = torch.empty_like(x)
    N.check(lib.wt_gauss_smooth2d_f64(_ptr(x), n1, n2, e, _ptr(half_kernel), half_kernel.numel() - 1, _ptr(tmp),
                                      _ptr(out), _stream()), "wt_gauss_smooth2d_f64")
    return out


def hsi_mix(ab: torch.Tensor, spectra: torch.Tensor, noise_sigma: float, noise: torch.Tensor | None,
            seed: int, lo: float = 0.0, hi: float = 1.0) -> torch.Tensor:
    """clip(ab @ spectra + sigma * z, lo, hi) as an (n1, n2, p) cube (wt_hsi_mix_f64)."""
    lib = N.require_gpu()
    n1, n2, e = ab.shape
    p = spectra.shape[1]
    ab = ab.contiguous()
    spectra = spectra.contiguous()
    out = torch.empty((n1, n2, p), dtype=F64, device=ab.device)
    N.check(lib.wt_hsi_mix_f64(_ptr(ab), _ptr(spectra), n1 * n2, e, p, float(noise_sigma), _ptr(noise),
                               int(seed) & ((1 << 64) - 1), lo, hi, _ptr(out), _stream()), "wt_hsi_mix_f64")
    return out
