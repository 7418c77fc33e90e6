"""Forward / inverse lazy-lifting transform along mode 3 -- drop-in for
``wten.lifting`` (/root/reference/pkg/src/wten/lifting.py).

Same names, signatures, error types and messages.  Arithmetic runs on the GPU
(K1/K2 in csrc/lift_fast.cu, general layouts in csrc/lift.cu) and is
bit-identical to the reference.

Two calling modes:
  * host arrays (numpy, lists, ...): inputs are copied to the GPU and results
    come back as C-contiguous float64 numpy arrays, as in the reference;
  * CUDA torch tensors: everything stays resident; a pyramid's blocks are
    strided views of one packed slice-major buffer that
    ``inverse_w`` consumes directly.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from . import engine as E
from .errors import LevelError, ShapeError


def max_levels(p):
    """Largest L such that 2**L divides p (0 for odd p) -- lifting.py:17-21."""
    if p < 1:
        raise ValueError(f"slice count must be positive, got {p}")
    return ((p & -p).bit_length()) - 1


_STREAM_MIN = 1 << 22  # host inputs from 4 M elements (32 MB) stream through the GPU in row chunks


def _is_dev(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


class WaveletPyramid:
    """Multilevel wavelet representation (lifting.py:24-60).

    ``smooth`` holds the coarsest smooth stack with ``p / 2**levels`` slices;
    ``details[j - 1]`` the level-j detail stack with ``p / 2**j`` slices.
    Pyramids produced on the device additionally carry their packed buffer.
    """

    def __init__(self, smooth, details=None):
        self._smooth = smooth
        self._details = list(details) if details is not None else []
        self._packed = None  # (buf, levels, (n1, n2, p), ids of the views handed out)
        self._host_flat = None  # (pinned flat host buffer, ids of its block views)

    # dataclass-like field access -------------------------------------------
    @property
    def smooth(self):
        return self._smooth

    @smooth.setter
    def smooth(self, value):
        self._smooth = value
        self._packed = None

    @property
    def details(self):
        return self._details

    @details.setter
    def details(self, value):
        self._details = list(value)
        self._packed = None

    def __repr__(self):
        return f"WaveletPyramid(levels={self.levels}, n1={self.n1}, n2={self.n2}, p={self.p})"

    def __eq__(self, other):  # dataclass semantics: field-wise
        if not isinstance(other, WaveletPyramid):
            return NotImplemented
        return self._smooth is other._smooth and self._details == other._details

    # properties (lifting.py:36-60) ------------------------------------------
    @property
    def levels(self):
        return len(self._details)

    @property
    def n1(self):
        return self._smooth.shape[0]

    @property
    def n2(self):
        return self._smooth.shape[1]

    @property
    def m(self):
        return self._smooth.shape[2]

    @property
    def p(self):
        return self._smooth.shape[2] * (2 ** len(self._details))

    def copy(self):
        if self._packed is not None and self._packed_intact():
            buf, levels, shape, _ = self._packed
            return _pyramid_from_packed(buf.clone(), levels, *shape)
        cp = (lambda a: a.clone()) if _is_dev(self._smooth) else (lambda a: a.copy())
        return WaveletPyramid(cp(self._smooth), [cp(d) for d in self._details])

    def total_slices(self):
        return self.m + sum(d.shape[2] for d in self._details)

    # packed-buffer bookkeeping ------------------------------------------------
    def _views(self):
        return (self._smooth,) + tuple(self._details)

    def _same_views(self, handed_out) -> bool:
        # identity (not id()) of the block objects handed out: the tuple keeps
        # them alive, so a replaced block can never alias a recycled id
        cur = self._views()
        return len(cur) == len(handed_out) and all(a is b for a, b in zip(cur, handed_out))

    def _packed_intact(self) -> bool:
        return self._packed is not None and self._same_views(self._packed[3])

    def packed(self):
        """The slice-major device buffer ``(p, n1, n2)`` if this pyramid still owns one."""
        return self._packed[0] if self._packed_intact() else None


def _pyramid_from_packed(buf: torch.Tensor, levels: int, n1: int, n2: int, p: int):
    views = {}
    for tag, off, cnt in E.block_slices(p, levels):
        views[tag] = buf[off:off + cnt].permute(1, 2, 0)
    details = [views[f"d{j}"] for j in range(1, levels + 1)]
    pyr = WaveletPyramid(views["s"], details)
    pyr._packed = (buf, levels, (n1, n2, p), pyr._views())
    return pyr


def _empty_pyramid(t, levels):
    n1, n2, p = t.shape
    if _is_dev(t):
        mk = lambda k: torch.zeros((n1, n2, k), dtype=torch.float64, device=t.device)  # noqa: E731
    else:
        mk = lambda k: np.zeros((n1, n2, k), dtype=np.float64)  # noqa: E731
    return WaveletPyramid(mk(p >> levels), [mk(p >> j) for j in range(1, levels + 1)])


def forward_w(t, levels):
    """Decompose ``t`` into a WaveletPyramid -- lifting.py:77-94.

    Requires ``levels >= 1`` and ``2**levels`` dividing the slice count;
    raises LevelError otherwise.
    """
    dev = _is_dev(t)
    if not dev:
        t = np.asarray(t, dtype=np.float64)
    p = t.shape[2]  # IndexError for ndim < 3, exactly like the reference (lifting.py:84)
    if levels < 1:
        raise LevelError(f"level count must be >= 1, got {levels}")
    if p % (2 ** levels) != 0:
        raise LevelError(f"2**{levels} does not divide slice count {p}")
    if t.ndim != 3:
        raise ShapeError(f"expected a third-order tensor, got ndim={t.ndim}")
    n1, n2 = t.shape[0], t.shape[1]
    if n1 * n2 * p == 0:
        return _empty_pyramid(t, levels)
    if dev:
        return _pyramid_from_packed(E.lift_forward(E.as_device(t), levels), levels, n1, n2, p)
    # host mode: tube-major blocks = the reference's own per-level arrays, all
    # views of one host buffer, pinned when host_buffer's pool has one to spare
    # (inverse_w re-uploads it without packing)
    if n1 * n2 * p >= _STREAM_MIN and t.flags.c_contiguous:
        host = E.hand_out(E.host_lift(t, n1, n2, p, levels, forward=True))
    else:
        host = E.to_host(E.lift_forward(E.as_device(t), levels, layout=N.LAYOUT_TUBE)).reshape(-1)
    nt = n1 * n2
    blocks = {tag: host[off * nt:(off + cnt) * nt].reshape(n1, n2, cnt)
              for tag, off, cnt in E.block_slices(p, levels)}
    pyr = WaveletPyramid(blocks["s"], [blocks[f"d{j}"] for j in range(1, levels + 1)])
    pyr._host_flat = (host, pyr._views())
    return pyr


def check_consistent(pyr):
    """Validate the slice-count chain of a pyramid; raises ShapeError (lifting.py:97-111)."""
    n1, n2, m = pyr.smooth.shape
    expect = m
    for j in range(pyr.levels, 0, -1):
        d = pyr.details[j - 1]
        if d.shape[0] != n1 or d.shape[1] != n2:
            raise ShapeError(
                f"detail level {j} has slice shape {tuple(d.shape[:2])}, expected {(n1, n2)}")
        if d.shape[2] != expect:
            raise ShapeError(f"detail level {j} has {d.shape[2]} slices, expected {expect}")
        expect *= 2


def _pack_blocks(pyr):
    """Tube-major packed buffer [d1 | ... | dL | s] on the device, plus the mode."""
    blocks = list(pyr.details) + [pyr.smooth]
    if any(_is_dev(b) for b in blocks):
        dev = next(b.device for b in blocks if _is_dev(b))
        flat = [E.as_device(b, dev).reshape(-1) for b in blocks]
        return torch.cat(flat), True
    host = np.concatenate([np.ascontiguousarray(np.asarray(b, dtype=np.float64)).ravel()
                           for b in blocks])
    return E.as_device(host), False


def inverse_w(pyr):
    """Reconstruct the spatial-domain tensor from a WaveletPyramid -- lifting.py:114-120."""
    check_consistent(pyr)
    n1, n2, levels, p = pyr.n1, pyr.n2, pyr.levels, pyr.p
    buf = pyr.packed() if isinstance(pyr, WaveletPyramid) else None
    if buf is not None:
        return E.lift_inverse(buf, n1, n2, p, levels)
    if n1 * n2 * p == 0:
        z = pyr.smooth
        if _is_dev(z):
            return torch.zeros((n1, n2, p), dtype=torch.float64, device=z.device)
        return np.zeros((n1, n2, p), dtype=np.float64)
    hf = getattr(pyr, "_host_flat", None)
    if hf is not None and pyr._same_views(hf[1]):
        if n1 * n2 * p >= _STREAM_MIN:          # streamed H2D | K2 | D2H in row chunks
            return E.hand_out(E.host_lift(torch.from_numpy(hf[0]), n1, n2, p, levels,
                                          forward=False)).reshape(n1, n2, p)
        flat, dev = E.as_device(hf[0]), False   # blocks are still views of the pinned buffer
    else:
        flat, dev = _pack_blocks(pyr)
    y = E.lift_inverse(flat, n1, n2, p, levels, layout=N.LAYOUT_TUBE)
    return y if dev else E.to_host(y)


def constant_pyramid(block, p, levels):
    """Pyramid whose every smooth and detail slice equals ``block`` (lifting.py:123-136)."""
    if levels < 1:
        raise LevelError(f"level count must be >= 1, got {levels}")
    if p % (2 ** levels) != 0:
        raise LevelError(f"2**{levels} does not divide slice count {p}")
    if _is_dev(block):
        b = block.to(torch.float64)
        rep = lambda k: b[:, :, None].expand(b.shape[0], b.shape[1], k).contiguous()  # noqa: E731
    else:
        b = np.asarray(block, dtype=np.float64)
        rep = lambda k: np.broadcast_to(b[:, :, None], b.shape + (k,)).copy()  # noqa: E731
    return WaveletPyramid(rep(p >> levels), [rep(p >> j) for j in range(1, levels + 1)])


def _energy(block) -> float:
    x = E.as_device(block)
    if x.numel() == 0:
        return 0.0
    return float(E.band_sums(x.reshape(-1, 1, 1), None, 0)[0].item())


def fine_detail_energy_ratio(pyr):
    """Fraction of squared coefficient mass in detail levels below the coarsest
    (lifting.py:139-155); deterministic GPU reductions."""
    total = _energy(pyr.smooth)
    fine = 0.0
    for j, d in enumerate(pyr.details, start=1):
        e = _energy(d)
        total += e
        if j < pyr.levels:
            fine += e
    if total == 0.0:
        return 0.0
    return fine / total
