"""The w-product and its ring structure -- drop-in for ``wten.algebra``
(/root/reference/pkg/src/wten/algebra.py).

``w_product`` is one fused device pipeline: K1 on both operands (packed
slice-major pyramids), ONE strided-batched DMMA GEMM over all p wavelet slices
(every level's slices are n1 x n2 matrices, so levels need no separate
launches), and K2 on the product.  No host round trip between stages.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from . import engine as E
from .errors import LevelError, OrthogonalityError, ShapeError
from .lifting import WaveletPyramid, _is_dev, _pyramid_from_packed, constant_pyramid, inverse_w


def _stack_to_slices(x: torch.Tensor) -> torch.Tensor:
    """(n1, n2, k) tube-fastest -> contiguous (k, n1, n2) via K1 at level 0."""
    n1, n2, k = x.shape
    return E.lift_forward(x.contiguous(), 0)


def slicewise_matmul(a, b):
    """Frontal-slice-wise matrix product of two slice stacks (algebra.py:18-28)."""
    if a.shape[1] != b.shape[0] or a.shape[2] != b.shape[2]:
        raise ShapeError(f"cannot face-multiply shapes {tuple(a.shape)} and {tuple(b.shape)}")
    dev = _is_dev(a) or _is_dev(b)
    n1, k = a.shape[0], a.shape[2]
    n3 = b.shape[1]
    if n1 * n3 * k == 0:
        z = np.zeros((n1, n3, k))
        return torch.from_numpy(z).cuda() if dev else z
    sa = _stack_to_slices(E.as_device(a))
    sb = _stack_to_slices(E.as_device(b))
    sc = E.gemm(sa, sb)
    out = E.lift_inverse(sc, n1, n3, k, 0)  # (k, n1, n3) -> (n1, n3, k)
    return out if dev else E.to_host(out)


def face_product(a, b):
    """Blockwise matrix product of two conformable pyramids (algebra.py:31-40)."""
    if a.levels != b.levels or a.p != b.p:
        raise ShapeError(
            f"pyramids disagree: levels {a.levels} vs {b.levels}, slices {a.p} vs {b.p}")
    pa, pb = a.packed(), b.packed()
    if pa is not None and pb is not None:
        if a.n2 != b.n1:
            raise ShapeError(f"cannot face-multiply shapes {(a.n1, a.n2, a.p)} and {(b.n1, b.n2, b.p)}")
        pc = E.gemm(pa, pb)
        return _pyramid_from_packed(pc, a.levels, a.n1, b.n2, a.p)
    smooth = slicewise_matmul(a.smooth, b.smooth)
    details = [slicewise_matmul(x, y) for x, y in zip(a.details, b.details)]
    return WaveletPyramid(smooth, details)


def _check_levels(p, levels):
    if levels < 1:
        raise LevelError(f"level count must be >= 1, got {levels}")
    if p % (2 ** levels) != 0:
        raise LevelError(f"2**{levels} does not divide slice count {p}")


def _as_operand(x):
    return x if _is_dev(x) else np.asarray(x, dtype=np.float64)


def w_product_device(a: torch.Tensor, b: torch.Tensor, levels: int,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """Device core of w_product on contiguous CUDA tensors (no validation): K1, K1, K3,
    K2 in one C-ABI call (engine.w_product)."""
    return E.w_product(a, b, levels, out=out)


def w_product(a, b, levels):
    """Wavelet-domain tensor product of a (n1 x n2 x p) with b (n2 x n3 x p) (algebra.py:43-51)."""
    a = _as_operand(a)
    b = _as_operand(b)
    if a.ndim != 3 or b.ndim != 3:
        raise ShapeError("w_product operands must be third-order tensors")
    if a.shape[1] != b.shape[0] or a.shape[2] != b.shape[2]:
        raise ShapeError(f"cannot multiply shapes {tuple(a.shape)} and {tuple(b.shape)}")
    _check_levels(a.shape[2], levels)
    dev = _is_dev(a) or _is_dev(b)
    n1, n2, p = a.shape
    n3 = b.shape[1]
    if n1 * n3 * p == 0:
        z = np.zeros((n1, n3, p))
        return torch.from_numpy(z).cuda() if dev else z
    if n2 == 0:
        z = np.zeros((n1, n3, p))
        return torch.from_numpy(z).cuda() if dev else z
    c = w_product_device(E.as_device(a), E.as_device(b), levels)
    return c if dev else E.to_host(c)


def identity_tensor(n, p, levels):
    """Spatial tensor whose every wavelet block is I_n (algebra.py:54-59)."""
    return inverse_w(constant_pyramid(np.eye(n), p, levels))


def inverse_tensor(a, levels):
    """Blockwise inverse: every wavelet-domain slice is matrix-inverted (algebra.py:62-91).

    Singularity follows the reference's np.linalg.inv (LAPACK dgetrf): a slice is
    singular when Gaussian elimination with partial pivoting meets an exactly
    zero pivot (wt_lu_pivot_check_f64), or when its inverse is not finite;
    finite ill-conditioned slices are inverted, as numpy does.  The inverse
    itself is V diag(1/s) U^T from K4.  Raises SingularSliceError(level,
    slice_index, cond) -- smooth block first (level 0), then details 1..L, like
    the reference's loop; ``cond`` is s_max / s_min (np.linalg.cond).
    """
    from .errors import SingularSliceError

    a = _as_operand(a)
    if a.shape[0] != a.shape[1]:
        raise ShapeError(f"inverse needs square frontal slices, got {tuple(a.shape[:2])}")
    _check_levels(a.shape[2], levels)
    dev = _is_dev(a)
    x = E.as_device(a)
    n, _, p = x.shape
    pyr = E.lift_forward(x, levels)
    singular = E.lu_zero_pivot(pyr) != 0
    sigma, vec, info = E.svd(pyr, n)
    bad = singular | ~torch.isfinite(sigma).all(dim=1)
    inv = E.pinv_blocks(pyr, sigma, vec, 0.0)
    bad |= ~torch.isfinite(inv.reshape(p, -1)).all(dim=1)
    if bool(bad.any()):
        bad_h = bad.cpu().numpy()
        s_h = sigma.cpu().numpy()
        for tag, off, cnt in [E.block_slices(p, levels)[-1]] + E.block_slices(p, levels)[:-1]:
            for k in range(cnt):
                if bad_h[off + k]:
                    lo, hi = s_h[off + k, -1], s_h[off + k, 0]
                    cond = float(hi / lo) if lo > 0 and np.isfinite(hi / lo) else float("inf")
                    level = 0 if tag == "s" else int(tag[1:])
                    raise SingularSliceError(level, k, cond)
    y = E.lift_inverse(inv, n, n, p, levels)
    return y if dev else E.to_host(y)


def orthogonal_tensor(q, p, levels, tol=1e-12):
    """Tensor whose every wavelet block is the orthogonal matrix ``q`` (algebra.py:102-112)."""
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 2 or q.shape[0] != q.shape[1]:
        raise ShapeError(f"expected a square matrix, got shape {q.shape}")
    residual = np.abs(q.T @ q - np.eye(q.shape[0])).max()
    if residual > tol:
        raise OrthogonalityError(f"q^T q deviates from identity by {residual:.3e} (tol {tol:.1e})")
    return inverse_w(constant_pyramid(q, p, levels))
