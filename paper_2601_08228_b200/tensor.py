"""Dense third-order tensor primitives -- drop-in for ``wten.tensor``
(/root/reference/pkg/src/wten/tensor.py).

A tensor is a float64 ``(n1, n2, p)`` array with the tube axis fastest; on the
device it is a contiguous CUDA tensor of the same shape.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine as E
from .errors import ShapeError
from .lifting import _is_dev


def as_tensor3(data, check_finite=True):
    """Coerce ``data`` to a float64, C-contiguous (n1, n2, p) array (tensor.py:17-30)."""
    if _is_dev(data):
        t = data.to(torch.float64).contiguous()
        finite = lambda: bool(torch.isfinite(t).all())  # noqa: E731
    else:
        t = np.ascontiguousarray(data, dtype=np.float64)
        finite = lambda: bool(np.isfinite(t).all())  # noqa: E731
    if t.ndim != 3:
        raise ShapeError(f"expected a third-order tensor, got ndim={t.ndim}")
    if min(t.shape) < 1:
        raise ShapeError(f"tensor axes must be positive, got shape {tuple(t.shape)}")
    if check_finite and not finite():
        raise ValueError("tensor contains non-finite entries")
    return t


def frontal_slice(t, k):
    """The k-th frontal slice ``t[:, :, k]`` as a writable view (tensor.py:33-42)."""
    p = t.shape[2]
    if not 0 <= k < p:
        raise IndexError(f"slice index {k} out of range for p={p}")
    return t[:, :, k]


def set_frontal_slice(t, k, m):
    """Overwrite the k-th frontal slice of ``t`` with matrix ``m`` (tensor.py:45-47)."""
    frontal_slice(t, k)[...] = m


def transpose(t):
    """Slicewise transpose: result[i, j, k] = t[j, i, k] (tensor.py:50-52).

    Device path: one pass of whole-tube copies (wt_tube_transpose_f64).
    """
    dev = _is_dev(t)
    x = E.as_device(t)
    n1, n2, p = x.shape
    if n1 * n2 * p == 0:
        z = torch.zeros((n2, n1, p), dtype=torch.float64, device=x.device)
        return z if dev else z.cpu().numpy()
    y = E.tube_transpose(x)                   # (n2, n1, p)
    return y if dev else E.to_host(y)


def trace(t):
    """Sum of the diagonals of every frontal slice (tensor.py:55-62)."""
    if t.shape[0] != t.shape[1]:
        raise ShapeError(f"trace needs square frontal slices, got {tuple(t.shape[:2])}")
    x = E.as_device(t)
    n, _, p = x.shape
    if n * p == 0:
        return 0.0
    diag = x.reshape(n * n, p)[:: n + 1].contiguous()      # (n, p) diagonal tubes
    return float(E.band_sums(diag.reshape(-1, 1, 1), None, 2)[0].item())


def frobenius_norm(t):
    """Square root of the sum of squared entries (tensor.py:65-67)."""
    x = E.as_device(t)
    if x.numel() == 0:
        return 0.0
    return math.sqrt(float(E.band_sums(x.reshape(-1, 1, 1), None, 0)[0].item()))


def matrix_svd(m):
    """Thin SVD of a matrix: (U, sigma, V) with m = U diag(sigma) V^T (tensor.py:70-77)."""
    dev = _is_dev(m)
    a = E.as_device(m)
    if a.ndim != 2:
        raise ShapeError(f"expected a matrix, got ndim={a.ndim}")
    n1, n2 = a.shape
    q = min(n1, n2)
    sigma, vec, info = E.svd(a[None], q)
    E.raise_if_failed(info)
    s = sigma[0]
    long_vecs = vec[0].t().contiguous()                       # (len, q)
    if n1 <= n2:   # long side = right vectors; U = A V / s
        other = E.gemm(a[None], vec, trans_b=True)[0]          # (n1, q)
    else:
        other = E.gemm(a[None], vec, trans_a=True, trans_b=True)[0]  # (n2, q)
    other = E.scale_cols(other[None].contiguous(), sigma, 1)
    # orthonormal columns to rounding for every rank, zero matrix included (LAPACK's
    # U and V are): the short side re-orthonormalised in sigma order, the long side's
    # numerically null columns (s_j <= 1e-12 s_max) completed
    other = E.orthonormal_fixup(other, sigma, 1.0)[0]
    long_vecs = E.orthonormal_fixup(long_vecs[None], sigma, 1e-12)[0]
    u, v = (other, long_vecs) if n1 <= n2 else (long_vecs, other)
    if dev:
        return u, s, v
    return u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()
