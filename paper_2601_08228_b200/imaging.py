"""Hyperspectral application helpers around the hot path (the
reference ships no code for them, so parity is against the SPEC/PAPER formulas).

* ``psnr`` / ``ssim``: PAPER.md:876-887 verbatim (PSNR numerator MPP, not MPP^2;
  SSIM with global per-band moments, population variance), reduced on the GPU
  with the deterministic band-reduction kernel.
* ``blur`` / ``deblur``: A_V *_w X *_w A_H^T and its pseudo-inverse sandwich
  (SPEC.md:485-503).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import engine as E
from .algebra import w_product
from .decomposition import pinv_w, sp_pinv_w
from .lifting import _is_dev
from .tensor import transpose


def _moments(x: torch.Tensor, y: torch.Tensor):
    n = x.shape[0] * x.shape[1]
    mx = E.band_sums(x, None, 2) / n
    my = E.band_sums(y, None, 2) / n
    xc = (x - mx).contiguous()
    yc = (y - my).contiguous()
    vx = E.band_sums(xc, None, 0) / n
    vy = E.band_sums(yc, None, 0) / n
    cxy = E.band_sums(xc, yc, 3) / n
    return mx, my, vx, vy, cxy


def _mpp(x, y, mpp):
    if mpp is not None:
        return float(mpp)
    return max(float(x.max().item()), float(y.max().item()))


def psnr(x1, x2, mpp=None) -> float:
    """10 log10(n1 n2 p MPP / ||x1 - x2||_F^2); +inf for identical inputs."""
    x = E.as_device(x1)
    y = E.as_device(x2)
    m = _mpp(x, y, mpp)
    err = float(E.band_sums(x, y, 1).sum().item())
    if err == 0.0:
        return float("inf")
    return 10.0 * math.log10(x.numel() * m / err)


def ssim(x1, x2, mpp=None) -> float:
    """Band-averaged global SSIM, c1 = (0.01 MPP)^2, c2 = (0.03 MPP)^2."""
    x = E.as_device(x1)
    y = E.as_device(x2)
    m = _mpp(x, y, mpp)
    c1, c2 = (0.01 * m) ** 2, (0.03 * m) ** 2
    mx, my, vx, vy, cxy = _moments(x, y)
    per_band = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    return float(per_band.mean().item())


def blur_vectors(b_v: int, b_h: int, n1: int, n2: int):
    """c_v(i) = (b_v - i) / (3 b_v) for i < b_v, else 0."""
    i1 = np.arange(n1, dtype=np.float64)
    i2 = np.arange(n2, dtype=np.float64)
    cv = np.where(i1 < b_v, (b_v - i1) / (3.0 * b_v), 0.0)
    ch = np.where(i2 < b_h, (b_h - i2) / (3.0 * b_h), 0.0)
    return cv, ch


def blur_operator(b_v: int, b_h: int, n1: int, n2: int, p: int, device=None):
    """Slice-constant Toeplitz operators A_V (n1 x n1 x p), A_H (n2 x n2 x p).

    With ``device`` (e.g. ``"cuda"``) the operators are written straight into HBM by
    ``wt_toeplitz_tensor_f64`` (bit-identical to the host construction; nothing but the
    two coefficient vectors crosses PCIe) and returned as CUDA tensors."""
    cv, ch = blur_vectors(b_v, b_h, n1, n2)
    if device is not None:
        return (E.toeplitz_tensor(E.as_device(cv, device), n1, p),
                E.toeplitz_tensor(E.as_device(ch, device), n2, p))
    av = cv[np.abs(np.subtract.outer(np.arange(n1), np.arange(n1)))]
    ah = ch[np.abs(np.subtract.outer(np.arange(n2), np.arange(n2)))]
    return (np.ascontiguousarray(np.broadcast_to(av[:, :, None], av.shape + (p,))),
            np.ascontiguousarray(np.broadcast_to(ah[:, :, None], ah.shape + (p,))))


def toeplitz_operator(c, n: int, p: int, device="cuda"):
    """(n, n, p) slice-constant operator with every slice A[i, j] = c[|i - j|] (0 beyond
    len(c)), built on the GPU: the 9 x 9 Gaussian-PSF operators of BASELINE configs[4]
    are ``toeplitz_operator(synth.gaussian_taps(9, 2.0)[4:], n, p)``."""
    return E.toeplitz_tensor(E.as_device(np.ascontiguousarray(c, dtype=np.float64), device), n, p)


def blur(x, a_v, a_h, levels):
    """A_V *_w X *_w A_H^T."""
    return w_product(w_product(a_v, x, levels), transpose(a_h), levels)


def deblur(b, a_v, a_h, levels, method="w", tol=1e-12):
    """A_V^+ * B * (A_H^T)^+ (SPEC.md:495-503): method "w" (pinv_w), "spw" (sp_pinv_w)
    under the w-product, or "t" (t_pinv under the t-product, the paper's comparator)."""
    if method not in ("w", "spw", "t"):
        raise ValueError(f"unknown deblur method {method!r}")
    if method == "t":
        from .baselines import t_pinv, t_product

        left = t_pinv(a_v, tol)
        right = t_pinv(transpose(a_h), tol)
        return t_product(t_product(left, b), right)
    if method == "w" and _is_dev(a_v) == _is_dev(a_h) and tuple(a_v.shape) == tuple(a_h.shape):
        # both operators' wavelet slices in one batched K4 call (independent per slice)
        from .decomposition import _check_levels, pinv_w_device_many

        dev = _is_dev(b) or _is_dev(a_v) or _is_dev(a_h)
        av = E.as_device(a_v)
        aht = E.as_device(transpose(a_h))
        _check_levels(av.shape[2], levels)
        left, right = pinv_w_device_many([av, aht], levels, tol)
        out = w_product(w_product(left, E.as_device(b), levels), right, levels)
        return out if dev else E.to_host(out)
    inv = pinv_w if method == "w" else sp_pinv_w
    left = inv(a_v, levels, tol)
    right = inv(transpose(a_h), levels, tol)
    return w_product(w_product(left, b, levels), right, levels)


def to_host(x):
    return x.cpu().numpy() if _is_dev(x) else np.asarray(x)
