"""Comparator tensor products (t-product, m-product) and the analytical
operation-count model -- drop-in for ``wten.baselines``
(/root/reference/pkg/src/wten/baselines.py).

These are the products the paper ranks the w-product against, built on the
w-path kernels plus cuFFT for the t-product's DFT (an O(p log p) transform, so
the w-vs-t comparison stays fair):

* t-product: half-spectrum rfft along mode 3; the complex facewise product
  of each of the p//2 + 1 frequencies is ONE real K3 GEMM,
  [Re A | Im A] [[Re B, Im B], [-Im B, Re B]] = [Re C | Im C]; irfft returns
  the real part the reference keeps (baselines.py:71-72).
* m-product: the mode-3 transforms are ONE K3 GEMM per operand, a (p x p)
  transform matrix times the (n1 n2 x p) tube matrix, written straight into
  the slice-major (p, n1, n2) stack the facewise K3 product needs.
* t_svd / t_pinv transform the tube deltas x_k - x_0 (wt_tube_delta_f64; DC
  restored with p x_0), so a constant tube has exactly zero off-DC
  coefficients as numpy's FFT butterflies give -- the relative pinv cutoff on
  the slice-constant blur operators depends on it -- and run K4 on the real
  embedding [[Re, -Im], [Im, Re]] of each
  frequency slice: its singular values are those of the complex slice, each
  twice, and truncation to 2r (or inversion with the same tol * sigma_max
  cutoff) commutes with the embedding, so the re/im blocks of the result are
  the complex rank-r truncation (pseudo-inverse).

Only the half spectrum (p//2 + 1 frequencies) is decomposed; numpy decomposes
all p and discards the imaginary residue.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import engine as E
from .errors import RankError, ShapeError
from .lifting import _is_dev

F64 = torch.float64


# ----------------------------------------------------------- transforms ----

@dataclass
class ModeTransform:
    """Invertible transform applied along the third mode (baselines.py:20-50).

    ``kind`` is ``"matrix"`` (explicit p x p pair ``M`` / ``Minv``) or ``"dft"``.
    The consistency check M @ Minv ~ I is the reference's host-side validation
    of a small p x p input (baselines.py:32-45), not product compute.
    """

    kind: str
    M: np.ndarray = None
    Minv: np.ndarray = None

    def __post_init__(self):
        if self.kind not in ("dft", "matrix"):
            raise ValueError(f"unknown transform kind {self.kind!r}")
        if self.kind != "matrix":
            return
        if self.M is None or self.Minv is None:
            raise ValueError("matrix transform needs both M and Minv")
        p = self.M.shape[0]
        if self.M.shape != (p, p) or self.Minv.shape != (p, p):
            raise ShapeError("transform matrices must be square and same size")
        residual = float(np.max(np.abs(np.asarray(self.M) @ np.asarray(self.Minv) - np.eye(p))))
        if residual > 1e-10:
            raise ValueError(f"M @ Minv deviates from identity by {residual:.3e}")

    @property
    def p(self):
        return None if self.kind == "dft" else self.M.shape[0]


def dct_transform(p):
    """Orthonormal DCT-II transform of size p, the default m-product M (baselines.py:53-56).

    Built from the closed form f_k cos(pi k (2n+1) / 2p) (f_0 = sqrt(1/p), else
    sqrt(2/p)); its transpose is its inverse."""
    k = np.arange(p)[:, None]
    n = np.arange(p)[None, :]
    m = np.cos(np.pi * ((k * (2 * n + 1)) % (4 * p)) / (2 * p)) * math.sqrt(2.0 / p)
    m[0, :] = math.sqrt(1.0 / p)
    return ModeTransform(kind="matrix", M=m, Minv=np.ascontiguousarray(m.T))


def _spectrum(x: torch.Tensor, neg_imag: bool = False, exact_dc: bool = True) -> torch.Tensor:
    """Half-spectrum mode-3 DFT of (n1, n2, p) as a frequency-major stack
    (2h, n1, n2) = [Re; Im] (plus [-Im] rows when ``neg_imag``), h = p//2 + 1.

    With ``exact_dc`` cuFFT transforms the tube deltas x_k - x_0
    (wt_tube_delta_f64) and the DC term gets p * x_0 back, so constant tubes
    have exactly zero off-DC coefficients (np.fft.fft's butterflies give the
    same, baselines.py:68) -- the pseudo-inverse's relative cutoff needs that;
    the products do not (one memory pass less)."""
    n1, n2, p = x.shape
    if exact_dc:
        spec = torch.fft.rfft(E.tube_delta(x), dim=2)        # (n1, n2, h) complex
        spec[:, :, 0] += p * x[:, :, 0]
    else:
        spec = torch.fft.rfft(x, dim=2)
    h = spec.shape[2]
    ri = torch.view_as_real(spec).permute(3, 2, 0, 1)        # (2, h, n1, n2) view
    # a fresh tensor: standard strides even for size-1 dims (the GEMM reads stride(1))
    out = torch.empty(((3 if neg_imag else 2) * h, n1, n2), dtype=F64, device=x.device)
    out[:2 * h].view(2, h, n1, n2).copy_(ri)
    if neg_imag:
        torch.neg(out[h:2 * h], out=out[2 * h:])
    return out


def _synthesis(fc: torch.Tensor, p: int) -> torch.Tensor:
    """Real part of the inverse DFT of a Hermitian half spectrum [Re; Im] (2h, n1, n2)."""
    h = fc.shape[0] // 2
    n1, n2 = fc.shape[1], fc.shape[2]
    spec = torch.view_as_complex(fc.view(2, h, n1, n2).permute(2, 3, 1, 0).contiguous())
    return torch.fft.irfft(spec, n=p, dim=2).contiguous()


def _mode3(x: torch.Tensor, f: torch.Tensor) -> torch.Tensor:
    """hat[k', i, j] = sum_k f[k', k] x[i, j, k] as a slice-major (q, n1, n2) stack (K3)."""
    n1, n2, p = x.shape
    out = E.gemm(f[None], x.reshape(1, n1 * n2, p), trans_b=True)   # (1, q, n1 n2)
    return out.view(f.shape[0], n1, n2)


def _unmode3(c: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """out[i, j, k] = sum_k' g[k, k'] c[k', i, j] from a (q, n1, n2) stack (K3)."""
    q, n1, n2 = c.shape
    out = E.gemm(c.reshape(1, q, n1 * n2), g[None], trans_a=True, trans_b=True)  # (1, n1 n2, p)
    return out.view(n1, n2, g.shape[0])


def _prep(x):
    if _is_dev(x):
        return x.to(F64)
    return np.asarray(x, dtype=np.float64)


def _out(t: torch.Tensor, dev: bool):
    return t if dev else E.to_host(t)


def _check_product_shapes(a, b):
    """baselines.py:58-61."""
    if a.ndim != 3 or b.ndim != 3:
        raise ShapeError("product operands must be third-order tensors")
    if a.shape[1] != b.shape[0] or a.shape[2] != b.shape[2]:
        raise ShapeError(f"cannot multiply shapes {tuple(a.shape)} and {tuple(b.shape)}")


def _check_p(p):
    if p < 1:
        raise ValueError(f"Invalid number of FFT data points ({p}) specified.")


# ------------------------------------------------------------- products ----

def t_product(a, b):
    """DFT-domain facewise product (block-circulant multiplication) (baselines.py:63-73)."""
    dev = _is_dev(a) or _is_dev(b)
    a, b = _prep(a), _prep(b)
    _check_product_shapes(a, b)
    n1, n2, p = a.shape
    n3 = b.shape[1]
    _check_p(p)
    if n1 * n3 == 0:
        z = np.zeros((n1, n3, p))
        return torch.from_numpy(z).cuda() if dev else z
    da, db = E.as_device(a), E.as_device(b)
    h = p // 2 + 1
    # per frequency k: [Re A | Im A] (n1 x 2n2) times [[Re B, Im B], [-Im B, Re B]]
    # (2n2 x 2n3) = [Re C | Im C]: the complex facewise product as ONE real K3
    # GEMM (four real products, N = 2 n3 keeps the tiles full)
    sa = torch.view_as_real(torch.fft.rfft(da, dim=2))       # (n1, n2, h, 2)
    sb = torch.view_as_real(torch.fft.rfft(db, dim=2))       # (n2, n3, h, 2)
    acat = torch.empty((h, n1, 2, n2), dtype=F64, device=da.device)
    acat.copy_(sa.permute(2, 0, 3, 1))
    bemb = torch.empty((h, 2, n2, 2, n3), dtype=F64, device=da.device)
    sbp = sb.permute(2, 0, 3, 1)                             # (h, n2, 2, n3) view
    bemb[:, 0].copy_(sbp)                                    # [Re B | Im B]
    bemb[:, 1, :, 0].copy_(sbp[:, :, 1]).neg_()              # -Im B
    bemb[:, 1, :, 1].copy_(sbp[:, :, 0])                     #  Re B
    ccat = E.gemm(acat.view(h, n1, 2 * n2), bemb.view(h, 2 * n2, 2 * n3))   # (h, n1, 2 n3)
    spec = torch.view_as_complex(ccat.view(h, n1, 2, n3).permute(1, 3, 0, 2).contiguous())
    return _out(torch.fft.irfft(spec, n=p, dim=2).contiguous(), dev)


def tube_identity(n, p):
    """Identity of the t-product: first frontal slice I_n, the rest zero (baselines.py:77-82)."""
    ident = np.zeros((n, n, p))
    ident[:, :, 0] = np.eye(n)
    return ident


def m_product(a, b, transform):
    """Facewise product after an invertible matrix transform along mode 3 (baselines.py:90-103)."""
    if transform.kind != "matrix":
        raise ValueError("m_product needs a matrix-kind transform")
    dev = _is_dev(a) or _is_dev(b)
    a, b = _prep(a), _prep(b)
    _check_product_shapes(a, b)
    if a.shape[2] != transform.p:
        raise ShapeError(f"transform size {transform.p} does not match slice count {a.shape[2]}")
    n1, n2, p = a.shape
    n3 = b.shape[1]
    if n1 * n3 == 0:
        z = np.zeros((n1, n3, p))
        return torch.from_numpy(z).cuda() if dev else z
    da, db = E.as_device(a), E.as_device(b)
    m = E.as_device(transform.M)
    minv = E.as_device(transform.Minv)
    hc = E.gemm(_mode3(da, m), _mode3(db, m))                 # (p, n1, n3) facewise
    return _out(_unmode3(hc, minv), dev)


def m_identity(n, p, transform):
    """Identity tensor of the m-product: M^-1 transform of identity blocks (baselines.py:106-109)."""
    minv = E.as_device(transform.Minv)
    blocks = torch.eye(n, dtype=F64, device=minv.device).expand(p, n, n).contiguous()
    return E.to_host(_unmode3(blocks, minv))


# ------------------------------------------------------- decompositions ----

def _embedded_spectrum(x: torch.Tensor):
    """Half-spectrum real embeddings [[Re, -Im], [Im, Re]] of every DFT slice: (h, 2n1, 2n2)."""
    n1, n2, p = x.shape
    h = p // 2 + 1
    f = _spectrum(x, neg_imag=True)                           # (3h, n1, n2): Re, Im, -Im
    emb = torch.empty((h, 2 * n1, 2 * n2), dtype=F64, device=x.device)
    E.copy2d(f[:h], False, out=emb[:, :n1, :n2])
    E.copy2d(f[:h], False, out=emb[:, n1:, n2:])
    E.copy2d(f[h:2 * h], False, out=emb[:, n1:, :n2])
    E.copy2d(f[2 * h:], False, out=emb[:, :n1, n2:])
    return emb


def _unembed(blocks: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    """(h, 2 rows, 2 cols) embeddings -> (2h, rows, cols) stack [Re; Im] (left block column)."""
    h = blocks.shape[0]
    fc = torch.empty((2 * h, rows, cols), dtype=F64, device=blocks.device)
    E.copy2d(blocks[:, :rows, :cols], False, out=fc[:h])
    E.copy2d(blocks[:, rows:, :cols], False, out=fc[h:])
    return fc


def t_svd(a, r):
    """Rank-r truncation of every DFT-domain slice's SVD (baselines.py:112-124)."""
    dev = _is_dev(a)
    a = _prep(a)
    if not 1 <= r <= min(a.shape[0], a.shape[1]):
        raise RankError(f"rank {r} outside [1, {min(a.shape[0], a.shape[1])}] "
                        f"for {a.shape[0]}x{a.shape[1]} slices")
    n1, n2, p = a.shape
    _check_p(p)
    emb = _embedded_spectrum(E.as_device(a))
    sigma, vec, info = E.svd(emb, 2 * r)
    E.raise_if_failed(info)
    rec = E.truncated_recon(emb, sigma, vec, 2 * r)
    return _out(_synthesis(_unembed(rec, n1, n2), p), dev)


def t_pinv(a, tol=1e-12):
    """Moore-Penrose inverse under the t-product, per-DFT-slice cutoff tol * sigma_max
    (baselines.py:127-138); returns n2 x n1 x p."""
    dev = _is_dev(a)
    a = _prep(a)
    n1, n2, p = a.shape
    _check_p(p)
    if n1 * n2 == 0:
        z = np.zeros((n2, n1, p))
        return torch.from_numpy(z).cuda() if dev else z
    emb = _embedded_spectrum(E.as_device(a))
    sigma, vec, info = E.svd(emb, 2 * min(n1, n2))
    E.raise_if_failed(info)
    blocks = E.pinv_blocks(emb, sigma, vec, tol)              # (h, 2 n2, 2 n1)
    return _out(_synthesis(_unembed(blocks, n2, n1), p), dev)


# ------------------------------------------------------------ op counts ----

@dataclass
class OpCountReport:
    """Closed-form operation count for one product kind and shape (baselines.py:141-150)."""

    kind: str
    n1: int
    n2: int
    n3: int
    p: int
    count: int


def _pow2(p):
    return p >= 1 and (p & (p - 1)) == 0


def _log2_term(p, scale):
    """scale * log2(p): exact integer at powers of two, rounded float otherwise."""
    if _pow2(p):
        return scale * (p.bit_length() - 1)
    return scale * math.log2(p)


def op_count(kind, n1, n2, n3, p):
    """Paper section III product operation counts as exact integers (baselines.py:156-190):
    m: n1n2n3p + X p^2, t: n1n2n3p + X p log2 p, w: n1n2n3p + 2pX, X = n1n2 + n2n3 + n1n3."""
    if min(n1, n2, n3, p) < 1:
        raise ValueError("dimensions must be positive")
    cross = n1 * n2 + n2 * n3 + n1 * n3
    base = n1 * n2 * n3 * p
    if kind == "m":
        count = base + cross * p * p
    elif kind == "t":
        extra = _log2_term(p, cross * p)
        count = base + (extra if isinstance(extra, int) else round(extra))
    elif kind == "w":
        if not _pow2(p):
            raise ValueError(f"w count is defined for power-of-two p, got {p}")
        count = base + 2 * p * cross
    else:
        raise ValueError(f"unknown product kind {kind!r}")
    return OpCountReport(kind=kind, n1=n1, n2=n2, n3=n3, p=p, count=count)


def svd_op_count(kind, p):
    """Cube-model tensor-SVD counts (baselines.py:193-213): m 3p^4, t p^4 + 2p^3 log2 p,
    w p^4 + 4p^3, spw 6p^3."""
    if p < 1:
        raise ValueError("p must be positive")
    if kind == "m":
        return 3 * p ** 4
    if kind == "t":
        return round(p ** 4 + _log2_term(p, 2 * p ** 3))
    if kind == "w":
        return p ** 4 + 4 * p ** 3
    if kind == "spw":
        return 6 * p ** 3
    raise ValueError(f"unknown svd kind {kind!r}")


def deblur_op_count(kind, p):
    """Cube-model deblurring-pipeline counts (baselines.py:216-236): m 5p^4,
    t 2p^4 + 3p^3 log2 p, w 2p^4 + 6p^3, spw 10p^3."""
    if p < 1:
        raise ValueError("p must be positive")
    if kind == "m":
        return 5 * p ** 4
    if kind == "t":
        return round(2 * p ** 4 + _log2_term(p, 3 * p ** 3))
    if kind == "w":
        return 2 * p ** 4 + 6 * p ** 3
    if kind == "spw":
        return 10 * p ** 3
    raise ValueError(f"unknown deblur kind {kind!r}")
