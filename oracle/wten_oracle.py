"""CPU oracle (TEST INFRASTRUCTURE ONLY) for the wten hot path.

A numpy restatement of the reference algorithms; each function cites the
reference file:line it follows (paths relative to
``/root/reference/pkg/src/wten/``). Tensors are float64 ``(n1, n2, p)`` arrays
with the tube (mode-3) axis fastest, as in the reference (``tensor.py:1-5``).

Pinned by ``tests/test_oracle_golden.py`` against the paper's worked examples
and against fixtures produced by the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# lifting (lifting.py)
# ----------------------------------------------------------------------------


def max_levels(p: int) -> int:
    """Largest L with 2**L | p -- lifting.py:17-21."""
    if p < 1:
        raise ValueError(f"slice count must be positive, got {p}")
    low_bit = p & -p
    return low_bit.bit_length() - 1


def lift_step(s: np.ndarray):
    """One forward lifting level -- lifting.py:63-66.

    Pairs (x[2k], x[2k+1]) along the last axis: detail d = x[2k] - x[2k+1],
    next smooth = x[2k+1] + d / 2 (0-based even index is the paper's "odd").
    """
    n1, n2, ell = s.shape
    pairs = s.reshape(n1, n2, ell // 2, 2)
    d = pairs[..., 0] - pairs[..., 1]
    return pairs[..., 1] + d / 2, d


def unlift_step(s: np.ndarray, d: np.ndarray) -> np.ndarray:
    """One inverse lifting level -- lifting.py:69-74.

    x[2k+1] = s - d / 2, then x[2k] = d + x[2k+1].
    """
    n1, n2, half = d.shape
    out = np.empty((n1, n2, half, 2), dtype=np.float64)
    out[..., 1] = s - d / 2
    out[..., 0] = d + out[..., 1]
    return out.reshape(n1, n2, 2 * half)


def lift_forward(t, levels: int):
    """Forward multilevel transform -- lifting.py:77-94.

    Returns ``(smooth, details)`` with ``details[j-1]`` the level-j stack
    (p / 2**j slices) and ``smooth`` the level-L smooth stack.
    """
    s = np.asarray(t, dtype=np.float64)
    p = s.shape[2]
    if levels < 1 or p % (2 ** levels):
        raise ValueError(f"invalid level count {levels} for p={p}")
    details = []
    for _ in range(levels):
        s, d = lift_step(s)
        details.append(np.ascontiguousarray(d))
    return np.ascontiguousarray(s), details


def lift_inverse(smooth, details) -> np.ndarray:
    """Inverse multilevel transform -- lifting.py:114-120 (coarsest first)."""
    s = np.asarray(smooth, dtype=np.float64)
    for d in details[::-1]:
        s = unlift_step(s, np.asarray(d, dtype=np.float64))
    return np.ascontiguousarray(s)


def fine_detail_energy_ratio(smooth, details) -> float:
    """Energy share of detail levels 1..L-1 -- lifting.py:139-155."""
    total = float(np.sum(smooth ** 2))
    fine = 0.0
    for j, d in enumerate(details, start=1):
        e = float(np.sum(d ** 2))
        total += e
        if j < len(details):
            fine += e
    return 0.0 if total == 0.0 else fine / total


def packed_slices(smooth, details) -> np.ndarray:
    """Pyramid -> slice-major packed buffer ``[d1 | d2 | ... | dL | sL]``.

    This is the product's HBM layout: p matrices of n1 x n2,
    row-major. Used by tests to check the device buffer slice by slice.
    """
    blocks = [np.moveaxis(d, 2, 0) for d in details] + [np.moveaxis(smooth, 2, 0)]
    return np.ascontiguousarray(np.concatenate(blocks, axis=0))


# ----------------------------------------------------------------------------
# w-algebra (algebra.py)
# ----------------------------------------------------------------------------


def face_matmul(a, b) -> np.ndarray:
    """Slice-by-slice matrix product of two (., ., k) stacks -- algebra.py:18-28."""
    lhs = np.moveaxis(a, 2, 0)
    rhs = np.moveaxis(b, 2, 0)
    return np.ascontiguousarray(np.moveaxis(lhs @ rhs, 0, 2))


def w_product(a, b, levels: int) -> np.ndarray:
    """w-product -- algebra.py:43-51 (face_product algebra.py:31-40)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    sa, da = lift_forward(a, levels)
    sb, db = lift_forward(b, levels)
    return lift_inverse(face_matmul(sa, sb), [face_matmul(x, y) for x, y in zip(da, db)])


def transpose(t) -> np.ndarray:
    """Slicewise transpose -- tensor.py:50-52."""
    return np.ascontiguousarray(np.swapaxes(np.asarray(t), 0, 1))


def frobenius_norm(t) -> float:
    """tensor.py:65-67."""
    return float(np.linalg.norm(np.asarray(t).ravel()))


def inverse_tensor(a, levels):
    """Blockwise inverse (algebra.py:62-91); raises ValueError naming
    (level, slice) of the first singular slice, smooth block (level 0) first."""
    a = np.asarray(a, dtype=np.float64)
    smooth, details = lift_forward(a, levels)

    def inv_stack(st, tag):
        out = np.empty_like(st)
        for k in range(st.shape[2]):
            try:
                m = np.linalg.inv(st[:, :, k])
            except np.linalg.LinAlgError:
                raise ValueError((tag, k)) from None
            if not np.isfinite(m).all():
                raise ValueError((tag, k))
            out[:, :, k] = m
        return out

    s_inv = inv_stack(smooth, 0)
    d_inv = [inv_stack(d, j) for j, d in enumerate(details, start=1)]
    return lift_inverse(s_inv, d_inv)


# ----------------------------------------------------------------------------
# decomposition (decomposition.py)
# ----------------------------------------------------------------------------


def stack_svd(stack):
    """Thin SVD of every slice of an (n1, n2, k) stack -- decomposition.py:64-67."""
    return np.linalg.svd(np.moveaxis(stack, 2, 0), full_matrices=False)


def truncated(u, s, vh, r) -> np.ndarray:
    """Rank-r reconstruction of each slice -- decomposition.py:70-72."""
    rec = u[:, :, :r] @ (s[:, :r, None] * vh[:, :r, :])
    return np.ascontiguousarray(np.moveaxis(rec, 0, 2))


def factor_blocks(u, s, vh, r):
    """U (n1,r,k), diag S (r,r,k), V (n2,r,k) -- decomposition.py:75-82."""
    k = s.shape[0]
    ub = np.ascontiguousarray(np.moveaxis(u[:, :, :r], 0, 2))
    vb = np.ascontiguousarray(np.moveaxis(np.swapaxes(vh[:, :r, :], 1, 2), 0, 2))
    sb = np.zeros((r, r, k))
    for i in range(r):
        sb[i, i, :] = s[:, i]
    return ub, sb, vb


def check_rank(r, n1, n2):
    """decomposition.py:59-61."""
    if not 1 <= r <= min(n1, n2):
        raise ValueError(f"rank {r} outside [1, {min(n1, n2)}]")


def w_svd(a, r, levels):
    """decomposition.py:85-120. Returns dict(U, S, V, sigma_table, recon)."""
    a = np.asarray(a, dtype=np.float64)
    check_rank(r, a.shape[0], a.shape[1])
    smooth, details = lift_forward(a, levels)
    stacks = [(f"d{j}", d) for j, d in enumerate(details, start=1)] + [("s", smooth)]
    table, parts = [], {"U": [], "S": [], "V": [], "R": []}
    for tag, st in stacks:
        u, s, vh = stack_svd(st)
        table.append((tag, s))
        parts["R"].append(truncated(u, s, vh, r))
        ub, sb, vb = factor_blocks(u, s, vh, r)
        parts["U"].append(ub)
        parts["S"].append(sb)
        parts["V"].append(vb)

    def back(lst):
        return lift_inverse(lst[-1], lst[:-1])

    return dict(U=back(parts["U"]), S=back(parts["S"]), V=back(parts["V"]),
                sigma_table=table, recon=back(parts["R"]))


def sp_w_svd(a, r, levels):
    """decomposition.py:140-154: truncate s_L and d_L, zero d_1..d_{L-1}."""
    a = np.asarray(a, dtype=np.float64)
    check_rank(r, a.shape[0], a.shape[1])
    smooth, details = lift_forward(a, levels)
    s_rec = truncated(*stack_svd(smooth), r)
    d_rec = truncated(*stack_svd(details[-1]), r)
    dets = [np.zeros_like(d) for d in details[:-1]] + [d_rec]
    return lift_inverse(s_rec, dets)


def pinv_stack(stack, tol):
    """Per-slice pseudo-inverse, cutoff tol*sigma_max -- decomposition.py:157-163."""
    u, s, vh = stack_svd(stack)
    cut = tol * s.max(axis=1, keepdims=True)
    keep = s > cut
    inv = np.zeros_like(s)
    np.divide(1.0, s, out=inv, where=keep & (s > 0))
    pinv = np.swapaxes(vh, 1, 2) @ (inv[:, :, None] * np.swapaxes(u, 1, 2))
    return np.ascontiguousarray(np.moveaxis(pinv, 0, 2))


def pinv_w(a, levels, tol=1e-12):
    """decomposition.py:166-177."""
    a = np.asarray(a, dtype=np.float64)
    smooth, details = lift_forward(a, levels)
    return lift_inverse(pinv_stack(smooth, tol), [pinv_stack(d, tol) for d in details])


def sp_pinv_w(a, levels, tol=1e-12):
    """decomposition.py:180-203 (without the warning): invert s_L, d_L only."""
    a = np.asarray(a, dtype=np.float64)
    smooth, details = lift_forward(a, levels)
    dets = [np.zeros((d.shape[1], d.shape[0], d.shape[2])) for d in details[:-1]]
    dets.append(pinv_stack(details[-1], tol))
    return lift_inverse(pinv_stack(smooth, tol), dets)


def truncation_bound(sigma_table, r) -> float:
    """decomposition.py:123-137 (bound only)."""
    acc = 0.0
    for _, sig in sigma_table:
        tail = sig[:, r:]
        acc += float(np.sum(tail * tail))
    return float(np.sqrt(acc))


# ----------------------------------------------------------------------------
# imaging metrics (SPEC only: PAPER.md:876-887) -- parity unpinned
# ----------------------------------------------------------------------------


def psnr(x1, x2, mpp=None) -> float:
    """PAPER.md:878 verbatim: 10 log10(n1 n2 p MPP / ||x1-x2||_F^2) (MPP not squared)."""
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    if mpp is None:
        mpp = max(float(x1.max()), float(x2.max()))
    err = float(np.sum((x1 - x2) ** 2))
    if err == 0.0:
        return float("inf")
    return 10.0 * np.log10(x1.size * mpp / err)


def ssim(x1, x2, mpp=None) -> float:
    """PAPER.md:882-887 / SPEC.md:525-534: global per-band moments (ddof=0), band mean."""
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    if mpp is None:
        mpp = max(float(x1.max()), float(x2.max()))
    c1 = (0.01 * mpp) ** 2
    c2 = (0.03 * mpp) ** 2
    vals = []
    for k in range(x1.shape[2]):
        a = x1[:, :, k]
        b = x2[:, :, k]
        ma, mb = a.mean(), b.mean()
        va = ((a - ma) ** 2).mean()
        vb = ((b - mb) ** 2).mean()
        cab = ((a - ma) * (b - mb)).mean()
        vals.append(((2 * ma * mb + c1) * (2 * cab + c2))
                    / ((ma * ma + mb * mb + c1) * (va + vb + c2)))
    return float(np.mean(vals))


# ----------------------------------------------------------------------------
# comparator products (baselines.py) -- restated with numpy's FFT / LAPACK
# ----------------------------------------------------------------------------


def dct_matrix(p: int) -> np.ndarray:
    """Orthonormal DCT-II matrix, the default m-product transform (baselines.py:53-56).

    Closed form M[k, n] = f_k cos(pi k (2n + 1) / (2p)), f_0 = sqrt(1/p), else sqrt(2/p)."""
    k = np.arange(p)[:, None]
    n = np.arange(p)[None, :]
    m = np.cos(np.pi * k * (2 * n + 1) / (2 * p)) * np.sqrt(2.0 / p)
    m[0] *= np.sqrt(0.5)
    return m


def _mode3_dft(a):
    """Frequency-major DFT stack (p, n1, n2) -- baselines.py:68-69."""
    return np.ascontiguousarray(np.fft.fft(a, axis=2).transpose(2, 0, 1))


def _mode3_idft_real(fc):
    """Real part of the inverse DFT of a (p, n1, n2) stack -- baselines.py:71-72."""
    return np.ascontiguousarray(np.fft.ifft(np.ascontiguousarray(fc.transpose(1, 2, 0)), axis=2).real)


def t_product(a, b):
    """baselines.py:63-73: FFT along mode 3, facewise complex product, real inverse."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return _mode3_idft_real(np.matmul(_mode3_dft(a), _mode3_dft(b)))


def t_product_circulant(a, b):
    """Brute-force block-circulant t-product: C_k = sum_j A_j B_(k-j mod p)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    p = a.shape[2]
    c = np.zeros((a.shape[0], b.shape[1], p))
    for k in range(p):
        for j in range(p):
            c[:, :, k] += a[:, :, j] @ b[:, :, (k - j) % p]
    return c


def tube_identity(n, p):
    """baselines.py:77-82."""
    out = np.zeros((n, n, p))
    out[:, :, 0] = np.eye(n)
    return out


def apply_mode3(t, m):
    """hat[i, j, k'] = sum_k m[k', k] t[i, j, k] -- baselines.py:85-87."""
    return np.einsum("ijk,lk->ijl", np.asarray(t, dtype=np.float64), m)


def m_product(a, b, m, minv):
    """baselines.py:90-103: mode-3 transform, facewise product, inverse transform."""
    ha = apply_mode3(a, m)
    hb = apply_mode3(b, m)
    return apply_mode3(face_matmul(ha, hb), minv)


def m_identity(n, p, minv):
    """baselines.py:106-109."""
    return apply_mode3(np.broadcast_to(np.eye(n)[:, :, None], (n, n, p)), minv)


def t_svd(a, r):
    """baselines.py:112-124: rank-r truncation of every DFT-domain slice."""
    a = np.asarray(a, dtype=np.float64)
    u, s, vh = np.linalg.svd(_mode3_dft(a), full_matrices=False)
    return _mode3_idft_real(np.matmul(u[:, :, :r], s[:, :r, None] * vh[:, :r, :]))


def t_pinv(a, tol=1e-12):
    """baselines.py:127-138: per-DFT-slice Moore-Penrose inverse, cutoff tol * sigma_max."""
    a = np.asarray(a, dtype=np.float64)
    u, s, vh = np.linalg.svd(_mode3_dft(a), full_matrices=False)
    cutoff = tol * s.max(axis=1, keepdims=True)
    keep = s > cutoff
    sinv = np.zeros_like(s)
    sinv[keep] = 1.0 / s[keep]
    fp = np.matmul(np.conj(vh).transpose(0, 2, 1), sinv[:, :, None] * np.conj(u).transpose(0, 2, 1))
    return _mode3_idft_real(fp)


def op_count(kind, n1, n2, n3, p) -> int:
    """baselines.py:156-190 (closed-form product operation counts)."""
    cross = n1 * n2 + n2 * n3 + n1 * n3
    base = n1 * n2 * n3 * p
    if kind == "m":
        return base + cross * p * p
    if kind == "t":
        if p & (p - 1) == 0:
            return base + cross * p * (p.bit_length() - 1)
        return base + round(cross * p * np.log2(p))
    if kind == "w":
        return base + 2 * p * cross
    raise ValueError(kind)
