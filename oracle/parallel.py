"""Multi-threaded CPU port of the reference hot path (TEST / BENCH INFRASTRUCTURE ONLY).

The same algorithms as ``wten_oracle.py`` (numpy + LAPACK ``dgesdd`` / BLAS
``dgemm``, the arithmetic the reference calls), spread over all host threads
the way a CPU user would run them, so that ``bench.py`` can time the reference
path on the box's own cores:

* the lifting transform is row-separable (every tube is independent,
  ``lifting.py:63-74``): forward / inverse run on row blocks in a thread pool
  (numpy releases the GIL inside its strided ufunc loops);
* the facewise SVDs / GEMMs are independent per wavelet slice
  (``decomposition.py:64-67``, ``algebra.py:18-28``): slices are spread over the
  pool, each worker calling LAPACK / BLAS single-threaded (one
  ``np.linalg.svd`` over 8 slices of 512^2 with 8 OpenBLAS threads is only
  1.1x faster than with one: dgesdd does not scale inside one call).

Only ``tests/``, ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs
and ``__graft_entry__.smoke()`` may import this; the product never does.
Results are identical to ``wten_oracle.py`` (same per-slice calls; the
transform is exact arithmetic), checked in ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import wten_oracle as O


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


class Pool:
    """Thread pool with BLAS limited to one thread per worker while it runs."""

    def __init__(self, threads: int | None = None):
        self.threads = threads or host_threads()
        self._ex = ThreadPoolExecutor(max_workers=self.threads)
        self._lim = None

    def __enter__(self):
        try:
            import threadpoolctl

            np.linalg.svd(np.ones((2, 2)))  # load OpenBLAS so threadpoolctl sees it
            self._lim = threadpoolctl.threadpool_limits(1)
        except Exception:  # noqa: BLE001 -- without threadpoolctl BLAS keeps its threads
            self._lim = None
        return self

    def __exit__(self, *exc):
        if self._lim is not None:
            self._lim.unregister() if hasattr(self._lim, "unregister") else self._lim.restore_original_limits()
        self._ex.shutdown()
        return False

    def map(self, fn, items):
        return list(self._ex.map(fn, items))


def _row_blocks(n1: int, parts: int):
    edges = np.linspace(0, n1, min(parts, max(n1, 1)) + 1).astype(int)
    return [slice(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def lift_forward(pool: Pool, t, levels: int):
    """``lifting.py:77-94`` on row blocks (bit-identical to the serial oracle)."""
    t = np.asarray(t, dtype=np.float64)
    n1, n2, p = t.shape
    m = p >> levels
    smooth = np.empty((n1, n2, m))
    details = [np.empty((n1, n2, p >> j)) for j in range(1, levels + 1)]

    def one(sl):
        s, d = O.lift_forward(t[sl], levels)
        smooth[sl] = s
        for dst, src in zip(details, d):
            dst[sl] = src

    pool.map(one, _row_blocks(n1, 2 * pool.threads))
    return smooth, details


def lift_inverse(pool: Pool, smooth, details):
    """``lifting.py:114-120`` on row blocks."""
    n1, n2, m = smooth.shape
    p = m << len(details)
    out = np.empty((n1, n2, p))

    def one(sl):
        out[sl] = O.lift_inverse(smooth[sl], [d[sl] for d in details])

    pool.map(one, _row_blocks(n1, 2 * pool.threads))
    return out


def _per_slice(pool: Pool, stack, fn, out_shape):
    """fn(k x n1 x n2 slice-major chunk) -> k x a x b, over slice chunks of the stack."""
    k = stack.shape[2]
    lhs = np.moveaxis(stack, 2, 0)
    out = np.empty((k,) + tuple(out_shape))
    edges = np.linspace(0, k, min(k, pool.threads) + 1).astype(int)

    def one(i):
        a, b = int(edges[i]), int(edges[i + 1])
        if b > a:
            out[a:b] = fn(np.ascontiguousarray(lhs[a:b]))

    pool.map(one, range(len(edges) - 1))
    return np.ascontiguousarray(np.moveaxis(out, 0, 2))


def truncated_stack(pool: Pool, stack, r: int):
    """``_stack_svd`` + ``_truncated_blocks`` (decomposition.py:64-72) per slice chunk."""
    n1, n2, _ = stack.shape

    def fn(ch):
        u, s, vh = np.linalg.svd(ch, full_matrices=False)
        return u[:, :, :r] @ (s[:, :r, None] * vh[:, :r, :])

    return _per_slice(pool, stack, fn, (n1, n2))


def pinv_stack(pool: Pool, stack, tol: float):
    """``_pinv_stack`` (decomposition.py:157-163) per slice chunk."""
    n1, n2, _ = stack.shape

    def fn(ch):
        u, s, vh = np.linalg.svd(ch, full_matrices=False)
        cut = tol * s.max(axis=1, keepdims=True)
        inv = np.zeros_like(s)
        np.divide(1.0, s, out=inv, where=(s > cut) & (s > 0))
        return np.swapaxes(vh, 1, 2) @ (inv[:, :, None] * np.swapaxes(u, 1, 2))

    return _per_slice(pool, stack, fn, (n2, n1))


def face_matmul(pool: Pool, a, b):
    """``slicewise_matmul`` (algebra.py:18-28) per slice chunk."""
    k = a.shape[2]
    rhs = np.moveaxis(b, 2, 0)
    edges = np.linspace(0, k, min(k, pool.threads) + 1).astype(int)
    lhs = np.moveaxis(a, 2, 0)
    out = np.empty((k, a.shape[0], b.shape[1]))

    def one(i):
        x, y = int(edges[i]), int(edges[i + 1])
        if y > x:
            out[x:y] = lhs[x:y] @ rhs[x:y]

    pool.map(one, range(len(edges) - 1))
    return np.ascontiguousarray(np.moveaxis(out, 0, 2))


def sp_w_svd(pool: Pool, a, r: int, levels: int):
    """``sp_w_svd`` (decomposition.py:140-154)."""
    a = np.asarray(a, dtype=np.float64)
    O.check_rank(r, a.shape[0], a.shape[1])
    smooth, details = lift_forward(pool, a, levels)
    s_rec = truncated_stack(pool, smooth, r)
    d_rec = truncated_stack(pool, details[-1], r)
    dets = [np.zeros_like(d) for d in details[:-1]] + [d_rec]
    return lift_inverse(pool, s_rec, dets)


def _chunks(pool: Pool, stack, fn):
    """[fn(slice-major chunk) for each of pool.threads slice chunks of an (n1, n2, k) stack]."""
    k = stack.shape[2]
    lhs = np.moveaxis(stack, 2, 0)
    edges = np.linspace(0, k, min(k, pool.threads) + 1).astype(int)
    spans = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]
    return pool.map(lambda ab: fn(np.ascontiguousarray(lhs[ab[0]:ab[1]])), spans)


def w_svd(pool: Pool, a, r: int, levels: int):
    """``w_svd`` (decomposition.py:85-120): sigma table, factor blocks U, S, V
    (decomposition.py:75-82) and the rank-r reconstruction, four inverse transforms."""
    a = np.asarray(a, dtype=np.float64)
    O.check_rank(r, a.shape[0], a.shape[1])
    smooth, details = lift_forward(pool, a, levels)
    table, parts = [], {"U": [], "S": [], "V": [], "R": []}
    for tag, st in [(f"d{j}", d) for j, d in enumerate(details, start=1)] + [("s", smooth)]:
        res = _chunks(pool, st, lambda ch: np.linalg.svd(ch, full_matrices=False))
        u = np.concatenate([x[0] for x in res])
        s = np.concatenate([x[1] for x in res])
        vh = np.concatenate([x[2] for x in res])
        table.append((tag, s))
        parts["R"].append(O.truncated(u, s, vh, r))
        ub, sb, vb = O.factor_blocks(u, s, vh, r)
        parts["U"].append(ub)
        parts["S"].append(sb)
        parts["V"].append(vb)

    def back(lst):
        return lift_inverse(pool, lst[-1], lst[:-1])

    return dict(U=back(parts["U"]), S=back(parts["S"]), V=back(parts["V"]),
                sigma_table=table, recon=back(parts["R"]))


def pinv_w(pool: Pool, a, levels: int, tol: float = 1e-12):
    """``pinv_w`` (decomposition.py:166-177)."""
    a = np.asarray(a, dtype=np.float64)
    smooth, details = lift_forward(pool, a, levels)
    return lift_inverse(pool, pinv_stack(pool, smooth, tol), [pinv_stack(pool, d, tol) for d in details])


def w_product(pool: Pool, a, b, levels: int):
    """``w_product`` (algebra.py:43-51)."""
    sa, da = lift_forward(pool, np.asarray(a, dtype=np.float64), levels)
    sb, db = lift_forward(pool, np.asarray(b, dtype=np.float64), levels)
    return lift_inverse(pool, face_matmul(pool, sa, sb), [face_matmul(pool, x, y) for x, y in zip(da, db)])


def deblur(pool: Pool, b, av, ah_t, levels: int, tol: float):
    """Config-5 recovery: w_product(w_product(pinv_w(A_V), B), pinv_w(A_H^T))."""
    left = pinv_w(pool, av, levels, tol)
    right = pinv_w(pool, ah_t, levels, tol)
    return w_product(pool, w_product(pool, left, b, levels), right, levels)
