"""ctypes binding of the in-tree C-ABI library ``libwten_b200.so``.

The library is the product: there is no CPU fallback.  Importing this module
does not need a GPU (the symbols can be inspected on a CPU-only host), but every
compute entry point calls :func:`require_gpu` first and raises
:class:`NativeUnavailable` when the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WT_LIB_PATH") or os.path.join(HERE, "libwten_b200.so")  # override: A/B builds

c_double_p = ctypes.c_void_p  # device pointers travel as integers
i64 = ctypes.c_int64
u64 = ctypes.c_uint64

LAYOUT_SLICE = 0
LAYOUT_TUBE = 1
MASK_ALL = (1 << 64) - 1
SCALE_MUL, SCALE_DIV, SCALE_PINV2 = 0, 1, 2

# name -> (restype, argtypes); mirrors include/wten_b200.h one to one.
SIGNATURES = {
    "wt_version": (ctypes.c_int, []),
    "wt_last_error": (ctypes.c_char_p, []),
    "wt_lift_fwd_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, ctypes.c_int, c_double_p,
                                       ctypes.c_int, i64, u64, ctypes.c_void_p]),
    "wt_lift_inv_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, ctypes.c_int, ctypes.c_int,
                                       i64, u64, c_double_p, ctypes.c_void_p]),
    "wt_lift_fwd_f64_peer": (ctypes.c_int, [c_double_p, i64, i64, i64, ctypes.c_int, ctypes.c_void_p,
                                            i64, u64, ctypes.c_void_p]),
    "wt_lift_inv_f64_peer": (ctypes.c_int, [ctypes.c_void_p, i64, i64, i64, ctypes.c_int, i64, u64,
                                            c_double_p, ctypes.c_void_p]),
    "wt_gemm_f64":(ctypes.c_int, [ctypes.c_int, ctypes.c_int, i64, i64, i64, ctypes.c_double,
                                   c_double_p, i64, i64, c_double_p, i64, i64, ctypes.c_double,
                                   c_double_p, i64, i64, i64, ctypes.c_void_p]),
    "wt_w_product_workspace_bytes": (ctypes.c_size_t, [i64, i64, i64, i64]),
    "wt_w_product_f64": (ctypes.c_int, [c_double_p, c_double_p, i64, i64, i64, i64, ctypes.c_int, c_double_p,
                                        ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "wt_svd_workspace_bytes": (ctypes.c_size_t, [i64, i64, i64]),
    "wt_svd_jacobi_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, i64, c_double_p,
                                         c_double_p, i64, ctypes.c_void_p, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                         ctypes.c_void_p]),
    "wt_set_option": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "wt_svd_topk_workspace_bytes": (ctypes.c_size_t, [i64, i64, i64, i64]),
    "wt_svd_topk_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, i64, i64, c_double_p, c_double_p, i64,
                                       ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_void_p]),
    "wt_svd_last_sweeps": (ctypes.c_int, []),
    "wt_svd_last_fallbacks": (ctypes.c_int, []),
    "wt_svd_last_jacobi_flops": (ctypes.c_double, []),
    "wt_scale_cols_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, c_double_p, i64, i64,
                                         ctypes.c_int, ctypes.c_double, ctypes.c_void_p]),
    "wt_copy2d_f64": (ctypes.c_int, [c_double_p, i64, i64, c_double_p, i64, i64, i64, i64, i64,
                                     ctypes.c_int, ctypes.c_void_p]),
    "wt_svd_truncate_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, i64, c_double_p, i64, i64,
                                           c_double_p, i64, i64, c_double_p, ctypes.c_void_p]),
    "wt_svd_factors_f64": (ctypes.c_int, [c_double_p, c_double_p, i64, c_double_p, i64, i64, i64, i64,
                                          c_double_p, c_double_p, ctypes.c_void_p]),
    "wt_pinv_from_svd_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, i64, c_double_p, c_double_p,
                                            ctypes.c_double, c_double_p, i64, i64, c_double_p,
                                            ctypes.c_void_p]),
    "wt_pinv_from_svd_ranked_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, i64, c_double_p,
                                                   c_double_p, ctypes.c_double, c_double_p, i64, i64,
                                                   c_double_p, ctypes.c_void_p, ctypes.c_void_p]),
    "wt_tube_delta_f64": (ctypes.c_int, [c_double_p, i64, i64, c_double_p, ctypes.c_void_p]),
    "wt_tube_transpose_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, c_double_p, ctypes.c_void_p]),
    "wt_readback_i32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, i64, ctypes.c_void_p]),
    "wt_orthonormal_fixup_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, i64, c_double_p, i64, i64,
                                                ctypes.c_double, ctypes.c_void_p]),
    "wt_lu_pivot_check_f64": (ctypes.c_int, [c_double_p, i64, i64, ctypes.c_void_p, ctypes.c_void_p]),
    "wt_diag_blocks_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, c_double_p, ctypes.c_void_p]),
    "wt_toeplitz_tensor_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, c_double_p, ctypes.c_void_p]),
    "wt_gauss_smooth2d_f64": (ctypes.c_int, [c_double_p, i64, i64, i64, c_double_p, i64, c_double_p, c_double_p,
                                             ctypes.c_void_p]),
    "wt_hsi_mix_f64": (ctypes.c_int, [c_double_p, c_double_p, i64, i64, i64, ctypes.c_double, c_double_p, u64,
                                      ctypes.c_double, ctypes.c_double, c_double_p, ctypes.c_void_p]),
    "wt_slice_reduce_scratch": (ctypes.c_size_t, [i64, i64]),
    "wt_slice_reduce_f64": (ctypes.c_int, [c_double_p, c_double_p, i64, i64, ctypes.c_int,
                                           c_double_p, ctypes.c_void_p]),
}


class NativeUnavailable(RuntimeError):
    """The CUDA library or device needed by the product path is missing."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lib = None


def load(path: str = LIB_PATH):
    """Load ``libwten_b200.so`` and bind every declared symbol (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2601_08228_b200/csrc`)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_gpu_checked = False


def require_gpu():
    """Return the loaded library; raise NativeUnavailable without a CUDA device."""
    global _gpu_checked
    lib = load()
    if not _gpu_checked:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the wten_b200 product path runs only on a GPU")
        _gpu_checked = True
    return lib


def check(status: int, what: str):
    if status != 0:
        msg = _lib.wt_last_error().decode(errors="replace") if _lib is not None else ""
        raise NativeError(f"{what} failed (status {status}): {msg}")
