"""paper_2601_08228_b200 -- B200-native (sm_100a) hot path of the w-product framework
(arXiv 2601.08228), a drop-in for the reference package ``wten``'s
``forward_w`` / ``inverse_w`` / ``w_product`` / ``w_svd`` / ``sp_w_svd`` / ``pinv_w``.

The compute runs in ``libwten_b200.so`` (hand-written CUDA for sm_100a, C ABI in
``include/wten_b200.h``).  There is no CPU fallback: on a host without the
library or a CUDA device, compute calls raise ``NativeUnavailable``.
"""

from . import baselines
from ._native import NativeError, NativeUnavailable
from .algebra import (
    face_product,
    identity_tensor,
    inverse_tensor,
    orthogonal_tensor,
    slicewise_matmul,
    w_product,
)
from .decomposition import (
    SvdFactors,
    TruncationBound,
    pinv_w,
    pinv_w_via_factors,
    sp_pinv_w,
    sp_w_svd,
    sp_w_svd_many,
    truncation_bound,
    w_svd,
)
from .engine import is_pinned_array, pinned_empty
from .errors import (
    FormatError,
    IoError,
    LevelError,
    OrthogonalityError,
    RankError,
    ShapeError,
    SingularSliceError,
)
from .lifting import (
    WaveletPyramid,
    check_consistent,
    constant_pyramid,
    fine_detail_energy_ratio,
    forward_w,
    inverse_w,
    max_levels,
)
from .tensor_io import load_tensor, save_preview, save_tensor
from .tensor import as_tensor3, frobenius_norm, frontal_slice, matrix_svd, set_frontal_slice, trace, transpose

__version__ = "0.1.0"

__all__ = [
    "baselines",
    "NativeError", "NativeUnavailable",
    "face_product", "identity_tensor", "inverse_tensor", "orthogonal_tensor", "slicewise_matmul", "w_product",
    "SvdFactors", "TruncationBound", "pinv_w", "pinv_w_via_factors", "sp_pinv_w", "sp_w_svd", "sp_w_svd_many",
    "truncation_bound", "w_svd",
    "FormatError", "IoError", "LevelError", "OrthogonalityError", "RankError", "ShapeError",
    "SingularSliceError",
    "WaveletPyramid", "check_consistent", "constant_pyramid", "fine_detail_energy_ratio",
    "forward_w", "inverse_w", "max_levels",
    "as_tensor3", "frobenius_norm", "frontal_slice", "matrix_svd", "set_frontal_slice", "trace",
    "transpose",
    "load_tensor", "save_preview", "save_tensor",
    "is_pinned_array", "pinned_empty",
]
