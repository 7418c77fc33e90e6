"""CPU-only checks of the drop-in boundary:
  * libwten_b200.so loads and exports every function include/wten_b200.h declares
    (and the ctypes table binds exactly those);
  * the product API raises the reference's exceptions, messages and check order
    (tests/golden/errors.json, recorded from the reference) before touching the GPU;
  * without a GPU the product path fails loudly (no CPU fallback).
"""

import json
import os
import re

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200 import _native as N
from wt_helpers import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "wten_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(wt_[a-z0-9_]+)\s*\(", src))


def test_header_and_ctypes_table_agree():
    assert header_functions() == set(N.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.wt_version() >= 100


def test_workspace_query_runs_without_gpu():
    lib = N.load()
    assert lib.wt_svd_workspace_bytes(256, 256, 192) >= 192 * 256 * 256 * 8
    assert lib.wt_svd_workspace_bytes(-1, 4, 1) == 0


ERRORS = {e["call"]: e for e in json.load(open(os.path.join(GOLDEN, "errors.json")))["errors"]}

ones = np.ones
CALLS = {
    "forward_w(ones(2,2,8), 0)": lambda: W.forward_w(ones((2, 2, 8)), 0),
    "forward_w(ones(2,2,8), 4)": lambda: W.forward_w(ones((2, 2, 8)), 4),
    "forward_w(ones(2,2,8), -1)": lambda: W.forward_w(ones((2, 2, 8)), -1),
    "forward_w(ones(2,8), 1)": lambda: W.forward_w(ones((2, 8)), 1),
    "forward_w(ones(2,2,6), 2)": lambda: W.forward_w(ones((2, 2, 6)), 2),
    "w_product(ones(2,3), ones(3,2,4), 1)": lambda: W.w_product(ones((2, 3)), ones((3, 2, 4)), 1),
    "w_product(ones(2,3,4), ones(2,2,4), 1)": lambda: W.w_product(ones((2, 3, 4)), ones((2, 2, 4)), 1),
    "w_product(ones(2,3,4), ones(3,2,8), 1)": lambda: W.w_product(ones((2, 3, 4)), ones((3, 2, 8)), 1),
    "w_product(ones(2,3,4), ones(3,2,4), 3)": lambda: W.w_product(ones((2, 3, 4)), ones((3, 2, 4)), 3),
    "w_svd(ones(3,4,4), 0, 3)": lambda: W.w_svd(ones((3, 4, 4)), 0, 3),
    "w_svd(ones(3,4,4), 4, 1)": lambda: W.w_svd(ones((3, 4, 4)), 4, 1),
    "w_svd(ones(3,4,4), 2, 3)": lambda: W.w_svd(ones((3, 4, 4)), 2, 3),
    "sp_w_svd(ones(3,4,4), 5, 1)": lambda: W.sp_w_svd(ones((3, 4, 4)), 5, 1),
    "sp_w_svd(ones(3,4,4), 1, 3)": lambda: W.sp_w_svd(ones((3, 4, 4)), 1, 3),
    "pinv_w(ones(3,4,4), 3)": lambda: W.pinv_w(ones((3, 4, 4)), 3),
    "max_levels(0)": lambda: W.max_levels(0),
    "inverse_tensor(ones(2,3,4), 1)": lambda: W.inverse_tensor(ones((2, 3, 4)), 1),
}


def _pyramid(shape_smooth, dshapes):
    return W.WaveletPyramid(np.ones(shape_smooth), [np.ones(s) for s in dshapes])


CALLS["inverse_w(bad slice count)"] = lambda: W.inverse_w(_pyramid((2, 2, 2), [(2, 2, 4), (2, 2, 1)]))
CALLS["inverse_w(bad slice shape)"] = lambda: W.inverse_w(_pyramid((2, 2, 2), [(1, 2, 4), (2, 2, 2)]))
CALLS["face_product(p4 L1, p8 L1)"] = lambda: W.face_product(
    _pyramid((2, 2, 2), [(2, 2, 2)]), _pyramid((2, 2, 4), [(2, 2, 4)]))


@pytest.mark.parametrize("call", sorted(CALLS))
def test_error_convention_matches_reference(call):
    ref = ERRORS[call]
    with pytest.raises(Exception) as ei:
        CALLS[call]()
    err = ei.value
    assert type(err).__name__ == ref["type"]
    assert str(err) == ref["message"]
    # same class hierarchy names as the reference (ShapeError < ValueError, ...)
    assert [k.__name__ for k in type(err).__mro__] == ref["mro"]


def test_max_levels_values():
    for call, e in ERRORS.items():
        if call.startswith("max_levels(") and "value" in e:
            assert W.max_levels(int(call[11:-1])) == e["value"]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(N.NativeUnavailable):
        W.forward_w(np.ones((2, 2, 4)), 1)
    with pytest.raises(N.NativeUnavailable):
        W.w_product(np.ones((2, 3, 4)), np.ones((3, 2, 4)), 1)
    with pytest.raises(N.NativeUnavailable):
        W.w_svd(np.ones((3, 3, 4)), 1, 1)
