"""NPY v1.0 / PGM file helpers.  Host-side IO: CPU tests,
plus one GPU test of the pinned device load."""

import os

import numpy as np
import pytest
import torch

import paper_2601_08228_b200 as W
from paper_2601_08228_b200.errors import FormatError, IoError, ShapeError
from wt_paper_examples import EX2_A


def test_roundtrip_is_bitwise_and_numpy_compatible(tmp_path):
    x = np.random.default_rng(0).standard_normal((4, 4, 4)) * 1e-300
    p = tmp_path / "x.npy"
    W.save_tensor(x, p)
    y = W.load_tensor(p)
    assert y.dtype == np.float64 and y.flags.c_contiguous and y.shape == (4, 4, 4)
    assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    assert np.array_equal(np.load(p), x)                       # numpy reads ours
    np.save(tmp_path / "n.npy", x)
    assert np.array_equal(W.load_tensor(tmp_path / "n.npy"), x)  # we read numpy's
    assert os.path.getsize(p) % 64 == (4 * 4 * 4 * 8) % 64


def test_example2_tensor_and_f32_widening(tmp_path):
    a = np.asarray(EX2_A, dtype=np.float64)
    p = tmp_path / "a.npy"
    W.save_tensor(a, p)
    assert np.array_equal(W.load_tensor(p), a)
    np.save(tmp_path / "f.npy", a.astype("<f4"))
    got = W.load_tensor(tmp_path / "f.npy")
    assert got.dtype == np.float64 and np.array_equal(got, a.astype(np.float32).astype(np.float64))


def test_format_errors_carry_offsets(tmp_path):
    x = np.ones((2, 3, 4))
    np.save(tmp_path / "fo.npy", np.asfortranarray(x))
    with pytest.raises(FormatError, match="fortran_order"):
        W.load_tensor(tmp_path / "fo.npy")
    np.save(tmp_path / "t.npy", x)
    raw = (tmp_path / "t.npy").read_bytes()
    (tmp_path / "cut.npy").write_bytes(raw[:-8])
    with pytest.raises(FormatError, match=r"truncated payload at offset \d+ \(184 of 192 bytes\)"):
        W.load_tensor(tmp_path / "cut.npy")
    (tmp_path / "bad.npy").write_bytes(b"NOTNPY" + raw[6:])
    with pytest.raises(FormatError, match="bad magic at offset 0"):
        W.load_tensor(tmp_path / "bad.npy")
    np.save(tmp_path / "2d.npy", np.ones((3, 4)))
    with pytest.raises(FormatError, match="shape"):
        W.load_tensor(tmp_path / "2d.npy")
    np.save(tmp_path / "i8.npy", np.ones((2, 2, 2), dtype=np.int64))
    with pytest.raises(FormatError, match="dtype"):
        W.load_tensor(tmp_path / "i8.npy")
    assert issubclass(FormatError, ValueError)


def test_io_and_shape_errors(tmp_path):
    with pytest.raises(IoError):
        W.load_tensor(tmp_path / "missing.npy")
    with pytest.raises(IoError):
        W.save_tensor(np.ones((2, 2, 2)), tmp_path / "no_dir" / "x.npy")
    with pytest.raises(ShapeError):
        W.save_tensor(np.ones((2, 0, 2)), tmp_path / "e.npy")
    assert not (tmp_path / "e.npy").exists()
    with pytest.raises(ShapeError):
        W.save_tensor(np.ones((2, 2)), tmp_path / "e.npy")
    assert issubclass(IoError, OSError)


def _pgm(path):
    raw = path.read_bytes()
    head, _, rest = raw.partition(b"\n255\n")
    w, h = (int(v) for v in head.split(b"\n")[1].split())
    return np.frombuffer(rest, dtype=np.uint8).reshape(h, w)


def test_preview(tmp_path):
    a = np.asarray(EX2_A, dtype=np.float64)                    # 2 x 3 x 4
    W.save_preview(a, tmp_path / "m.pgm", "mean")
    img = _pgm(tmp_path / "m.pgm")
    mean = a.mean(axis=2)
    want = np.rint((mean - mean.min()) * 255.0 / (mean.max() - mean.min()))
    assert img.shape == (2, 3) and np.array_equal(img, want.astype(np.uint8))
    assert img.min() == 0 and img.max() == 255
    assert (tmp_path / "m.pgm").read_bytes().startswith(b"P5\n3 2\n255\n")
    W.save_preview(np.full((3, 5, 2), 7.0), tmp_path / "c.pgm", 1)
    assert np.all(_pgm(tmp_path / "c.pgm") == 128)
    with pytest.raises(IndexError):
        W.save_preview(a, tmp_path / "k.pgm", 4)
    W.save_preview(a, tmp_path / "k0.pgm", 0)
    W.save_preview(a.copy(), tmp_path / "k0b.pgm", 0)          # deterministic bytes
    assert (tmp_path / "k0.pgm").read_bytes() == (tmp_path / "k0b.pgm").read_bytes()


@pytest.mark.gpu
def test_pinned_device_load(tmp_path):
    x = np.random.default_rng(5).standard_normal((16, 8, 32))
    W.save_tensor(torch.from_numpy(x).cuda(), tmp_path / "d.npy")
    t = W.load_tensor(tmp_path / "d.npy", device="cuda")
    assert t.is_cuda and t.dtype == torch.float64 and torch.equal(t.cpu(), torch.from_numpy(x))
    pyr = W.forward_w(t, 3)                                     # straight into the GPU path
    assert torch.equal(W.inverse_w(pyr).cpu(), torch.from_numpy(x)) or \
        float((W.inverse_w(pyr).cpu() - torch.from_numpy(x)).abs().max()) < 1e-12
