"""Tensor files and previews: NPY v1.0 ('<f8', C order) load / save and 8-bit
PGM (P5) band previews -- the `cli-io` operations of SPEC.md:566-600, which the
reference package describes but does not ship.

B200 note: ``load_tensor(path, device="cuda")`` reads the payload straight into
pinned host memory and returns a CUDA tensor (one H2D copy, no staging copy);
``save_tensor`` and ``save_preview`` accept CUDA tensors (one D2H copy).
Errors: malformed files raise ``FormatError`` with the byte offset of the
problem; OS-level failures raise ``IoError``; tensors that are not third-order
or have an empty axis raise ``ShapeError`` before anything is written.
"""

from __future__ import annotations

import ast

import numpy as np

from .errors import FormatError, IoError, ShapeError

MAGIC = b"\x93NUMPY"
_ALIGN = 64  # header + preamble padded to a multiple of 64 bytes (NPY v1.0 allows any multiple of 16)


def _as_host3(t) -> np.ndarray:
    if hasattr(t, "is_cuda") and hasattr(t, "cpu"):
        t = t.detach().cpu().numpy()
    a = np.ascontiguousarray(t, dtype=np.float64)
    if a.ndim != 3:
        raise ShapeError(f"expected a third-order tensor, got ndim={a.ndim}")
    if min(a.shape) < 1:
        raise ShapeError(f"tensor axes must be positive, got shape {a.shape}")
    return a


def _parse_header(raw: bytes, path) -> tuple[str, tuple]:
    try:
        hdr = ast.literal_eval(raw.decode("latin1"))
    except (ValueError, SyntaxError) as e:
        raise FormatError(f"{path}: unparsable header dictionary at offset 10 ({e})") from None
    if not isinstance(hdr, dict) or not {"descr", "fortran_order", "shape"} <= set(hdr):
        raise FormatError(f"{path}: header at offset 10 lacks descr / fortran_order / shape")
    descr, fortran, shape = hdr["descr"], hdr["fortran_order"], hdr["shape"]
    if descr not in ("<f8", "<f4"):
        raise FormatError(f"{path}: dtype {descr!r} at offset 10 is unsupported (need '<f8' or '<f4')")
    if fortran:
        raise FormatError(f"{path}: fortran_order=True at offset 10 is unsupported (C order only)")
    if (not isinstance(shape, tuple) or len(shape) != 3
            or not all(isinstance(n, int) and n >= 1 for n in shape)):
        raise FormatError(f"{path}: shape {shape!r} at offset 10 is not a positive (n1, n2, p) triple")
    return descr, shape


def load_tensor(path, device=None):
    """Read an NPY v1.0 file as a float64 (n1, n2, p) array ('<f4' is widened);
    ``device="cuda"`` returns a CUDA tensor instead."""
    try:
        with open(path, "rb") as f:
            pre = f.read(10)
            if len(pre) < 10 or pre[:6] != MAGIC:
                raise FormatError(f"{path}: bad magic at offset 0 (expected \\x93NUMPY + version + "
                                  f"header length, got {pre[:10]!r})")
            if (pre[6], pre[7]) != (1, 0):
                raise FormatError(f"{path}: NPY version {pre[6]}.{pre[7]} at offset 6 is unsupported (1.0 only)")
            hlen = int.from_bytes(pre[8:10], "little")
            raw = f.read(hlen)
            if len(raw) < hlen:
                raise FormatError(f"{path}: header truncated at offset {10 + len(raw)} "
                                  f"({len(raw)} of {hlen} bytes)")
            descr, shape = _parse_header(raw, path)
            item = 8 if descr == "<f8" else 4
            nbytes = item * shape[0] * shape[1] * shape[2]
            start = 10 + hlen
            if device is not None:
                import torch

                host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                got = f.readinto(memoryview(host.numpy()))
            else:
                host = bytearray(nbytes)
                got = f.readinto(host)
            if got < nbytes:
                raise FormatError(f"{path}: truncated payload at offset {start + got} "
                                  f"({got} of {nbytes} bytes)")
    except OSError as e:
        raise IoError(f"{path}: {e.strerror or e}") from e
    if device is not None:
        import torch

        t = host.view(torch.float64 if item == 8 else torch.float32).view(shape)
        return t.to(device, non_blocking=False).to(torch.float64)
    return np.frombuffer(host, dtype=descr).reshape(shape).astype(np.float64)


def save_tensor(t, path) -> None:
    """Write ``t`` as NPY v1.0, '<f8', C order; load_tensor(path) returns it bitwise."""
    a = _as_host3(t)
    body = "{'descr': '<f8', 'fortran_order': False, 'shape': (%d, %d, %d), }" % a.shape
    pad = (-(10 + len(body) + 1)) % _ALIGN
    header = (body + " " * pad + "\n").encode("latin1")
    try:
        with open(path, "wb") as f:
            f.write(MAGIC + bytes([1, 0]) + len(header).to_bytes(2, "little") + header)
            f.write(a.astype("<f8", copy=False).tobytes(order="C"))
    except OSError as e:
        raise IoError(f"{path}: {e.strerror or e}") from e


def save_preview(t, path, band="mean") -> None:
    """8-bit binary PGM (P5) of one band (``band`` = k) or the band mean (``"mean"``),
    min-max normalised to 0..255 (round half to even); a constant image maps to 128."""
    a = _as_host3(t)
    if isinstance(band, str):
        if band != "mean":
            raise ValueError(f"band selector must be 'mean' or an index, got {band!r}")
        img = a.mean(axis=2)
    else:
        k = int(band)
        if not 0 <= k < a.shape[2]:
            raise IndexError(f"band {k} out of range for {a.shape[2]} bands")
        img = a[:, :, k]
    lo, hi = float(img.min()), float(img.max())
    if hi > lo:
        pix = np.rint((img - lo) * (255.0 / (hi - lo))).astype(np.uint8)
    else:
        pix = np.full(img.shape, 128, dtype=np.uint8)
    try:
        with open(path, "wb") as f:
            f.write(b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0]))
            f.write(np.ascontiguousarray(pix).tobytes())
    except OSError as e:
        raise IoError(f"{path}: {e.strerror or e}") from e


__all__ = ["load_tensor", "save_tensor", "save_preview"]
