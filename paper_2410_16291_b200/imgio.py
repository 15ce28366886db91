"""File front door: binary PGM (P5) and raw + JSON sidecar rasters.

Drop-in for the readers and writers of pkg/src/satsweep/imgio.py (read_pgm
:72-103, write_pgm :106-116, read_sidecar :142-157, read_raw :160-174,
read_raw_result :177-187, write_raw :127-139): same names, formats, result
kinds and error messages (ImageFormatError carries the same byte_offset).

Additive: every reader takes ``device=``.  With a CUDA device the payload is
streamed from the file straight into a device tensor by the native
``ssb_file_to_device`` (pinned double-buffered staging, parallel reads,
big-endian 16-bit samples swapped on the device), so a multi-Gpx raster never
becomes a Python bytes object or a numpy array.  Writers
accept device-resident grids and results and stream them out through
``ssb_device_to_file``.  Headers are tiny and parsed here, over a memory map
of the file, exactly as the reference parses them.
"""

from __future__ import annotations

import json
import mmap
import os
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np

from . import _device, _lib
from .errors import GridValidationError, ImageFormatError, UnsupportedFormatError
from .grid import ElemKind, ImageGrid, ResultGrid, _is_torch

_WS = b" \t\n\r\v\f"

RAW_DTYPES = {
    "u8": np.dtype("u1"),
    "u16": np.dtype("<u2"),
    "f32": np.dtype("<f4"),
    "u64": np.dtype("<u8"),
    "f64": np.dtype("<f8"),
}


@dataclass(frozen=True)
class RawSidecar:
    """Geometry of a raw file (imgio.py:31-39); the byte length must equal rows*cols*width."""

    rows: int
    cols: int
    dtype: str
    endianness: str = "little"


# ----------------------------------------------------------------------------- PGM header
class _Bytes:
    """Read-only byte view of a file (memory-mapped; empty files map to b"")."""

    def __init__(self, path):
        self._f = open(path, "rb")
        size = os.fstat(self._f.fileno()).st_size
        self.buf = mmap.mmap(self._f.fileno(), 0, access=mmap.ACCESS_READ) if size else b""
        self.size = size

    def close(self):
        if isinstance(self.buf, mmap.mmap):
            self.buf.close()
        self._f.close()


def _token(buf, size: int, pos: int) -> tuple[bytes, int]:
    """Next header token after whitespace and '#'-to-newline comments (imgio.py:45-61)."""
    while pos < size:
        c = buf[pos:pos + 1]
        if c in _WS:
            pos += 1
        elif c == b"#":
            while pos < size and buf[pos:pos + 1] != b"\n":
                pos += 1
        else:
            break
    if pos >= size:
        raise ImageFormatError("unexpected end of PGM header", byte_offset=pos)
    start = pos
    while pos < size:
        c = buf[pos:pos + 1]
        if c in _WS or c == b"#":
            break
        pos += 1
    return bytes(buf[start:pos]), pos


def _number(buf, size: int, pos: int, what: str) -> tuple[int, int]:
    tok, end = _token(buf, size, pos)
    if not tok.isdigit():
        raise ImageFormatError(f"invalid PGM {what} {tok!r}", byte_offset=end - len(tok))
    return int(tok), end


@dataclass(frozen=True)
class PgmHeader:
    rows: int
    cols: int
    maxval: int
    payload_offset: int
    file_bytes: int

    @property
    def kind(self) -> ElemKind:
        return ElemKind.U8 if self.maxval <= 255 else ElemKind.U16

    @property
    def payload_bytes(self) -> int:
        return self.rows * self.cols * (1 if self.maxval <= 255 else 2)


def read_pgm_header(path) -> PgmHeader:
    """Validate a P5 header and the payload length (imgio.py:78-99) without reading the payload."""
    f = _Bytes(path)
    try:
        buf, size = f.buf, f.size
        magic, pos = _token(buf, size, 0)
        if magic != b"P5":
            raise ImageFormatError(f"not a binary PGM file (magic {magic!r})", byte_offset=0)
        cols, pos = _number(buf, size, pos, "width")
        rows, pos = _number(buf, size, pos, "height")
        maxval, pos = _number(buf, size, pos, "maxval")
        if rows < 1 or cols < 1:
            raise ImageFormatError(f"invalid PGM dimensions {cols}x{rows}", byte_offset=pos)
        if maxval < 1 or maxval > 65535:
            raise ImageFormatError(f"PGM maxval {maxval} outside 1..65535", byte_offset=pos)
        if pos >= size or buf[pos:pos + 1] not in _WS:
            raise ImageFormatError("missing single whitespace byte after maxval", byte_offset=pos)
        pos += 1
        hdr = PgmHeader(rows, cols, maxval, pos, size)
        found = max(0, min(size - pos, hdr.payload_bytes))
        if found < hdr.payload_bytes:
            raise ImageFormatError(
                f"truncated PGM payload: expected {hdr.payload_bytes} bytes, found {found}", byte_offset=size)
        return hdr
    finally:
        f.close()


# ----------------------------------------------------------------------------- device transfer
def _to_device(path, offset: int, shape, kind_dtype: np.dtype, device, swap16: bool):
    t = _device.torch()
    dev = t.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {device!r}")
    nbytes = int(np.prod(shape)) * kind_dtype.itemsize
    out = _device.empty(shape, kind_dtype, dev, f"a {shape[0]}x{shape[1]} raster")
    with t.cuda.device(dev):
        rc = _lib.load().ssb_file_to_device(os.fsencode(str(path)), offset, nbytes, int(out.data_ptr()),
                                            1 if swap16 else 0, _device.stream_ptr(dev))
    _lib.check(rc, "file read")
    return out


def _check_finite_device(x) -> None:
    flag = _device.torch().zeros(1, dtype=_device.torch().int32, device=x.device)
    rc = _lib.load().ssb_f32_nonfinite(int(x.data_ptr()), x.numel(), int(flag.data_ptr()), _device.stream_ptr(x.device))
    _lib.check(rc, "finiteness check")
    if int(flag.item()) != 0:
        raise GridValidationError("F32 grid contains NaN or Inf; only finite values are admitted")


def _host_or_tensor(obj):
    values = obj.values
    return values, _is_torch(values)


def _write_payload(path, offset: int, values, swap16: bool) -> None:
    x = values.contiguous()
    with _device.torch().cuda.device(x.device):
        rc = _lib.load().ssb_device_to_file(os.fsencode(str(path)), offset, int(x.data_ptr()),
                                            x.numel() * x.element_size(), 1 if swap16 else 0,
                                            _device.stream_ptr(x.device))
    _lib.check(rc, "file write")


# ----------------------------------------------------------------------------- PGM
def read_pgm(path, device=None) -> ImageGrid:
    """Decode a binary PGM: maxval <= 255 -> U8, 256..65535 -> U16 (big-endian samples).

    ``device``: None returns a host grid like the reference; a CUDA device
    streams the payload into a device grid."""
    hdr = read_pgm_header(path)
    shape = (hdr.rows, hdr.cols)
    kind = hdr.kind
    if device is None:
        src = np.dtype("u1") if kind is ElemKind.U8 else np.dtype(">u2")
        raw = np.fromfile(path, dtype=src, count=hdr.rows * hdr.cols, offset=hdr.payload_offset)
        return ImageGrid(np.ascontiguousarray(raw.reshape(shape), dtype=kind.dtype))
    x = _to_device(path, hdr.payload_offset, shape, kind.dtype, device, swap16=kind is ElemKind.U16)
    return ImageGrid(x, kind)


def write_pgm(img: ImageGrid, path) -> None:
    """Encode a U8/U16 grid as binary PGM (imgio.py:106-116); F32 has no lossless PGM form."""
    if img.elem_kind is ElemKind.F32:
        raise UnsupportedFormatError("PGM cannot represent F32 grids losslessly; use raw")
    if img.elem_kind is ElemKind.I32:
        raise UnsupportedFormatError("PGM cannot represent I32 grids; use raw")
    header = f"P5\n{img.cols} {img.rows}\n{int(img.elem_kind.max_value)}\n".encode("ascii")
    values, on_dev = _host_or_tensor(img)
    if not on_dev:
        payload = values.tobytes() if img.elem_kind is ElemKind.U8 else values.astype(">u2").tobytes()
        Path(path).write_bytes(header + payload)
        return
    Path(path).write_bytes(header)
    _write_payload(path, len(header), values, swap16=img.elem_kind is ElemKind.U16)


# ----------------------------------------------------------------------------- raw + sidecar
def read_sidecar(sidecar_path) -> RawSidecar:
    """Parse and validate a sidecar (imgio.py:142-157)."""
    try:
        doc = json.loads(Path(sidecar_path).read_text(encoding="utf-8"))
    except json.JSONDecodeError as exc:
        raise ImageFormatError(f"sidecar is not valid JSON: {exc}") from None
    keys = {"rows", "cols", "dtype", "endianness"}
    if not isinstance(doc, dict) or set(doc) != keys:
        raise ImageFormatError(f"sidecar must contain exactly the keys {sorted(keys)}")
    side = RawSidecar(**doc)
    if side.endianness != "little":
        raise ImageFormatError(f"unsupported endianness {side.endianness!r}; raw files are little-endian")
    if side.dtype not in RAW_DTYPES:
        raise ImageFormatError(f"unknown raw dtype {side.dtype!r}")
    if side.rows < 1 or side.cols < 1:
        raise ImageFormatError(f"invalid raw dimensions {side.rows}x{side.cols}")
    return side


def _raw_len(raw_path) -> int:
    return os.stat(raw_path).st_size


def read_raw(raw_path, sidecar_path, device=None) -> ImageGrid:
    """Read an image raster (u8/u16/f32); u64/f64 result rasters are refused (imgio.py:160-174)."""
    side = read_sidecar(sidecar_path)
    if side.dtype not in ("u8", "u16", "f32"):
        raise ImageFormatError(f"raw dtype {side.dtype!r} is a result raster, not an image input")
    dt = RAW_DTYPES[side.dtype]
    n = _raw_len(raw_path)
    expected = side.rows * side.cols * dt.itemsize
    if n != expected:
        raise ImageFormatError(
            f"raw length {n} does not match sidecar {side.rows}x{side.cols} {side.dtype} ({expected} bytes)")
    kind = ElemKind(side.dtype)
    shape = (side.rows, side.cols)
    if device is None:
        raw = np.fromfile(raw_path, dtype=dt, count=side.rows * side.cols)
        return ImageGrid(np.ascontiguousarray(raw.reshape(shape), dtype=kind.dtype))
    x = _to_device(raw_path, 0, shape, kind.dtype, device, swap16=False)
    if kind is ElemKind.F32:
        _check_finite_device(x)
    return ImageGrid(x, kind)


def read_raw_result(raw_path, sidecar_path, device=None):
    """Read back a u64/f64 result raster written by write_raw (imgio.py:177-187)."""
    side = read_sidecar(sidecar_path)
    if side.dtype not in ("u64", "f64"):
        raise ImageFormatError(f"raw dtype {side.dtype!r} is not a result raster")
    dt = RAW_DTYPES[side.dtype]
    n = _raw_len(raw_path)
    expected = side.rows * side.cols * dt.itemsize
    if n != expected:
        raise ImageFormatError(f"raw length {n} does not match sidecar ({expected} bytes)")
    shape = (side.rows, side.cols)
    if device is None:
        return np.fromfile(raw_path, dtype=dt, count=side.rows * side.cols).reshape(shape).copy()
    return _to_device(raw_path, 0, shape, np.dtype(np.uint64 if side.dtype == "u64" else np.float64), device, False)


def write_raw(obj, raw_path, sidecar_path) -> None:
    """Packed little-endian samples plus the JSON sidecar (imgio.py:127-139).

    Result grids carry "u64" (exact integer sums) or "f64".  ``obj`` may be an
    ImageGrid, a ResultGrid, or a result array/tensor; device data is streamed
    out without a host copy of the whole raster."""
    if isinstance(obj, ImageGrid):
        token, values = obj.elem_kind.value, obj.values
        if token == "i32":
            raise UnsupportedFormatError("raw files carry u8/u16/f32 images; I32 grids have no raw token")
    else:
        values = obj.values if isinstance(obj, ResultGrid) else obj
        if _is_torch(values):
            import torch

            token = "f64" if values.dtype == torch.float64 else "u64"
        else:
            token = "u64" if values.dtype == np.uint64 else "f64"
    rows, cols = int(values.shape[0]), int(values.shape[1])
    if _is_torch(values) and values.is_cuda:
        Path(raw_path).write_bytes(b"")
        _write_payload(raw_path, 0, values, swap16=False)
    else:
        arr = values.numpy() if _is_torch(values) else values
        Path(raw_path).write_bytes(np.ascontiguousarray(arr, dtype=RAW_DTYPES[token]).tobytes())
    side = RawSidecar(rows=rows, cols=cols, dtype=token)
    Path(sidecar_path).write_text(json.dumps(asdict(side)) + "\n", encoding="utf-8")


# ----------------------------------------------------------------------------- synthetic grids
def generate(kind: str, rows: int, cols: int, elem_kind: ElemKind, *, seed: int = 0, value: float = 1,
             tile: int = 1) -> ImageGrid:
    """Deterministic synthetic grid (imgio.py:193-235): "random" (PCG64; integers
    uniform over the kind's full range, F32 uniform in [0, 1)), "constant" or
    "checkerboard" (0/1 cells of tile x tile pixels).  Same bytes as the
    reference for the same arguments."""
    if rows < 1 or cols < 1:
        raise GridValidationError(f"grid dims must be >= 1, got {rows}x{cols}")
    dt = elem_kind.dtype
    if kind == "random":
        gen = np.random.Generator(np.random.PCG64(seed))
        if elem_kind.is_integer:
            hi = int(elem_kind.max_value) + 1 if elem_kind is not ElemKind.I32 else 2**31
            vals = gen.integers(0, hi, size=(rows, cols), dtype=dt)
        else:
            vals = gen.random(size=(rows, cols), dtype=np.float32)
    elif kind == "constant":
        if elem_kind.is_integer:
            if not float(value).is_integer() or not 0 <= value <= elem_kind.max_value:
                raise GridValidationError(f"constant {value!r} outside the {elem_kind.value} range")
            vals = np.full((rows, cols), int(value), dtype=dt)
        else:
            vals = np.full((rows, cols), np.float32(value), dtype=dt)
    elif kind == "checkerboard":
        if tile < 1:
            raise GridValidationError(f"checkerboard tile must be >= 1, got {tile}")
        cell = np.arange(rows)[:, None] // tile + np.arange(cols)[None, :] // tile
        vals = (cell % 2).astype(dt)
    else:
        raise GridValidationError(f"unknown generator kind {kind!r}; expected random, constant, or checkerboard")
    return ImageGrid(vals)


__all__ = [
    "PgmHeader",
    "generate",
    "RAW_DTYPES",
    "RawSidecar",
    "read_pgm",
    "read_pgm_header",
    "read_raw",
    "read_raw_result",
    "read_sidecar",
    "write_pgm",
    "write_raw",
]
