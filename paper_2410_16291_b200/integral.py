"""Summed-area tables in HBM and O(1)-per-window queries (drop-in for
pkg/src/satsweep/integral.py).

``build_sat`` launches the reduce-then-scan table kernels
(csrc/sat_build.cu); ``swa_integral`` / ``swa_multi_window`` run the corner
sweep with fused finalisation (csrc/window_eval.cu).  Tables stay on the
device; ``IntegralImage.table`` copies one back to the host on first access.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _device, _engine, _lib
from .errors import InvalidWindowError, ResourceLimitError
from .grid import ElemKind, ImageGrid, ResultGrid, StatKind, WindowSpec, output_dims
from .stats import needs_squares

U64_MAX = 2**64 - 1


class AccumKind(enum.Enum):
    """Accumulator of a table (integral.py:28-41)."""

    U64 = "u64"    # exact unsigned 64-bit
    U128 = "u128"  # exact beyond 64 bits (host view reconstructed from the modular device table)
    F64 = "f64"

    @property
    def dtype(self):
        if self is AccumKind.U64:
            return np.dtype(np.uint64)
        if self is AccumKind.F64:
            return np.dtype(np.float64)
        return np.dtype(object)


def select_accum(elem_kind: ElemKind, rows: int, cols: int, squared: bool) -> AccumKind:
    """Narrowest accumulator that provably cannot overflow (integral.py:44-55).

    The device always stores integer tables modulo 2^64; window sums stay
    exact whenever they fit 64 bits, and the U128 host view is rebuilt exactly
    (see IntegralImage.table)."""
    if not elem_kind.is_integer:
        return AccumKind.F64
    peak = int(elem_kind.max_value) ** (2 if squared else 1) * rows * cols
    limit = U64_MAX if elem_kind is not ElemKind.I32 else 2**63 - 1
    return AccumKind.U64 if peak <= limit else AccumKind.U128


@dataclass(frozen=True, eq=False)
class IntegralImage:
    """Zero-padded (rows+1) x (cols+1) table resident on the device.

    ``device_table`` is a (rows+1) x pitch tensor (int64 storage for integer
    tables, float64 for F32); ``table`` is the reference-shaped host array.
    """

    device_table: object
    accum_kind: AccumKind
    source_dims: tuple[int, int]
    squared: bool = False
    elem_kind: ElemKind = ElemKind.U8
    pitch: int = 0
    _host: dict = field(default_factory=dict, repr=False)

    @property
    def rows(self) -> int:
        return self.source_dims[0]

    @property
    def cols(self) -> int:
        return self.source_dims[1]

    @property
    def table(self) -> np.ndarray:
        if "t" not in self._host:
            dev = self.device_table[:, : self.cols + 1]
            if self.accum_kind is AccumKind.F64:
                host = _device.to_host(dev, np.float64)
            else:
                host = _device.to_host(dev, np.uint64)
                if self.elem_kind is ElemKind.I32:
                    host = host.view(np.int64)
                if self.accum_kind is AccumKind.U128:
                    host = _unwrap_rows(host)
            host.flags.writeable = False
            self._host["t"] = host
        return self._host["t"]


def _unwrap_rows(mod: np.ndarray) -> np.ndarray:
    """Exact values of a non-negative table stored modulo 2^64.

    Along a row the increment t[i][j] - t[i][j-1] is a column-prefix sum of
    i pixels (< 2^64 at any in-core size), so a wrap happened exactly where the
    stored value decreases; counting wraps gives the high word."""
    hi = np.zeros(mod.shape, dtype=np.int64)
    np.cumsum(mod[:, 1:] < mod[:, :-1], axis=1, out=hi[:, 1:])
    return hi.astype(object) * (1 << 64) + mod.astype(object)


def allocate_table(elem_kind: ElemKind, rows: int, cols: int, squared: bool, device=None):
    """Device table of the reference shape; ResourceLimitError names the bytes (integral.py:76-83)."""
    kind = select_accum(elem_kind, rows, cols, squared)
    required = (rows + 1) * (cols + 1) * 8
    what = f"a {rows + 1}x{cols + 1} integral table"
    try:
        device = device or _device.current_device()
    except Exception:
        raise ResourceLimitError(required, what) from None
    dt = np.float64 if kind is AccumKind.F64 else np.uint64
    return _device.empty((rows + 1, _engine.sat_ld_for(cols)), dt, device, what), kind


@_engine.device_scoped
def _build(img: ImageGrid, squared: bool) -> IntegralImage:
    if img.elem_kind is ElemKind.I32 and squared:
        raise TypeError("squared tables are not supported for int32 input")
    kind = select_accum(img.elem_kind, img.rows, img.cols, squared)
    x, dev = _engine.device_input(img)
    flag = _engine.new_flag(dev) if img.elem_kind is ElemKind.F32 else None
    sat, sq, ld = _engine.build_tables(x, img.elem_kind, img.rows, img.cols, dev, squared=squared,
                                       plain=not squared, flag=flag)
    _engine.check_nonfinite(flag)
    return IntegralImage(sq if squared else sat, kind, (img.rows, img.cols), squared, img.elem_kind, ld)


def build_sat(img: ImageGrid, squared: bool = False) -> IntegralImage:
    """Table of the image (or of its squared pixels), built on the device."""
    return _build(img, squared)


def window_sum(sat: IntegralImage, top: int, left: int, w: int):
    """Four-corner lookup of the w x w region at (top, left) (integral.py:119-130)."""
    rows, cols = sat.source_dims
    if w < 1 or top < 0 or left < 0 or top + w > rows or left + w > cols:
        raise InvalidWindowError(f"{w}x{w} region at ({top}, {left}) does not lie within the {rows}x{cols} source")
    import ctypes

    lib = _lib.load()
    buf = ctypes.c_uint64(0)
    dev = sat.device_table.device
    rc = lib.ssb_window_sum_at(int(sat.device_table.data_ptr()), 1 if sat.accum_kind is AccumKind.F64 else 0, rows,
                               cols, sat.pitch, top, left, w, ctypes.byref(buf), _device.stream_ptr(dev))
    _lib.check(rc, "window_sum")
    raw = np.array([buf.value], dtype=np.uint64)
    if sat.accum_kind is AccumKind.F64:
        return raw.view(np.float64)[0]
    if sat.elem_kind is ElemKind.I32:
        return raw.view(np.int64)[0]
    if sat.accum_kind is AccumKind.U128:
        return int(raw[0])  # region sums always fit 64 bits; exact
    return raw[0]


@_engine.device_scoped
def swa_with_table(img: ImageGrid, win: WindowSpec, stat: StatKind) -> tuple[IntegralImage, ResultGrid]:
    """build_sat(img) and swa_integral(img, win, stat) from one pass over the raster.

    The builder and sweep seams (integral.py:166-189) fused: the kernel that
    writes a table row also emits the windows whose bottom corner row it is,
    so the table is written once and never read back (ssb_sat_build_swa).
    Integer rasters, sum/mean, stride 1, w <= 257; any other request builds
    the table and then sweeps it (same results)."""
    win.validate_for(img.rows, img.cols)
    if not _engine.sweep_supported(img.elem_kind, win.w, win.stride, (stat,)):
        return _build(img, False), _run_tables(img, [win], stat)[0]
    kind = select_accum(img.elem_kind, img.rows, img.cols, False)
    x, dev = _engine.device_input(img)
    sat, ld, outs = _engine.table_and_sweep(x, img.elem_kind, img.rows, img.cols, win.w, (stat,), dev)
    table = IntegralImage(sat, kind, (img.rows, img.cols), False, img.elem_kind, ld)
    return table, ResultGrid(stat, _finish(img, (stat,), outs, win.w)[stat])


def _finish(img: ImageGrid, stats, res, w: int = 0) -> dict:
    out = {}
    for s in stats:
        v = res[s]
        if not img.on_device:
            v = _engine.result_to_host(v, img.elem_kind, s, w)
        out[s] = v
    return out


@_engine.device_scoped
def _run_tables(img: ImageGrid, wins, stat: StatKind, force_table: bool = False):
    """Tables once, then the corner sweep(s) (integral.py:166-189, :199-210).

    Stride-1 window sets go through ssb_window_eval_multi: one pass over the
    table serves every window."""
    import ctypes

    x, dev = _engine.device_input(img)
    flag = _engine.new_flag(dev) if img.elem_kind is ElemKind.F32 else None
    sq_needed = needs_squares(stat)
    if not force_table and img.elem_kind is ElemKind.F32:
        # float windows eligible for the fused kernel take it on every entry
        # point (_engine.float_fused), one launch per window; the others share
        # one table set
        fz = [_engine.float_fused(img.elem_kind, w.w, w.stride) for w in wins]
        if any(fz):
            rest = iter(_run_tables(img, [w for w, f in zip(wins, fz) if not f], stat, force_table=True)
                        if not all(fz) else [])
            out = []
            for win, f in zip(wins, fz):
                if f:
                    r = _engine.fused(x, img.elem_kind, img.rows, img.cols, win.w, (stat,), dev, flag=flag)
                    _engine.check_nonfinite(flag)
                    out.append(ResultGrid(stat, _finish(img, (stat,), r)[stat]))
                else:
                    out.append(next(rest))
            return out
    if len(wins) == 1 and _engine.sweep_supported(img.elem_kind, wins[0].w, wins[0].stride, (stat,)):
        # one window: table and sweep in one pass (the table stays in scratch)
        _, _, outs = _engine.table_and_sweep(x, img.elem_kind, img.rows, img.cols, wins[0].w, (stat,), dev,
                                             scratch=True)
        return [ResultGrid(stat, _finish(img, (stat,), outs, wins[0].w)[stat])]
    sat, sq, ld = _engine.build_tables(x, img.elem_kind, img.rows, img.cols, dev, squared=sq_needed, flag=flag,
                                       scratch=True)
    results = []
    if len(wins) > 1 and all(w.stride == 1 for w in wins):
        lib = _lib.load()
        outs = [_engine.alloc_outputs(img.elem_kind, (stat,), img.rows - w.w + 1, img.cols - w.w + 1, dev)[stat]
                for w in wins]
        n = len(wins)
        arr = lambda t, vals: (t * n)(*vals)  # noqa: E731
        ptrs = [int(o.data_ptr()) for o in outs]
        none = [None] * n
        rc = lib.ssb_window_eval_multi(
            int(sat.data_ptr()), None if sq is None else int(sq.data_ptr()), img.elem_kind.abi_code, img.rows,
            img.cols, ld, n, arr(ctypes.c_int64, [w.w for w in wins]), stat.bit,
            arr(ctypes.c_void_p, ptrs if stat is StatKind.SUM else none),
            arr(ctypes.c_void_p, ptrs if stat is StatKind.MEAN else none),
            arr(ctypes.c_void_p, ptrs if stat is StatKind.STD else none),
            arr(ctypes.c_int64, [img.cols - w.w + 1 for w in wins]), _device.stream_ptr(dev))
        _lib.check(rc, "multi-window evaluation")
        results = [{stat: o} for o in outs]
    else:
        for win in wins:
            results.append(_engine.eval_tables(sat, sq, ld, img.elem_kind, img.rows, img.cols, win.w, win.stride,
                                               (stat,), dev))
    _engine.check_nonfinite(flag)
    return [ResultGrid(stat, _finish(img, (stat,), r, w.w)[stat]) for r, w in zip(results, wins)]


def swa_integral(img: ImageGrid, win: WindowSpec, stat: StatKind) -> ResultGrid:
    """Sliding-window ``stat`` via device tables: build once, O(1) per window."""
    win.validate_for(img.rows, img.cols)
    return _run_tables(img, [win], stat)[0]


def swa_multi_window(img: ImageGrid, windows: list[WindowSpec], stat: StatKind) -> list[ResultGrid]:
    """Several window sizes from one set of tables; output i equals swa_integral(img, windows[i], stat)."""
    if not windows:
        raise ValueError("windows list must be non-empty")
    for win in windows:
        output_dims(img.rows, img.cols, win)
    return _run_tables(img, list(windows), stat)
