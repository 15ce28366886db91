"""Array-in, array-out entry points (drop-in for pkg/src/satsweep/api.py).

``swa`` / ``multi_window`` keep the reference signatures and contracts: the
caller's buffer is never mutated, results are freshly allocated (uint64 for
integer sums, float64 otherwise), non-contiguous input is copied once, and
errors use the reference's exception types.

Placement follows the input: a numpy array goes through the C-ABI streaming
path ``ssb_swa_host`` (host -> device -> host, banded and overlapped) and
returns numpy; a CUDA ``torch.Tensor`` stays on the device and returns CUDA
tensors.  Keyword-only extensions: ``pipeline`` ("auto" | "table" | "fused")
and ``out`` (preallocated result array, e.g. in pinned memory).
"""

from __future__ import annotations

import numpy as np

from . import _device, _engine
from .grid import ImageGrid, StatKind, WindowSpec, _is_torch

METHODS = ("naive", "dp", "integral", "parallel")


def _as_grid(array) -> ImageGrid:
    if _is_torch(array):
        if array.dim() != 2:
            raise ValueError(f"expected a 2-D array, got {array.dim()} dimensions")
        return ImageGrid.from_array(array) if array.is_cuda else _as_grid(array.numpy())
    arr = np.asarray(array)
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-D array, got {arr.ndim} dimensions")
    # F32 finiteness is checked on the device by the first kernel that reads the
    # raster (same GridValidationError), saving the reference's extra host pass.
    return ImageGrid(np.ascontiguousarray(arr), _check_finite=False)


def _check_method(method: str, threads: int) -> None:
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}; expected naive, dp, integral, or parallel")
    if method == "parallel" and threads < 0:
        raise ValueError(f"workers must be >= 0 (0 = auto), got {threads}")


def _run(img: ImageGrid, win: WindowSpec, kinds, pipeline, outs, devices):
    if devices is not None:
        from . import multidev

        if img.on_device:
            if win.stride != 1:
                raise ValueError("the multi-device path for CUDA rasters needs stride 1")
            if outs is not None:
                raise ValueError("out= is not supported with devices= for CUDA rasters")
            return multidev.swa_device(img, win.w, kinds, devices)[0]
        return multidev.swa_host(img, win.w, win.stride, kinds, devices, pipeline, outs=outs)
    if img.on_device:
        return _engine.run_device(img, win.w, win.stride, kinds, pipeline, outs=outs)
    return _engine.run_host(img, win.w, win.stride, kinds, pipeline, outs=outs)


def swa_stats(array, window: int, stats=("sum",), stride: int = 1, *, pipeline: str = "auto", out=None,
              devices=None) -> dict:
    """Several statistics of one window from one pass (e.g. BASELINE C2's sum + mean).

    Returns {stat name: array}.  ``devices``: see ``swa``."""
    img = _as_grid(array)
    win = WindowSpec(window, stride)
    kinds = []
    for s in stats:
        k = StatKind.parse(s)
        if k not in kinds:
            kinds.append(k)
    win.validate_for(img.rows, img.cols)
    outs = None if out is None else {StatKind.parse(k): v for k, v in out.items()}
    res = _run(img, win, kinds, pipeline, outs, devices)
    return {k.value: res[k] for k in kinds}


def swa(array, window: int, stat: str = "sum", method: str = "parallel", stride: int = 1, threads: int = 0, *,
        pipeline: str = "auto", out=None, devices=None):
    """Sliding-window statistic over a 2-D array (api.py:28-55).

    ``method`` is accepted for compatibility; every method runs the GPU path
    (the reference guarantees all methods agree).  ``threads`` is ignored.
    ``devices`` (extension): ``None`` runs on the current GPU (a CUDA raster's
    own); ``"all"`` or a list of GPUs fans contiguous output-row bands over
    them from this process, the reference's worker partition
    (parallel.py:80-90) with GPUs as workers (multidev.py)."""
    img = _as_grid(array)
    win = WindowSpec(window, stride)
    kind = StatKind.parse(stat)
    _check_method(method, threads)
    win.validate_for(img.rows, img.cols)
    outs = None if out is None else {kind: out}
    return _run(img, win, [kind], pipeline, outs, devices)[kind]


def multi_window(array, windows: list[int], stat: str = "sum", *, pipeline: str = "auto") -> list:
    """Several window sizes (api.py:58-67); stride 1.

    ``"auto"``: large integer rasters evaluate every window without a table,
    the launches overlapped on concurrent streams (C3: 8.7 ms vs 10.8 ms for
    one table + one multi-window sweep; integer results are exact either
    way); small integer rasters build the table once, like the reference;
    float windows follow the same rule as ``swa`` (so output i is
    bit-identical to ``swa(array, windows[i], stat)``).
    ``"table"`` forces one table set for every window; ``"fused"`` evaluates
    each window without a table."""
    img = _as_grid(array)
    specs = [WindowSpec(w) for w in windows]
    kind = StatKind.parse(stat)
    if not specs:
        raise ValueError("windows list must be non-empty")
    for s in specs:
        s.validate_for(img.rows, img.cols)
    if pipeline not in ("auto", "table", "fused"):
        raise ValueError(f"unknown pipeline {pipeline!r}; expected auto, table, or fused")
    from .integral import _run_tables

    if pipeline == "auto" and _engine.multi_fused_wins(img.elem_kind, img.rows, img.cols, windows):
        pipeline = "fused"
    if pipeline in ("auto", "table"):
        grid = img if img.on_device else ImageGrid(img.values, img.elem_kind, _check_finite=False)
        return [r.values for r in _run_tables(grid, specs, kind, force_table=pipeline == "table")]
    if max(windows) > _engine.fused_max_w():
        raise ValueError("the fused pipeline needs w <= %d" % _engine.fused_max_w())
    # fused: every window from the raster, the launches on concurrent streams
    with _engine.on_device(img):
        x, dev = _engine.device_input(img)
        flag = _engine.new_flag(dev) if img.elem_kind.value == "f32" else None
        res = _engine.fused_windows(x, img.elem_kind, img.rows, img.cols, list(windows), [kind], dev, flag=flag)
        _engine.check_nonfinite(flag)
        out = [r[kind] for r in res]
        if not img.on_device:
            out = [_engine.result_to_host(o, img.elem_kind, kind, w) for o, w in zip(out, windows)]
        return out
