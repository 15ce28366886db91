"""Device-side orchestration of the CUDA kernels (tables, corner sweep, fused path).

Every function here launches work from libsatsweep_b200.so on the current
torch stream; nothing computes on the host.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _device, _lib
from .grid import ElemKind, ImageGrid, StatKind

STAT_ORDER = (StatKind.SUM, StatKind.MEAN, StatKind.STD)


def stat_mask(stats) -> int:
    m = 0
    for s in stats:
        m |= s.bit
    return m


def result_dtype(kind: ElemKind, stat: StatKind) -> np.dtype:
    """stats.py:49-74: integer SUM keeps exact integers, everything else float64."""
    return kind.sum_dtype if stat is StatKind.SUM else np.dtype(np.float64)


def sat_ld_for(cols: int) -> int:
    """Row pitch of a device table: a multiple of 4 elements (32-byte aligned rows), >= cols + 1."""
    return (cols + 4) & ~3


def device_input(img: ImageGrid):
    """Return (device tensor, device) for an ImageGrid, copying host rasters once.

    Device rasters must be 16-byte aligned for the TMA row staging; an unaligned
    view (e.g. a row slice) is copied once."""
    if img.on_device:
        x = img.values
        if x.data_ptr() % 16:
            x = x.clone()
        return x, x.device
    dev = _device.current_device()
    return _device.to_device(img.values, dev), dev


def _ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def check_nonfinite(flag) -> None:
    if flag is not None and int(flag.item()) != 0:
        _lib.check(_lib.ENONFINITE)


def new_flag(device):
    t = _device.torch()
    return t.zeros(1, dtype=t.int32, device=device)


class _Scratch(threading.local):
    """Grow-only scratch buffers for tables that never leave the library
    (swa / multi_window), so repeated calls do not churn multi-GB allocations
    through the caching allocator.  Keyed by thread, device AND stream: every
    kernel touching a buffer runs on the stream it was allocated for, so a call
    on another stream can never overwrite a table or workspace that an earlier
    call's kernels are still reading, and growing a buffer frees the old one in
    that stream's order.  release_scratch() frees them."""

    def __init__(self):
        self.bufs = {}

    def get(self, key, nbytes: int, device):
        k = (key, str(device), _device.stream_ptr(device))
        cur = self.bufs.get(k)
        if cur is None or cur.numel() < nbytes:
            self.bufs.pop(k, None)
            cur = _device.empty((max(nbytes, 8),), np.uint8, device, f"{nbytes} bytes of scratch")
            self.bufs[k] = cur
        return cur

    def clear(self):
        self.bufs.clear()


_SCRATCH = _Scratch()


def release_scratch() -> None:
    """Free the cached scratch tables (reused across swa/multi_window calls) and
    the host path's band buffers (kept reserved in the library's private pool)."""
    _SCRATCH.clear()
    if _lib.LIB_PATH.exists() and _device.torch().cuda.is_available():
        _lib.load().ssb_host_release()
    t = _device.torch()
    if t.cuda.is_available():
        t.cuda.empty_cache()


def _table_view(buf, rows: int, ld: int, acc_dt):
    n = (rows + 1) * ld
    return buf[: n * 8].view(_device.storage_dtype(acc_dt)).view(rows + 1, ld)


def build_tables(x, kind: ElemKind, rows: int, cols: int, device, *, squared: bool, plain: bool = True,
                 carry=None, carry_sq=None, flag=None, scratch: bool = False):
    """Build the (rows+1) x (cols+1) table(s) in HBM.  Returns (sat, sat_sq, sat_ld).

    ``plain=False`` with ``squared=True`` builds only the squared table (build_sat(img, squared=True)).
    ``scratch=True`` places the tables in the reusable scratch cache (callers that do not return them)."""
    lib = _lib.load()
    ld = sat_ld_for(cols)
    acc_dt = np.float64 if kind is ElemKind.F32 else np.uint64
    tbytes = (rows + 1) * ld * 8
    what = f"a {rows + 1}x{cols + 1} integral table"
    sat = sq = None
    if plain:
        sat = (_table_view(_SCRATCH.get("sat", tbytes, device), rows, ld, acc_dt) if scratch
               else _device.empty((rows + 1, ld), acc_dt, device, what))
    if squared:
        sq = (_table_view(_SCRATCH.get("sat_sq", tbytes, device), rows, ld, acc_dt) if scratch
              else _device.empty((rows + 1, ld), acc_dt, device, what))
    ws_bytes = int(lib.ssb_sat_workspace_bytes(kind.abi_code, rows, cols, 1 if squared else 0))
    ws = _SCRATCH.get("ws", ws_bytes, device)
    st = _device.stream_ptr(device)
    rc = lib.ssb_sat_build(_ptr(x), kind.abi_code, rows, cols, cols, _ptr(sat), _ptr(sq), ld, _ptr(carry),
                           _ptr(carry_sq), _ptr(ws), ws_bytes, _ptr(flag), st)
    _lib.check(rc, "build_sat", (rows + 1) * (cols + 1) * 8)
    return sat, sq, ld


def alloc_outputs(kind: ElemKind, stats, out_r: int, out_c: int, device):
    return {s: _device.empty((out_r, out_c), result_dtype(kind, s), device, f"a {out_r}x{out_c} result grid")
            for s in stats}


def eval_tables(sat, sq, ld: int, kind: ElemKind, rows: int, cols: int, w: int, stride: int, stats, device,
                outs=None):
    """Corner sweep + fused finalize for every requested stat in one launch."""
    lib = _lib.load()
    out_r, out_c = (rows - w) // stride + 1, (cols - w) // stride + 1
    outs = outs or alloc_outputs(kind, stats, out_r, out_c, device)
    o_sum, o_mean, o_std = (outs.get(StatKind.SUM), outs.get(StatKind.MEAN), outs.get(StatKind.STD))
    rc = lib.ssb_window_eval(_ptr(sat), _ptr(sq), kind.abi_code, rows, cols, ld, w, stride, stat_mask(stats),
                             _ptr(o_sum), _ptr(o_mean), _ptr(o_std), out_c, _device.stream_ptr(device))
    _lib.check(rc, "window evaluation")
    return outs


def sweep_supported(kind: ElemKind, w: int, stride: int, stats) -> bool:
    """Whether ssb_sat_build_swa (table + window sums in one pass) takes this request."""
    return stride == 1 and bool(_lib.load().ssb_sat_swa_supported(kind.abi_code, w, stat_mask(stats)))


def table_and_sweep(x, kind: ElemKind, rows: int, cols: int, w: int, stats, device, *, outs=None,
                    scratch: bool = False, onepass: bool = False):
    """Integral image AND its stride-1 window stats (ssb_sat_build_swa).

    Same table as build_tables and same outputs as eval_tables on it, but the
    table is never read back.  ``onepass`` selects the one-pass kernel
    (ssb_sat_build_swa_onepass).  Returns (sat, sat_ld, outs)."""
    lib = _lib.load()
    ld = sat_ld_for(cols)
    tbytes = (rows + 1) * ld * 8
    sat = (_table_view(_SCRATCH.get("sat", tbytes, device), rows, ld, np.uint64) if scratch
           else _device.empty((rows + 1, ld), np.uint64, device, f"a {rows + 1}x{cols + 1} integral table"))
    out_r, out_c = rows - w + 1, cols - w + 1
    outs = outs or alloc_outputs(kind, stats, out_r, out_c, device)
    ws_bytes = int(lib.ssb_sat_swa_workspace_bytes(kind.abi_code, rows, cols))
    ws = _SCRATCH.get("ws", ws_bytes, device)
    fn = lib.ssb_sat_build_swa_onepass if onepass else lib.ssb_sat_build_swa
    rc = fn(_ptr(x), kind.abi_code, rows, cols, cols, _ptr(sat), ld, w, stat_mask(stats),
            _ptr(outs.get(StatKind.SUM)), _ptr(outs.get(StatKind.MEAN)), out_c, _ptr(ws), ws_bytes,
            _device.stream_ptr(device))
    _lib.check(rc, "table + window sweep", (rows + 1) * (cols + 1) * 8)
    return sat, ld, outs


def fused(x, kind: ElemKind, rows: int, cols: int, w: int, stats, device, flag=None, outs=None, segments: int = 0):
    lib = _lib.load()
    out_r, out_c = rows - w + 1, cols - w + 1
    outs = outs or alloc_outputs(kind, stats, out_r, out_c, device)
    o_sum, o_mean, o_std = (outs.get(StatKind.SUM), outs.get(StatKind.MEAN), outs.get(StatKind.STD))
    rc = lib.ssb_window_fused(_ptr(x), kind.abi_code, rows, cols, cols, w, stat_mask(stats), _ptr(o_sum),
                              _ptr(o_mean), _ptr(o_std), out_c, _ptr(flag), segments, _device.stream_ptr(device))
    _lib.check(rc, "fused window evaluation")
    return outs


_SIDE: dict = {}


def _side_streams(device, n: int):
    t = _device.torch()
    key = str(device)
    cur = _SIDE.setdefault(key, [])
    while len(cur) < n:
        cur.append(t.cuda.Stream(device))
    return cur[:n]


def fused_windows(x, kind: ElemKind, rows: int, cols: int, windows, stats, device, flag=None):
    """Several stride-1 windows without a table, each on its own stream forked
    from (and joined back into) the current one, so the launches overlap and
    fill each other's tails.  Returns one {StatKind: tensor} per window."""
    t = _device.torch()
    cur = t.cuda.current_stream(device)
    outs = [alloc_outputs(kind, stats, rows - w + 1, cols - w + 1, device) for w in windows]
    sides = _side_streams(device, len(windows))
    for st in sides:
        st.wait_stream(cur)
    for w, o, st in zip(windows, outs, sides):
        with t.cuda.stream(st):
            fused(x, kind, rows, cols, w, stats, device, flag=flag, outs=o)
    for st in sides:
        cur.wait_stream(st)
    return outs


def multi_fused_wins(kind: ElemKind, rows: int, cols: int, windows) -> bool:
    """multi_window "auto": integer rasters of >= 2^24 pixels whose windows all
    fit the fused kernel take concurrent fused launches instead of one table
    (measured at C3, 30,000^2 u8, w = 25..400: 8.65 vs 10.79 ms)."""
    return (kind is not ElemKind.F32 and rows * cols >= (1 << 24) and len(windows) > 1
            and max(windows) <= fused_max_w())


def fused_max_w() -> int:
    return int(_lib.load().ssb_window_fused_max_w())


def choose_pipeline(pipeline: str, kind: ElemKind, w: int, stride: int) -> str:
    if pipeline not in ("auto", "table", "fused"):
        raise ValueError(f"unknown pipeline {pipeline!r}; expected auto, table, or fused")
    fusable = stride == 1 and w <= fused_max_w()
    if pipeline == "fused":
        if not fusable:
            raise ValueError("the fused pipeline needs stride 1 and w <= %d" % fused_max_w())
        return "fused"
    if pipeline == "table":
        return "table"
    # auto: integer results are exact on both pipelines, so take the cheaper
    # one (measured: the fused strip kernel wins for uint8 with w <= 256,
    # uint16 with w <= 128 and int32 with w <= 256 -- C2 0.69 vs 0.74 ms).
    # float results: see float_fused -- every entry point (swa, swa_integral,
    # swa_parallel, multi_window) routes a float window the same way, so all
    # methods still agree bit for bit (test_api.py:68-79).
    if not fusable:
        return "table"
    if kind is ElemKind.U8 and w <= 256:
        return "fused"
    if kind is ElemKind.U16 and w <= 128:
        return "fused"
    if kind is ElemKind.I32 and w <= 256:
        return "fused"
    if float_fused(kind, w, stride):
        return "fused"
    return "table"


def float_fused(kind: ElemKind, w: int, stride: int) -> bool:
    """Float windows evaluated without a table (vertical sliding sums + row
    prefix in float64, window_fused.cu): stride 1 and w <= 256 (the 512-column
    strips).  Measured at C4 (20,000 x 24,000 f32, mean + std, w=64) against the
    table pipeline's 4.6 ms; the results differ from the table's only in
    summation order (max rel. difference ~1e-10, rtol 1e-6 contract)."""
    return kind is ElemKind.F32 and stride == 1 and w <= 256


def run_device(img: ImageGrid, w: int, stride: int, stats, pipeline: str = "auto", outs=None):
    """All requested stats for one window on the device; returns {StatKind: tensor}."""
    with on_device(img):
        return _run_device(img, w, stride, stats, pipeline, outs)


def on_device(img: ImageGrid):
    """Make the raster's device current (streams, scratch and allocations follow it)."""
    import contextlib

    if img.on_device:
        return _device.torch().cuda.device(img.values.device)
    return contextlib.nullcontext()


def device_scoped(fn):
    """Decorator: run ``fn(img, ...)`` with the raster's device current."""
    import functools

    @functools.wraps(fn)
    def wrapper(img, *args, **kwargs):
        with on_device(img):
            return fn(img, *args, **kwargs)

    return wrapper


def _run_device(img: ImageGrid, w: int, stride: int, stats, pipeline: str, outs):
    x, dev = device_input(img)
    rows, cols = img.rows, img.cols
    pipe = choose_pipeline(pipeline, img.elem_kind, w, stride)
    flag = new_flag(dev) if img.elem_kind is ElemKind.F32 else None
    if pipe == "fused":
        res = fused(x, img.elem_kind, rows, cols, w, stats, dev, flag=flag, outs=outs)
    elif sweep_supported(img.elem_kind, w, stride, stats):
        res = table_and_sweep(x, img.elem_kind, rows, cols, w, stats, dev, outs=outs, scratch=True)[2]
    else:
        need_sq = StatKind.STD in stats
        sat, sq, ld = build_tables(x, img.elem_kind, rows, cols, dev, squared=need_sq, flag=flag, scratch=True)
        res = eval_tables(sat, sq, ld, img.elem_kind, rows, cols, w, stride, stats, dev, outs=outs)
    check_nonfinite(flag)
    return res


def result_to_host(tensor, kind: ElemKind, stat: StatKind, w: int = 0) -> np.ndarray:
    """A device result as the host array the reference returns (api.py:28-67).  Unsigned integer
    sums with a known window go through the narrow wire (ssb_sums_to_host): their bound
    w * w * max pixel decides whether they may cross PCIe as uint32 / uint16."""
    dt = result_dtype(kind, stat)
    if stat is StatKind.SUM and w > 0 and kind in (ElemKind.U8, ElemKind.U16):
        return _device.sums_to_host(tensor, w * w * int(kind.max_value))
    if np.dtype(dt).itemsize == 8:  # float64 / int64: no bound, copied through the ring as they are
        return _device.sums_to_host(tensor, 0).view(np.dtype(dt))
    return _device.to_host(tensor, dt)


def run_host(img: ImageGrid, w: int, stride: int, stats, pipeline: str = "auto", outs=None, band_rows: int = 0):
    """Host raster in, host results out, through the C-ABI streaming entry point ssb_swa_host."""
    lib = _lib.load()
    _device.require_cuda()
    kind = img.elem_kind
    pipe = choose_pipeline(pipeline, kind, w, stride)
    rows, cols = img.rows, img.cols
    out_r, out_c = (rows - w) // stride + 1, (cols - w) // stride + 1
    if outs is None:
        outs = {s: np.empty((out_r, out_c), dtype=result_dtype(kind, s)) for s in stats}
    for s, a in outs.items():
        if a.shape != (out_r, out_c) or a.dtype != result_dtype(kind, s) or not a.flags.c_contiguous:
            raise ValueError(f"out[{s.value}] must be a C-contiguous {result_dtype(kind, s)} array of shape "
                             f"{(out_r, out_c)}")
    src = img.values
    ptr = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    t = _device.torch()
    rc = lib.ssb_swa_host(src.ctypes.data_as(ctypes.c_void_p), kind.abi_code, rows, cols, cols, w, stride,
                          stat_mask(stats), ptr(outs.get(StatKind.SUM)), ptr(outs.get(StatKind.MEAN)),
                          ptr(outs.get(StatKind.STD)), out_c, _lib.PIPE_FUSED if pipe == "fused" else _lib.PIPE_TABLE,
                          t.cuda.current_device(), band_rows)
    _lib.check(rc, "swa")
    return outs
