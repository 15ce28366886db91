"""numpy restatement of the reference's integral-image SWA path (oracle; tests only).

Each function names the reference lines it restates (paths relative to
/root/reference/pkg/src/satsweep).  Arithmetic deliberately follows the same
numpy operations in the same order -- cumsum along rows then along columns,
the (br - tr) - (bl - tl) corner order, the exact-numerator std -- so integer
results and integer-input mean/std are bit-identical to the reference and F32
results match it to the last bit as well.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

U64_MAX = (1 << 64) - 1

_MAXV = {np.dtype(np.uint8): 255, np.dtype(np.uint16): 65535, np.dtype(np.int32): 1 << 31}


def is_int(values: np.ndarray) -> bool:
    return values.dtype.kind in "ui"


def accum_dtype(values: np.ndarray, squared: bool):
    """integral.py:44-55 select_accum -> storage dtype (object == the U128 arm)."""
    if not is_int(values):
        return np.dtype(np.float64)
    rows, cols = values.shape
    bound = _MAXV[values.dtype] ** (2 if squared else 1) * rows * cols
    if values.dtype == np.int32:  # extension: signed input accumulates in int64
        return np.dtype(np.int64) if bound <= (1 << 63) - 1 else np.dtype(object)
    return np.dtype(np.uint64) if bound <= U64_MAX else np.dtype(object)


def build_table(values: np.ndarray, squared: bool = False, row_blocks: int = 1, col_blocks: int = 1,
                pool: ThreadPoolExecutor | None = None) -> np.ndarray:
    """Zero-bordered (R+1) x (C+1) table: fill (+square), cumsum rows, cumsum cols.

    integral.py:76-116 (sequential) and parallel.py:106-121 (row blocks then
    column blocks, same bits for any block count)."""
    rows, cols = values.shape
    dt = accum_dtype(values, squared)
    t = np.zeros((rows + 1, cols + 1), dtype=dt)
    body = t[1:, 1:]

    def fill_scan(lo: int, hi: int) -> None:  # integral.py:86-101
        seg = body[lo:hi]
        if dt == object:
            seg[...] = values[lo:hi].astype(object)
            if squared:
                seg[...] = seg * seg
        elif squared:
            np.multiply(values[lo:hi], values[lo:hi], out=seg, dtype=dt, casting="unsafe")
        else:
            np.copyto(seg, values[lo:hi], casting="unsafe")
        np.cumsum(seg, axis=1, out=seg)

    def scan_down(lo: int, hi: int) -> None:  # integral.py:104-106
        seg = body[:, lo:hi]
        np.cumsum(seg, axis=0, out=seg)

    _blocks(fill_scan, rows, row_blocks, pool)
    _blocks(scan_down, cols, col_blocks, pool)
    return t


def split(n: int, p: int) -> list[tuple[int, int]]:
    """parallel.py:80-90: at most p balanced contiguous blocks, the first n % p one larger."""
    p = max(1, min(p, n))
    q, r = divmod(n, p)
    out, lo = [], 0
    for k in range(p):
        hi = lo + q + (1 if k < r else 0)
        out.append((lo, hi))
        lo = hi
    return out


def _blocks(fn, n: int, p: int, pool) -> None:
    parts = split(n, p)
    if len(parts) == 1 or pool is None:
        for lo, hi in parts:
            fn(lo, hi)
        return
    for f in [pool.submit(fn, lo, hi) for lo, hi in parts]:
        f.result()


def out_shape(rows: int, cols: int, w: int, stride: int) -> tuple[int, int]:
    """grid.py:150-156."""
    if w < 1 or stride < 1 or w > min(rows, cols):
        raise ValueError("invalid window")
    return (rows - w) // stride + 1, (cols - w) // stride + 1


def corner_sums(t: np.ndarray, w: int, stride: int, out_r: int, out_c: int, lo: int = 0,
                hi: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """integral.py:133-163: (br - tr) - (bl - tl) for output rows [lo, hi)."""
    hi = out_r if hi is None else hi
    rs = slice(lo * stride, (hi - 1) * stride + 1, stride)
    rb = slice(lo * stride + w, (hi - 1) * stride + w + 1, stride)
    cl = slice(0, (out_c - 1) * stride + 1, stride)
    cr = slice(w, (out_c - 1) * stride + w + 1, stride)
    dst = np.empty((hi - lo, out_c), dtype=t.dtype) if out is None else out[lo:hi]
    np.subtract(t[rb, cr], t[rs, cr], out=dst)
    dst -= t[rb, cl] - t[rs, cl]
    return dst


def std_numerator_fits_u64(w: int, values: np.ndarray) -> bool:
    """stats.py:28-32."""
    return is_int(values) and values.dtype != np.int32 and w**4 * _MAXV[values.dtype] ** 2 <= U64_MAX


def finalize(stat: str, s: np.ndarray, q: np.ndarray | None, w: int, values: np.ndarray) -> np.ndarray:
    """stats.py:35-74."""
    n = w * w
    if stat == "sum":
        if values.dtype == np.int32:
            return np.asarray(s, dtype=np.int64)
        return np.asarray(s, dtype=np.uint64 if is_int(values) else np.float64)
    if stat == "mean":
        return np.asarray(s, dtype=np.float64) / n
    if is_int(values):
        if s.dtype == np.uint64 and std_numerator_fits_u64(w, values):
            num = n * q - s * s
        else:
            so = np.asarray(s).astype(object)
            num = n * np.asarray(q).astype(object) - so * so
        return np.sqrt(num.astype(np.float64)) / n
    m = np.asarray(s, dtype=np.float64) / n
    v = np.asarray(q, dtype=np.float64) / n - m * m
    np.maximum(v, 0.0, out=v)
    return np.sqrt(v)


def swa(values: np.ndarray, w: int, stat: str = "sum", stride: int = 1) -> np.ndarray:
    """integral.py:192-196 swa_integral (sequential)."""
    out_r, out_c = out_shape(*values.shape, w, stride)
    t = build_table(values)
    s = corner_sums(t, w, stride, out_r, out_c)
    q = None
    if stat == "std":
        q = corner_sums(build_table(values, True), w, stride, out_r, out_c)
    return finalize(stat, s, q, w, values)


def swa_threaded(values: np.ndarray, w: int, stat: str = "sum", stride: int = 1, threads: int = 0) -> np.ndarray:
    """parallel.py:137-149 swa_parallel: blocked table build + row-blocked sweep on a thread pool."""
    p = threads or (os.cpu_count() or 1)
    rows, cols = values.shape
    out_r, out_c = out_shape(rows, cols, w, stride)
    with ThreadPoolExecutor(max_workers=p) as pool:
        def tab(sq: bool) -> np.ndarray:
            return build_table(values, sq, p, p, pool)

        def sweep(t: np.ndarray) -> np.ndarray:
            o = np.empty((out_r, out_c), dtype=t.dtype)
            _blocks(lambda lo, hi: corner_sums(t, w, stride, out_r, out_c, lo, hi, o), out_r, p, pool)
            return o

        s = sweep(tab(False))
        q = sweep(tab(True)) if stat == "std" else None
    return finalize(stat, s, q, w, values)


def multi_window(values: np.ndarray, windows, stat: str = "sum") -> list[np.ndarray]:
    """integral.py:199-210: every window validated first, tables built once."""
    if not windows:
        raise ValueError("windows list must be non-empty")
    for w in windows:
        out_shape(*values.shape, w, 1)
    t = build_table(values)
    tq = build_table(values, True) if stat == "std" else None
    res = []
    for w in windows:
        out_r, out_c = out_shape(*values.shape, w, 1)
        s = corner_sums(t, w, 1, out_r, out_c)
        q = corner_sums(tq, w, 1, out_r, out_c) if tq is not None else None
        res.append(finalize(stat, s, q, w, values))
    return res


def window_sum(t: np.ndarray, top: int, left: int, w: int):
    """integral.py:119-130."""
    rows, cols = t.shape[0] - 1, t.shape[1] - 1
    if w < 1 or top < 0 or left < 0 or top + w > rows or left + w > cols:
        raise ValueError("region outside the source")
    return (t[top + w, left + w] - t[top, left + w]) - (t[top + w, left] - t[top, left])


def brute_force(values: np.ndarray, w: int, stat: str = "sum", stride: int = 1) -> np.ndarray:
    """naive.py:27-60: direct window sums, two-pass std (independent of the tables)."""
    out_r, out_c = out_shape(*values.shape, w, stride)
    win = sliding_window_view(values, (w, w))[::stride, ::stride]
    acc = np.int64 if values.dtype == np.int32 else (np.uint64 if is_int(values) else np.float64)
    s = win.sum(axis=(2, 3), dtype=acc)
    if stat == "sum":
        return s
    mean = s.astype(np.float64) / (w * w)
    if stat == "mean":
        return mean
    dev = win.astype(np.float64) - mean[:, :, None, None]
    return np.sqrt((dev * dev).sum(axis=(2, 3)) / (w * w))
