"""One process, several GPUs: the reference's worker fan-out with devices as workers.

The reference's default ``swa(method="parallel")`` spreads one image over all
worker threads of the process (``api.py:51-52`` -> ``swa_parallel``,
``parallel.py:137-149``; workers default to ``os.cpu_count()``,
``parallel.py:71-72``), partitioning output rows with ``partition``
(``parallel.py:80-90``).  Here the workers are GPUs, with the same partition
rule:

* host rasters (numpy): every device streams its own output band through the
  C-ABI host path (``ssb_swa_host``: H2D of its input rows, compute, D2H into
  its slice of the result) from its own host thread -- each GPU brings its own
  PCIe link, and no device-to-device exchange is needed;
* device rasters (CUDA tensors): the owned rows are scattered to per-device
  band buffers and ``ssb_sharded_swa`` exchanges the (w-1)-row halos by peer
  copies, evaluates every band with the fused window kernel and, on request,
  builds the GLOBAL integral image by an exclusive scan of the bands' column
  totals (``ShardedTable``).
"""

from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _device, _engine, _lib
from .grid import ElemKind, ImageGrid, StatKind
from .parallel import partition


def resolve_devices(devices) -> list[int]:
    """``"all"`` -> every visible GPU; an int or a list of ints/torch devices -> their indices."""
    t = _device.torch()
    _device.require_cuda()
    if devices == "all":
        return list(range(t.cuda.device_count()))
    if isinstance(devices, (int, str)) or hasattr(devices, "type"):
        devices = [devices]
    out = []
    for d in devices:
        idx = t.device(d if not isinstance(d, int) else f"cuda:{d}").index
        out.append(t.cuda.current_device() if idx is None else idx)
    if not out:
        raise ValueError("devices must name at least one GPU")
    n = t.cuda.device_count()
    for i in out:
        if not 0 <= i < n:
            raise ValueError(f"no CUDA device {i} (visible: {n})")
    return out


@dataclass(frozen=True)
class BandGeom:
    """Rows of band g (ssb_sharded_plan): owned image rows, needed image rows,
    output rows, and the band buffer's row capacity (it starts at own_lo)."""

    own: tuple[int, int]
    need: tuple[int, int]
    out: tuple[int, int]
    cap_rows: int


def plan(rows: int, cols: int, w: int, ndev: int) -> list[BandGeom]:
    lib = _lib.load()
    buf = (ctypes.c_int64 * (7 * ndev))()
    _lib.check(lib.ssb_sharded_plan(rows, cols, w, ndev, buf), "sharding plan")
    v = list(buf)
    return [BandGeom((v[7 * g], v[7 * g + 1]), (v[7 * g + 2], v[7 * g + 3]), (v[7 * g + 4], v[7 * g + 5]),
                     v[7 * g + 6]) for g in range(ndev)]


# ----------------------------------------------------------------------------- host rasters
def swa_host(img: ImageGrid, w: int, stride: int, stats, devices, pipeline: str = "auto", outs=None):
    """Host raster in, host results out: output rows partitioned over ``devices``
    (parallel.py:80-90), each band streamed by ssb_swa_host on its device from
    its own thread (ctypes releases the GIL)."""
    lib = _lib.load()
    devs = resolve_devices(devices)
    kind = img.elem_kind
    pipe = _engine.choose_pipeline(pipeline, kind, w, stride)
    rows, cols = img.rows, img.cols
    out_r, out_c = (rows - w) // stride + 1, (cols - w) // stride + 1
    if outs is None:
        outs = {s: np.empty((out_r, out_c), dtype=_engine.result_dtype(kind, s)) for s in stats}
    for s, a in outs.items():
        if a.shape != (out_r, out_c) or a.dtype != _engine.result_dtype(kind, s) or not a.flags.c_contiguous:
            raise ValueError(f"out[{s.value}] must be a C-contiguous {_engine.result_dtype(kind, s)} array of shape "
                             f"{(out_r, out_c)}")
    src = img.values
    es = src.dtype.itemsize
    parts = [p for p in partition(out_r, len(devs)) if p[1] > p[0]]

    def band(g):
        lo, hi = parts[g]
        nrows = (hi - lo - 1) * stride + w
        base = src.ctypes.data + lo * stride * cols * es
        ptr = lambda a: None if a is None else a.ctypes.data + lo * out_c * 8  # noqa: E731
        rc = lib.ssb_swa_host(base, kind.abi_code, nrows, cols, cols, w, stride, _engine.stat_mask(stats),
                              ptr(outs.get(StatKind.SUM)), ptr(outs.get(StatKind.MEAN)), ptr(outs.get(StatKind.STD)),
                              out_c, _lib.PIPE_FUSED if pipe == "fused" else _lib.PIPE_TABLE, devs[g % len(devs)], 0)
        return rc

    if len(parts) == 1:
        codes = [band(0)]
    else:
        # the concurrent calls share the host cores for widening narrow-wire results
        prev = lib.ssb_host_threads(max(1, (os.cpu_count() or 2) // len(parts) - 1))
        try:
            with ThreadPoolExecutor(len(parts)) as ex:
                codes = list(ex.map(band, range(len(parts))))
        finally:
            lib.ssb_host_threads(prev)
    for rc in codes:
        _lib.check(rc, "swa")
    return outs


# ----------------------------------------------------------------------------- device rasters
@dataclass
class ShardedTable:
    """The global (rows+1) x (cols+1) integral image, sharded by row bands:
    ``tables[g]`` on ``devices[g]`` holds global table rows [own[g][0], own[g][1]]."""

    tables: list
    own: list
    devices: list
    pitch: int
    cols: int

    def to_host(self) -> np.ndarray:
        dt = np.float64 if self.tables[0].dtype == _device.torch().float64 else np.uint64
        pieces = [_device.to_host(t[: (b - a + 1) if g == len(self.tables) - 1 else (b - a)], dt)[:, : self.cols + 1]
                  for g, (t, (a, b)) in enumerate(zip(self.tables, self.own))]
        return np.concatenate(pieces, axis=0)


def swa_device(img: ImageGrid, w: int, stats, devices, *, with_table: bool = False, gather: bool = True):
    """Stride-1 window statistics (and optionally the global table) of a CUDA raster,
    sharded over ``devices`` by ssb_sharded_swa.

    Returns ({StatKind: tensor on the raster's device} (or per-device lists with
    gather=False), ShardedTable or None)."""
    t = _device.torch()
    lib = _lib.load()
    devs = resolve_devices(devices)
    n = len(devs)
    kind = img.elem_kind
    x = img.values
    rows, cols = img.rows, img.cols
    if w > _engine.fused_max_w():
        raise ValueError(f"the multi-device path needs w <= {_engine.fused_max_w()}")
    geo = plan(rows, cols, w, n)
    out_c = cols - w + 1
    bands, sats, outs, wss, wsb, streams = [], [], [], [], [], []
    flags = []
    ld = _engine.sat_ld_for(cols)
    acc = np.float64 if kind is ElemKind.F32 else np.uint64
    for g, (d, gm) in enumerate(zip(devs, geo)):
        dev = t.device("cuda", d)
        with t.cuda.device(dev):
            b = _device.empty((max(gm.cap_rows, 1), cols), kind.dtype, dev, "band buffer")
            a0, a1 = gm.own
            if a1 > a0:
                b[: a1 - a0].copy_(x[a0:a1], non_blocking=True)  # scatter (peer copy across devices)
            if kind is ElemKind.F32 and a1 > a0:
                f = t.zeros(1, dtype=t.int32, device=dev)
                _lib.check(lib.ssb_f32_nonfinite(b.data_ptr(), (a1 - a0) * cols, f.data_ptr(),
                                                 _device.stream_ptr(dev)), "finiteness")
                flags.append(f)
            bands.append(b)
            nout = gm.out[1] - gm.out[0]
            outs.append({s: _device.empty((max(nout, 1), out_c), _engine.result_dtype(kind, s), dev, "band result")
                         for s in stats})
            if with_table:
                sats.append(_device.empty((a1 - a0 + 1, ld), acc, dev, "band table"))
            nb = int(lib.ssb_sharded_workspace_bytes(kind.abi_code, rows, cols, w, n, g, 1 if with_table else 0))
            wss.append(_device.empty((nb,), np.uint8, dev, "workspace"))
            wsb.append(nb)
            streams.append(_device.stream_ptr(dev))
    # the scatter above runs on the source device's stream: order it before the band streams
    src_ev = t.cuda.Event()
    src_ev.record(t.cuda.current_stream(x.device))
    for d in devs:
        t.cuda.current_stream(t.device("cuda", d)).wait_event(src_ev)

    P = ctypes.c_void_p
    arr = lambda typ, vals: (typ * n)(*vals)  # noqa: E731
    optr = lambda s: arr(P, [o[s].data_ptr() if s in o else None for o in outs]) if s in stats else None  # noqa: E731
    rc = lib.ssb_sharded_swa(n, arr(ctypes.c_int, devs), kind.abi_code, rows, cols, w, _engine.stat_mask(stats),
                             arr(P, [b.data_ptr() for b in bands]),
                             arr(P, [s.data_ptr() for s in sats]) if with_table else None, ld,
                             optr(StatKind.SUM), optr(StatKind.MEAN), optr(StatKind.STD), out_c,
                             arr(P, [wv.data_ptr() for wv in wss]), arr(ctypes.c_int64, wsb), arr(P, streams))
    _lib.check(rc, "sharded swa")
    for f in flags:
        _engine.check_nonfinite(f)
    res = {}
    for s in stats:
        pieces = [o[s][: gm.out[1] - gm.out[0]] for o, gm in zip(outs, geo) if gm.out[1] > gm.out[0]]
        res[s] = t.cat([p.to(x.device) for p in pieces]) if gather else pieces
    table = ShardedTable(sats, [gm.own for gm in geo], devs, ld, cols) if with_table else None
    return res, table


def build_sat_devices(img: ImageGrid, devices) -> ShardedTable:
    """build_sat (integral.py:109-116) of a CUDA raster, sharded over ``devices``."""
    return swa_device(img, 1, [], devices, with_table=True)[1]
