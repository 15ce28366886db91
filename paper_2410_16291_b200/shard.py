"""Row-band sharding across GPUs (one process per GPU, torch.distributed over NCCL).

The reference splits its table build and sweep over CPU threads
(pkg/src/satsweep/parallel.py:80-134); here the unit of parallelism is a GPU
holding a contiguous band of image rows:

* Window statistics (``swa_sharded``): rank g owns output rows
  [o_g, o_{g+1}) (the reference's ``partition`` rule) and the matching input
  rows; the (w-1)-row halo below its band arrives from the following ranks by
  point-to-point send/recv.  Each rank then evaluates its band locally -- the
  table offsets of rows above the band cancel in the four-corner difference,
  so no other global exchange is needed.
* Global table (``build_sat_sharded``): rank g owns input rows
  [a_g, a_{g+1}), reduces its band's column totals (the last row of its local
  table), all-gathers them and takes the exclusive scan over ranks as the
  carry row fed to the table kernel -- each rank ends up holding global table
  rows [a_g, a_{g+1}] without any extra pass over its table.

The orchestration is backend-agnostic: ``CudaBackend`` launches the library's
kernels; the CPU tests drive the same code over ``gloo`` with a numpy backend.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import ElemKind, StatKind
from .parallel import partition


def _dist():
    import torch.distributed as dist

    return dist


def world(group=None) -> tuple[int, int]:
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


# ----------------------------------------------------------------------------- geometry
def output_partition(out_r: int, n: int) -> list[tuple[int, int]]:
    """Output rows per rank (parallel.py:80-90 rule); ranks beyond out_r get empty bands."""
    parts = partition(out_r, n)
    while len(parts) < n:
        parts.append((out_r, out_r))
    return parts


def window_input_bands(rows: int, w: int, stride: int, n: int) -> list[tuple[int, int]]:
    """Input rows each rank OWNS for the window path: the rows that start its outputs,
    the last rank also owning the trailing rows."""
    out_r = (rows - w) // stride + 1
    parts = output_partition(out_r, n)
    owned = []
    for g, (lo, hi) in enumerate(parts):
        a = lo * stride
        b = parts[g + 1][0] * stride if g + 1 < n else rows
        owned.append((min(a, rows), min(max(b, a), rows)))
    # make the ownership a partition of [0, rows): empty output bands own nothing
    fixed, cur = [], 0
    for a, b in owned:
        a = max(a, cur)
        b = max(b, a)
        fixed.append((a, b))
        cur = b
    lo, hi = fixed[-1]
    fixed[-1] = (lo, rows)
    return fixed


def window_needed_rows(rows: int, w: int, stride: int, n: int) -> list[tuple[int, int]]:
    """Input rows each rank must HOLD to evaluate its output band (band + halo)."""
    out_r = (rows - w) // stride + 1
    need = []
    for lo, hi in output_partition(out_r, n):
        if hi <= lo:
            need.append((0, 0))
        else:
            need.append((lo * stride, (hi - 1) * stride + w))
    return need


def table_input_bands(rows: int, n: int) -> list[tuple[int, int]]:
    parts = partition(rows, n)
    while len(parts) < n:
        parts.append((rows, rows))
    return parts


# ----------------------------------------------------------------------------- exchange
def band_storage(rows: int, cols: int, w: int, stride: int, dtype, device=None, group=None):
    """Zero-copy layout for the window path: a tensor with room for this rank's
    band plus its halo, and the view holding the owned rows.  Fill the view,
    then pass both to ``halo_exchange(view, ..., storage=storage)``: the halo
    rows are received straight into the tail, so no per-step concatenation
    (a full read + write of the band) is needed."""
    import torch

    rank, n = world(group)
    a_own, b_own = window_input_bands(rows, w, stride, n)[rank]
    a_need, b_need = window_needed_rows(rows, w, stride, n)[rank]
    lo, hi = min(a_own, a_need) if b_need > a_need else a_own, max(b_own, b_need)
    storage = torch.empty((hi - lo, cols), dtype=dtype, device=device)
    return storage, storage[a_own - lo:b_own - lo]


def halo_exchange(band, rows: int, w: int, stride: int, group=None, storage=None):
    """Return this rank's band extended by the halo rows it needs (P2P send/recv).

    ``band`` is a 2-D tensor holding exactly the rows ``window_input_bands``
    assigns to this rank.  With ``storage`` (from ``band_storage``, ``band``
    being its owned-rows view) the halo is received in place and the needed
    rows are returned as a view -- no copy of the band."""
    import torch

    dist = _dist()
    rank, n = world(group)
    owned = window_input_bands(rows, w, stride, n)
    need = window_needed_rows(rows, w, stride, n)
    a_own, b_own = owned[rank]
    assert band.shape[0] == b_own - a_own, (band.shape, owned[rank])
    a_need, b_need = need[rank]
    if n == 1 or b_need <= a_need:
        return band[max(0, a_need - a_own):max(0, b_need - a_own)]
    base = None  # global row held by storage[0]
    if storage is not None:
        base = min(a_own, a_need)
        assert storage.shape[0] >= max(b_own, b_need) - base
        assert band.data_ptr() == storage[a_own - base:].data_ptr(), "band must be the owned-rows view of storage"
    ops, recv = [], []
    # what I receive: rows of [a_need, b_need) owned by other ranks
    for src in range(n):
        if src == rank:
            continue
        a, b = owned[src]
        lo, hi = max(a, a_need), min(b, b_need)
        if hi > lo:
            if base is not None:
                buf = storage[lo - base:hi - base]
            else:
                buf = torch.empty((hi - lo,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
            recv.append((lo, buf))
            ops.append(dist.P2POp(dist.irecv, buf, src, group))
    # what I send: my rows inside other ranks' needs
    for dst in range(n):
        if dst == rank:
            continue
        a, b = need[dst]
        lo, hi = max(a, a_own), min(b, b_own)
        if hi > lo:
            ops.append(dist.P2POp(dist.isend, band[lo - a_own:hi - a_own].contiguous(), dst, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if base is not None:
        return storage[a_need - base:b_need - base]
    pieces = []
    lo_own, hi_own = max(a_own, a_need), min(b_own, b_need)
    if hi_own > lo_own:
        pieces.append((lo_own, band[lo_own - a_own:hi_own - a_own]))
    pieces.extend(recv)
    pieces.sort(key=lambda p: p[0])
    return torch.cat([p[1] for p in pieces], dim=0)


def exclusive_scan_over_ranks(vec, add, group=None):
    """All-gather per-rank vectors and return (sum of lower ranks' vectors, sum of all)."""
    import torch

    dist = _dist()
    rank, n = world(group)
    if n == 1:
        return None, vec
    parts = [torch.empty_like(vec) for _ in range(n)]
    dist.all_gather(parts, vec.contiguous(), group)
    carry = None
    for g in range(rank):
        carry = parts[g].clone() if carry is None else add(carry, parts[g])
    total = None
    for p in parts:
        total = p.clone() if total is None else add(total, p)
    return carry, total


# ----------------------------------------------------------------------------- backends
class CudaBackend:
    """Local compute through libsatsweep_b200.so on this rank's device."""

    def __init__(self, device=None):
        from . import _device

        self.device = device or _device.current_device()

    def window(self, x, kind: ElemKind, w: int, stride: int, stats, pipeline: str = "auto"):
        from . import _engine
        from .grid import ImageGrid

        img = ImageGrid(x, kind)
        return _engine.run_device(img, w, stride, list(stats), pipeline)

    def band_totals(self, x, kind: ElemKind, squared: bool):
        import ctypes

        from . import _device, _engine, _lib

        lib = _lib.load()
        rows, cols = int(x.shape[0]), int(x.shape[1])
        acc = np.float64 if kind is ElemKind.F32 else np.uint64
        ws_bytes = int(lib.ssb_sat_workspace_bytes(kind.abi_code, rows, cols, 1 if squared else 0))
        ws = _device.empty((max(ws_bytes, 8),), np.uint8, self.device, "table workspace")
        tot = _device.empty((cols + 1,), acc, self.device, "band totals")
        tot_sq = _device.empty((cols + 1,), acc, self.device, "band totals") if squared else None
        rc = lib.ssb_sat_prepare(x.data_ptr(), kind.abi_code, rows, cols, cols, 1 if squared else 0, ws.data_ptr(),
                                 ws_bytes, tot.data_ptr(), None if tot_sq is None else tot_sq.data_ptr(), None,
                                 _device.stream_ptr(self.device))
        _lib.check(rc, "band totals")
        del ctypes, _engine
        return {"ws": ws, "ws_bytes": ws_bytes, "tot": tot, "tot_sq": tot_sq}

    def add(self, a, b):
        return a + b  # int64 storage wraps like uint64; float64 adds

    def finish(self, x, kind: ElemKind, state, carry, carry_sq, squared: bool):
        from . import _device, _engine, _lib

        lib = _lib.load()
        rows, cols = int(x.shape[0]), int(x.shape[1])
        ld = _engine.sat_ld_for(cols)
        acc = np.float64 if kind is ElemKind.F32 else np.uint64
        sat = None if squared else _device.empty((rows + 1, ld), acc, self.device, "band table")
        sq = _device.empty((rows + 1, ld), acc, self.device, "band table") if squared else None
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        rc = lib.ssb_sat_finish(x.data_ptr(), kind.abi_code, rows, cols, cols, ptr(sat), ptr(sq), ld, ptr(carry),
                                ptr(carry_sq), state["ws"].data_ptr(), state["ws_bytes"],
                                _device.stream_ptr(self.device))
        _lib.check(rc, "band table")
        return (sq if squared else sat), ld


# ----------------------------------------------------------------------------- entry points
@dataclass
class ShardedResult:
    """This rank's slice of a sharded result."""

    rows: tuple[int, int]   # global output rows [lo, hi) (window path) or table rows [lo, hi] (table path)
    values: dict            # {StatKind: tensor} or {"table": tensor}
    pitch: int = 0


def swa_sharded(band, rows: int, cols: int, kind: ElemKind, w: int, stats=(StatKind.SUM,), stride: int = 1,
                pipeline: str = "auto", backend=None, group=None, storage=None) -> ShardedResult:
    """Window statistics of a row-sharded image; outputs stay sharded on the ranks.

    ``storage``: see ``band_storage`` (zero-copy halo)."""
    rank, n = world(group)
    backend = backend or CudaBackend()
    x = halo_exchange(band, rows, w, stride, group, storage=storage)
    out_r = (rows - w) // stride + 1
    lo, hi = output_partition(out_r, n)[rank]
    if hi <= lo:
        return ShardedResult((lo, hi), {})
    assert x.shape[0] == (hi - lo - 1) * stride + w and x.shape[1] == cols
    return ShardedResult((lo, hi), backend.window(x, kind, w, stride, stats, pipeline))


def build_sat_sharded(band, rows: int, cols: int, kind: ElemKind, squared: bool = False, backend=None,
                      group=None) -> ShardedResult:
    """Global table rows [a_g, a_{g+1}] on rank g, from its image rows [a_g, a_{g+1})."""
    rank, n = world(group)
    backend = backend or CudaBackend()
    a, b = table_input_bands(rows, n)[rank]
    assert band.shape[0] == b - a
    state = backend.band_totals(band, kind, squared)
    mine = state["tot_sq"] if squared else state["tot"]
    carry, _ = exclusive_scan_over_ranks(mine, backend.add, group)
    table, ld = backend.finish(band, kind, state, None if squared else carry, carry if squared else None, squared)
    return ShardedResult((a, b), {"table": table}, ld)
