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
    if n == 1:
        return band[max(0, a_need - a_own):max(0, b_need - a_own)]
    # a rank with no output rows receives nothing but still sends its rows to
    # the ranks whose windows reach into them
    empty = b_need <= a_need
    base = None  # global row held by storage[0]
    if storage is not None and not empty:
        base = min(a_own, a_need)
        assert storage.shape[0] >= max(b_own, b_need) - base
        assert band.data_ptr() == storage[a_own - base:].data_ptr(), "band must be the owned-rows view of storage"
    ops, recv = [], []
    # what I receive: rows of [a_need, b_need) owned by other ranks
    for src in range(n):
        if src == rank or empty:
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
    if empty:
        return band[:0]
    if base is not None:
        return storage[a_need - base:b_need - base]
    pieces = []
    lo_own, hi_own = max(a_own, a_need), min(b_own, b_need)
    if hi_own > lo_own:
        pieces.append((lo_own, band[lo_own - a_own:hi_own - a_own]))
    pieces.extend(recv)
    pieces.sort(key=lambda p: p[0])
    return torch.cat([p[1] for p in pieces], dim=0)


def gather_over_ranks(vec, group=None):
    """All-gather every rank's (len,) vector into one (n, len) tensor (rank order)."""
    import torch

    dist = _dist()
    rank, n = world(group)
    vec = vec.contiguous()
    if n == 1:
        return vec.unsqueeze(0)
    if vec.is_cuda:  # NCCL: one collective straight into the stacked buffer
        out = torch.empty((n,) + tuple(vec.shape), dtype=vec.dtype, device=vec.device)
        dist.all_gather_into_tensor(out, vec, group)
        return out
    parts = [torch.empty_like(vec) for _ in range(n)]
    dist.all_gather(parts, vec, group)
    return torch.stack(parts)


def exclusive_scan_over_ranks(vec, backend, group=None):
    """(sum of lower ranks' vectors, or None on rank 0) -- the carry row of this
    rank's band: the exclusive scan over bands of their column-total vectors,
    summed in rank order by ``backend.carry`` (a kernel on the CUDA backend)."""
    rank, n = world(group)
    if n == 1 or rank == 0:
        if n > 1:
            gather_over_ranks(vec, group)  # every rank takes part in the collective
        return None
    return backend.carry(gather_over_ranks(vec, group), rank)


# ----------------------------------------------------------------------------- backends
class CudaBackend:
    """Local compute through libsatsweep_b200.so on this rank's device.

    Buffers (workspace, totals, band table, outputs) are allocated on first
    use and reused by later calls of the same shape, so a repeated step
    (bench.py) allocates nothing."""

    def __init__(self, device=None):
        from . import _device

        self.device = device or _device.current_device()
        self._bufs: dict = {}
        self._side = None

    def _buf(self, key, shape, np_dtype, what):
        from . import _device

        cur = self._bufs.get(key)
        if cur is None or tuple(cur.shape) != tuple(shape) or cur.dtype != _device.storage_dtype(np_dtype):
            self._bufs.pop(key, None)
            cur = _device.empty(shape, np_dtype, self.device, what)
            self._bufs[key] = cur
        return cur

    def _outs(self, kind: ElemKind, stats, out_r: int, out_c: int):
        from . import _engine

        return {s: self._buf(("out", s), (out_r, out_c), _engine.result_dtype(kind, s), "band result") for s in stats}

    def window(self, x, kind: ElemKind, w: int, stride: int, stats, pipeline: str = "auto", outs=None):
        from . import _engine
        from .grid import ImageGrid

        img = ImageGrid(x, kind)
        return _engine.run_device(img, w, stride, list(stats), pipeline, outs=outs)

    def window_start(self, x, kind: ElemKind, w: int, stats):
        """Stride-1 window stats of ``x`` into reused outputs, on a side stream
        forked from the current one (overlaps the table phases); window_finish joins."""
        torch = __import__("torch")
        rows, cols = int(x.shape[0]), int(x.shape[1])
        outs = self._outs(kind, list(stats), rows - w + 1, cols - w + 1)
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        cur = torch.cuda.current_stream(self.device)
        self._side.wait_stream(cur)
        with torch.cuda.stream(self._side):
            pipe = "fused" if w <= _fused_max_w() else "table"
            res = self.window(x, kind, w, 1, stats, pipe, outs=outs)
        return res

    def window_finish(self, handle):
        torch = __import__("torch")
        torch.cuda.current_stream(self.device).wait_stream(self._side)
        return handle

    def band_totals(self, x, kind: ElemKind, squared: bool):
        from . import _device, _lib

        lib = _lib.load()
        rows, cols = int(x.shape[0]), int(x.shape[1])
        acc = np.float64 if kind is ElemKind.F32 else np.uint64
        ws_bytes = int(lib.ssb_sat_workspace_bytes(kind.abi_code, rows, cols, 1 if squared else 0))
        ws = self._buf("ws", (max(ws_bytes, 8),), np.uint8, "table workspace")
        tot = self._buf("tot", (cols + 1,), acc, "band totals")
        tot_sq = self._buf("tot_sq", (cols + 1,), acc, "band totals") if squared else None
        rc = lib.ssb_sat_prepare(x.data_ptr(), kind.abi_code, rows, cols, cols, 1 if squared else 0, ws.data_ptr(),
                                 ws_bytes, tot.data_ptr(), None if tot_sq is None else tot_sq.data_ptr(), None,
                                 _device.stream_ptr(self.device))
        _lib.check(rc, "band totals")
        return {"ws": ws, "ws_bytes": ws_bytes, "tot": None if squared else tot, "tot_sq": tot_sq}

    def carry(self, gathered, rank: int):
        """Sum of rows [0, rank) of the gathered (n, len) totals, in row order (ssb_band_carry)."""
        from . import _device, _lib

        lib = _lib.load()
        length = int(gathered.shape[1])
        out = self._buf(("carry", gathered.dtype), (length,), np.float64 if gathered.dtype == _device.torch().float64
                        else np.uint64, "carry row")
        is_float = 1 if gathered.dtype == _device.torch().float64 else 0
        _lib.check(lib.ssb_band_carry(gathered.data_ptr(), rank, length, length, is_float, out.data_ptr(),
                                      _device.stream_ptr(gathered.device)), "band carry")
        return out

    def finish(self, x, kind: ElemKind, state, carry, carry_sq, squared: bool):
        from . import _device, _engine, _lib

        lib = _lib.load()
        rows, cols = int(x.shape[0]), int(x.shape[1])
        ld = _engine.sat_ld_for(cols)
        acc = np.float64 if kind is ElemKind.F32 else np.uint64
        tab = self._buf(("table", squared), (rows + 1, ld), acc, "band table")
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        rc = lib.ssb_sat_finish(x.data_ptr(), kind.abi_code, rows, cols, cols, None if squared else ptr(tab),
                                ptr(tab) if squared else None, ld, ptr(carry), ptr(carry_sq), state["ws"].data_ptr(),
                                state["ws_bytes"], _device.stream_ptr(self.device))
        _lib.check(rc, "band table")
        return tab, ld


def _fused_max_w() -> int:
    from . import _engine

    return _engine.fused_max_w()


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
    carry = exclusive_scan_over_ranks(mine, backend, group)
    table, ld = backend.finish(band, kind, state, None if squared else carry, carry if squared else None, squared)
    return ShardedResult((a, b), {"table": table}, ld)


def swa_table_sharded(band, rows: int, cols: int, kind: ElemKind, w: int, stats=(StatKind.SUM,), backend=None,
                      group=None, storage=None):
    """The multi-GPU step of bench.py: the stride-1 window statistics of this
    rank's output band AND the global integral-image rows of its owned band.

    ``band`` holds the rows ``window_input_bands`` assigns to this rank (the
    owned-rows view of ``storage`` for the zero-copy halo).  The halo arrives by
    P2P, the windows run on a side stream (``backend.window_start``) while the
    table phases run on the current one: band column totals -> all-gather ->
    exclusive scan over ranks (the carry row) -> table rows written with the
    carry.  Returns (window result, table result); the table result holds
    global table rows [a_g, b_g] of the owned rows [a_g, b_g)."""
    rank, n = world(group)
    backend = backend or CudaBackend()
    x = halo_exchange(band, rows, w, 1, group, storage=storage)
    lo, hi = output_partition(rows - w + 1, n)[rank]
    a, b = window_input_bands(rows, w, 1, n)[rank]
    assert band.shape[0] == b - a
    handle = backend.window_start(x, kind, w, stats) if hi > lo else None
    if b > a:
        state = backend.band_totals(band, kind, False)
        carry = exclusive_scan_over_ranks(state["tot"], backend, group)
        table, ld = backend.finish(band, kind, state, carry, None, False)
    else:  # an empty band still joins the collective; its table is the carry row
        import torch

        acc = torch.float64 if kind is ElemKind.F32 else torch.int64
        zero = torch.zeros(cols + 1, dtype=acc, device=getattr(band, "device", None))
        carry = exclusive_scan_over_ranks(zero, backend, group)
        table, ld = (zero if carry is None else carry).unsqueeze(0).clone(), cols + 1
    vals = backend.window_finish(handle) if handle is not None else {}
    return ShardedResult((lo, hi), vals), ShardedResult((a, b), {"table": table}, ld)
