"""Worker configuration, partitioning and the write census
(drop-in for pkg/src/satsweep/parallel.py).

On the GPU the "workers" of the reference are CTAs: the table build tiles the
padded grid into strips x segments (csrc/sat_build.cu) and the sweep covers
output rows with a persistent grid.  ``build_sat_parallel`` / ``swa_parallel``
run the same kernels as the sequential names -- results are bit-identical by
construction, as parallel.py:1-7 requires of every worker count.  Multi-GPU
row bands live in ``shard.py``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grid import ImageGrid, ResultGrid, StatKind, WindowSpec, output_dims
from .integral import IntegralImage, _build, _run_tables, select_accum  # noqa: F401
from .stats import needs_squares


@dataclass
class WriteCensus:
    """Which index ranges each phase wrote (parallel.py:35-51).

    The GPU path records the tiles its kernels actually use: table segments
    (``rows/*``), table strips (``cols/*``) and output rows (``query/*``),
    expressed in image / output index space."""

    ranges: dict[str, list[tuple[int, int]]] = field(default_factory=dict)

    def record(self, phase: str, lo: int, hi: int) -> None:
        self.ranges.setdefault(phase, []).append((lo, hi))

    def assert_disjoint_cover(self, phase: str, total: int) -> None:
        hits = np.zeros(total, dtype=np.int64)
        for lo, hi in self.ranges.get(phase, []):
            hits[lo:hi] += 1
        bad = np.flatnonzero(hits != 1)
        if bad.size:
            i = int(bad[0])
            raise AssertionError(f"phase {phase!r}: index {i} written {int(hits[i])} times")


@dataclass(frozen=True)
class ParallelConfig:
    """Worker count (0 = detected parallelism) and the sequential threshold (parallel.py:54-77).

    Kept for signature compatibility; the GPU kernels size their own grids."""

    workers: int = 0
    min_parallel_elems: int = 2**20
    census: WriteCensus | None = None

    def __post_init__(self):
        if self.workers < 0:
            raise ValueError(f"workers must be >= 0 (0 = auto), got {self.workers}")
        if self.min_parallel_elems < 0:
            raise ValueError("min_parallel_elems must be >= 0")

    def resolved_workers(self) -> int:
        return self.workers if self.workers >= 1 else (os.cpu_count() or 1)

    def effective_workers(self, total_elems: int) -> int:
        return 1 if total_elems < self.min_parallel_elems else self.resolved_workers()


def partition(n: int, p: int) -> list[tuple[int, int]]:
    """[0, n) as at most p contiguous non-empty blocks whose sizes differ by <= 1."""
    p = max(1, min(p, n))
    q, r = divmod(n, p)
    bounds = [0]
    for k in range(p):
        bounds.append(bounds[-1] + q + (k < r))
    return list(zip(bounds[:-1], bounds[1:]))


def sat_tiling(img: ImageGrid, squared: bool) -> tuple[int, int, int, int]:
    """(strip width, segment height, strips, segments) of the device table build."""
    info = (ctypes.c_int64 * 4)()
    _lib.check(_lib.load().ssb_sat_plan(img.elem_kind.abi_code, img.rows, img.cols, 1 if squared else 0, info))
    return tuple(int(v) for v in info)


class _DeviceCensus:
    """Counters the kernels themselves write while the census is enabled
    (ssb_census_enable): one per table row, table column and output row.  On
    exit the counts become WriteCensus records, so ``assert_disjoint_cover``
    checks what the device actually stored: index i is recorded once when its
    count is exactly one full row/column of stores, twice when it was stored
    more often or only partly (an overlap or a partial write fails the check),
    and not at all when nothing was stored (a gap fails it)."""

    def __init__(self, census: WriteCensus, img: ImageGrid, out_dims=None, table: bool = True):
        self.census, self.img, self.out_dims, self.table = census, img, out_dims, table

    def __enter__(self):
        import torch

        from . import _device

        dev = _device.current_device()
        pr, pc = self.img.rows + 1, self.img.cols + 1
        z = lambda n: torch.zeros(max(n, 1), dtype=torch.int64, device=dev)  # noqa: E731
        self.trow, self.tcol = (z(pr), z(pc)) if self.table else (None, None)
        self.orow = z(self.out_dims[0]) if self.out_dims else None
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _lib.check(_lib.load().ssb_census_enable(p(self.trow), pr, p(self.tcol), pc, p(self.orow),
                                                 self.out_dims[0] if self.out_dims else 0), "census")
        return self

    def __exit__(self, *exc):
        import torch

        _lib.load().ssb_census_disable()
        if exc[0] is not None:
            return False
        torch.cuda.synchronize()
        self.counts = {k: None if t is None else t.cpu().numpy() for k, t in
                       (("trow", self.trow), ("tcol", self.tcol), ("orow", self.orow))}
        return False

    def record(self, phase: str, which: str, expected: int, skip: int = 0) -> None:
        """counts[skip:] -> census records for indices 0.. (skip = the table's zero border)."""
        c = self.counts[which][skip:]
        full = c == expected
        i, n = 0, c.size
        while i < n:
            if full[i]:  # one record per run of exactly-covered indices
                j = i
                while j < n and full[j]:
                    j += 1
                self.census.record(phase, i, j)
                i = j
                continue
            if c[i] != 0:  # over- or partially-written: a double record fails the check
                self.census.record(phase, i, i + 1)
                self.census.record(phase, i, i + 1)
            i += 1

    def record_table(self, suffixes) -> None:
        """Table phases; nothing when no table was written (float windows that
        take the fused kernel, _engine.float_fused, never build one)."""
        pr, pc = self.img.rows + 1, self.img.cols + 1
        if not self.counts["trow"].any() and not self.counts["tcol"].any():
            return
        for sfx in suffixes:
            self.record(f"rows/{sfx}", "trow", pc, skip=1)
            self.record(f"cols/{sfx}", "tcol", pr, skip=1)
        # the zero border row/column are stores too: exactly one full row / column
        if self.counts["trow"][0] != pc or self.counts["tcol"][0] != pr:
            for sfx in suffixes:
                self.census.record(f"rows/{sfx}", 0, 1)  # forces a failed check on the border


def build_sat_parallel(img: ImageGrid, squared: bool = False, cfg: ParallelConfig | None = None) -> IntegralImage:
    """Same table as build_sat, for every worker count (parallel.py:106-121)."""
    cfg = cfg or ParallelConfig()
    if cfg.census is None:
        return _build(img, squared)
    with _DeviceCensus(cfg.census, img) as dc:
        table = _build(img, squared)
    dc.record_table(["sq" if squared else "sum"])
    return table


def swa_parallel(img: ImageGrid, win: WindowSpec, stat: StatKind, cfg: ParallelConfig | None = None) -> ResultGrid:
    """Table build plus corner sweep; bit-identical to swa_integral (parallel.py:137-149)."""
    cfg = cfg or ParallelConfig()
    win.validate_for(img.rows, img.cols)
    if cfg.census is None:
        return _run_tables(img, [win], stat)[0]
    out_r, out_c = output_dims(img.rows, img.cols, win)
    # the kernels count their own stores: table entries (the plain and squared
    # tables are written by one kernel) and output positions
    with _DeviceCensus(cfg.census, img, (out_r, out_c)) as dc:
        res = _run_tables(img, [win], stat)[0]
    sq = needs_squares(stat)
    dc.record_table(["sum", "sq"] if sq else ["sum"])
    dc.record("query/sum", "orow", out_c)
    if sq:
        dc.record("query/sq", "orow", out_c)
    return res
