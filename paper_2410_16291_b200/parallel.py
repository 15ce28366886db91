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
from .grid import ImageGrid, ResultGrid, StatKind, WindowSpec
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


def _census_build(census: WriteCensus | None, img: ImageGrid, squared: bool, suffix: str) -> None:
    if census is None:
        return
    tw, sr, n_j, n_k = sat_tiling(img, squared)
    pr, pc = img.rows + 1, img.cols + 1
    for k in range(n_k):  # table rows [k0, k1) hold image rows [k0-1, k1-1)
        lo, hi = max(k * sr - 1, 0), min((k + 1) * sr, pr) - 1
        if hi > lo:
            census.record(f"rows/{suffix}", lo, hi)
    for j in range(n_j):
        lo, hi = max(j * tw - 1, 0), min((j + 1) * tw, pc) - 1
        if hi > lo:
            census.record(f"cols/{suffix}", lo, hi)


def build_sat_parallel(img: ImageGrid, squared: bool = False, cfg: ParallelConfig | None = None) -> IntegralImage:
    """Same table as build_sat, for every worker count (parallel.py:106-121)."""
    cfg = cfg or ParallelConfig()
    _census_build(cfg.census, img, squared, "sq" if squared else "sum")
    return _build(img, squared)


def swa_parallel(img: ImageGrid, win: WindowSpec, stat: StatKind, cfg: ParallelConfig | None = None) -> ResultGrid:
    """Table build plus corner sweep; bit-identical to swa_integral (parallel.py:137-149)."""
    cfg = cfg or ParallelConfig()
    win.validate_for(img.rows, img.cols)
    if cfg.census is not None:
        _census_build(cfg.census, img, needs_squares(stat), "sum")
        if needs_squares(stat):
            _census_build(cfg.census, img, True, "sq")
        out_r = (img.rows - win.w) // win.stride + 1
        cfg.census.record("query/sum", 0, out_r)
        if needs_squares(stat):
            cfg.census.record("query/sq", 0, out_r)
    return _run_tables(img, [win], stat)[0]
