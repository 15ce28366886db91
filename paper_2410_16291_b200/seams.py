"""Adapters for the reference's internal seams.

The reference engine takes a *builder* ``builder(img, squared) -> IntegralImage``
in ``_sats_for_stat`` (pkg/src/satsweep/integral.py:166-169) and a *sweep*
``sweep(sat, win, out_r, out_c) -> ndarray`` in ``_finalize_from_sats``
(integral.py:178-189); ``parallel.py:147-149`` and ``bench.py:96-104`` already
swap them.  These two callables run the B200 kernels behind exactly those
signatures, so a maintainer can A/B the GPU table build and corner sweep inside
the reference's own harness:

    sum_sat, sq_sat = satsweep.integral._sats_for_stat(img, stat, seams.builder)
    res = satsweep.integral._finalize_from_sats(img, win, stat, sum_sat, sq_sat, sweep=seams.sweep)

They accept the reference's objects by duck typing (``img.values``,
``sat.table`` / ``win.w`` / ``win.stride``) and never import the reference.
"""

from __future__ import annotations

import numpy as np

from . import _device, _engine
from .grid import ElemKind, ImageGrid, StatKind
from .integral import IntegralImage, _build


def builder(img, squared: bool = False) -> IntegralImage:
    """GPU table of ``img.values``; the result's ``.table`` is the reference-shaped numpy table."""
    return _build(ImageGrid(np.ascontiguousarray(img.values), _check_finite=False), squared)


def sweep(sat, win, out_r: int, out_c: int) -> np.ndarray:
    """Corner sums ``(br - tr) - (bl - tl)`` of a table (ours, or a numpy one from the reference)."""
    w, s = int(win.w), int(getattr(win, "stride", 1))
    if isinstance(sat, IntegralImage):
        dev_table, ld, rows, cols = sat.device_table, sat.pitch, sat.rows, sat.cols
        is_float = sat.accum_kind.value == "f64"
        kind = ElemKind.F32 if is_float else (ElemKind.I32 if sat.elem_kind is ElemKind.I32 else ElemKind.U16)
    else:
        table = np.asarray(sat.table)
        if table.dtype == object:
            raise TypeError("object (U128) tables are not supported by the GPU sweep")
        rows, cols = table.shape[0] - 1, table.shape[1] - 1
        is_float = table.dtype == np.float64
        dev = _device.current_device()
        ld = _engine.sat_ld_for(cols)
        dev_table = _device.empty((rows + 1, ld), np.float64 if is_float else np.uint64, dev, "table")
        t = _device.torch()
        src = t.from_numpy(np.ascontiguousarray(table).view(np.float64 if is_float else np.int64))
        dev_table[:, : cols + 1].copy_(src)
        kind = ElemKind.F32 if is_float else ElemKind.U16
    res = _engine.eval_tables(dev_table, None, ld, kind, rows, cols, w, s, (StatKind.SUM,), dev_table.device)
    got = res[StatKind.SUM]
    assert tuple(got.shape) == (out_r, out_c)
    return _device.to_host(got, np.float64 if is_float else np.uint64)
