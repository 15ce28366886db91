"""Exactness dispatch of the statistic finalisation (pkg/src/satsweep/stats.py).

The arithmetic itself (SUM cast, MEAN = f64(s)/n, integer STD from the exact
numerator n*q - s^2, float STD from the clamped one-pass formula) is fused
into the CUDA kernels (csrc/ssb_common.cuh fin_*); these helpers expose the
same host-side decisions the reference makes.
"""

from __future__ import annotations

from .grid import ElemKind, StatKind

U64_MAX = 2**64 - 1


def exact_u64_numerator_ok(w: int, elem_kind: ElemKind) -> bool:
    """stats.py:28-32: n*q - s^2 provably fits uint64 for a w x w window."""
    if not elem_kind.is_integer or elem_kind is ElemKind.I32:
        return False
    return w**4 * int(elem_kind.max_value) ** 2 <= U64_MAX


def needs_squares(stat: StatKind) -> bool:
    """stats.py:77-78: only STD needs the squared table."""
    return stat is StatKind.STD
