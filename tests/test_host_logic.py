"""Host-side logic of the drop-in facade (no kernel launches): data model,
validation and error contract, accumulator selection, partitioning, census.
Mirrors the reference's unit tests (pkg/tests/test_grid.py, test_stats.py,
test_parallel.py, test_api.py) for everything that does not compute."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

import paper_2410_16291_b200 as sb
from paper_2410_16291_b200 import api, integral, stats


class TestOutputDims:
    def test_whole_grid(self):
        assert sb.output_dims(5, 5, sb.WindowSpec(5)) == (1, 1)

    def test_large(self):
        assert sb.output_dims(30000, 30000, sb.WindowSpec(7000)) == (23001, 23001)

    def test_strided(self):
        assert sb.output_dims(10, 10, sb.WindowSpec(4, 3)) == (3, 3)

    def test_c5(self):
        assert sb.output_dims(70000, 85000, sb.WindowSpec(256)) == (69745, 84745)

    def test_too_large(self):
        with pytest.raises(sb.InvalidWindowError):
            sb.output_dims(4, 4, sb.WindowSpec(5))

    @given(rows=st.integers(1, 200), cols=st.integers(1, 200), w1=st.integers(1, 200), w2=st.integers(1, 200),
           stride=st.integers(1, 50))
    def test_monotone_in_window(self, rows, cols, w1, w2, stride):
        lo, hi = sorted((w1, w2))
        if hi > min(rows, cols):
            return
        a = sb.output_dims(rows, cols, sb.WindowSpec(hi, stride))
        b = sb.output_dims(rows, cols, sb.WindowSpec(lo, stride))
        assert a[0] <= b[0] and a[1] <= b[1]


class TestWindowSpec:
    def test_zero(self):
        with pytest.raises(sb.InvalidWindowError):
            sb.WindowSpec(0)
        with pytest.raises(sb.InvalidWindowError):
            sb.WindowSpec(3, 0)

    def test_is_value_error(self):
        with pytest.raises(ValueError):
            sb.WindowSpec(-1)


class TestImageGrid:
    def test_requires_2d(self):
        with pytest.raises(sb.GridValidationError):
            sb.ImageGrid(np.zeros(4, dtype=np.uint8))

    def test_empty(self):
        with pytest.raises(sb.GridValidationError):
            sb.ImageGrid(np.zeros((0, 3), dtype=np.uint8))

    def test_nan_inf(self):
        for bad in ([[1.0, np.nan]], [[np.inf, 1.0]]):
            with pytest.raises(sb.GridValidationError):
                sb.ImageGrid(np.array(bad, dtype=np.float32))

    def test_unsupported_dtype(self):
        with pytest.raises(TypeError):
            sb.ImageGrid(np.zeros((2, 2), dtype=np.int64))
        with pytest.raises(TypeError):
            sb.ImageGrid(np.zeros((2, 2), dtype=np.float64))

    def test_int32_extension(self):
        g = sb.ImageGrid(np.zeros((2, 2), dtype=np.int32))
        assert g.elem_kind is sb.ElemKind.I32 and g.elem_kind.sum_dtype == np.int64

    def test_readonly_view(self):
        arr = np.ones((3, 3), dtype=np.uint16)
        g = sb.ImageGrid(arr)
        with pytest.raises(ValueError):
            g.values[0, 0] = 5
        arr[0, 0] = 7
        assert g.values[0, 0] == 7

    def test_crop(self):
        g = sb.ImageGrid(np.arange(12, dtype=np.uint8).reshape(3, 4))
        assert g.crop(2, 3).values[1, 2] == 6


class TestStatKind:
    def test_parse(self):
        assert sb.StatKind.parse("MEAN") is sb.StatKind.MEAN
        with pytest.raises(ValueError):
            sb.StatKind.parse("median")


class TestSelectAccum:
    def test_bounds(self):
        assert sb.select_accum(sb.ElemKind.U16, 2 * 10**7, 14 * 10**6, False) is sb.AccumKind.U64
        assert sb.select_accum(sb.ElemKind.U16, 2 * 10**7, 15 * 10**6, False) is sb.AccumKind.U128
        assert sb.select_accum(sb.ElemKind.U16, 70000, 85000, True) is sb.AccumKind.U128
        assert sb.select_accum(sb.ElemKind.U16, 8192, 8192, True) is sb.AccumKind.U64
        assert sb.select_accum(sb.ElemKind.F32, 10**9, 10**9, True) is sb.AccumKind.F64
        assert sb.select_accum(sb.ElemKind.U8, 70000, 85000, False) is sb.AccumKind.U64

    def test_unwrap_modular_table(self):
        # exact values of a table that overflowed 2^64, recovered from its modular image
        rng = np.random.default_rng(3)
        exact = np.cumsum(rng.integers(0, 2**62, size=(3, 40), dtype=np.uint64).astype(object), axis=1)
        exact = np.concatenate([np.zeros((3, 1), dtype=object), exact], axis=1)
        mod = np.array([[int(x) % 2**64 for x in row] for row in exact], dtype=np.uint64)
        back = integral._unwrap_rows(mod)
        assert back.tolist() == exact.tolist()


class TestNumeratorBound:
    def test_u16(self):
        assert stats.exact_u64_numerator_ok(256, sb.ElemKind.U16)
        assert not stats.exact_u64_numerator_ok(257, sb.ElemKind.U16)

    def test_u8(self):
        limit = max(w for w in range(1, 6000) if w**4 * 255**2 <= 2**64 - 1)
        assert stats.exact_u64_numerator_ok(limit, sb.ElemKind.U8)
        assert not stats.exact_u64_numerator_ok(limit + 1, sb.ElemKind.U8)

    def test_float(self):
        assert not stats.exact_u64_numerator_ok(2, sb.ElemKind.F32)


class TestPartition:
    @given(n=st.integers(1, 5000), p=st.integers(1, 64))
    def test_cover(self, n, p):
        b = sb.partition(n, p)
        assert 1 <= len(b) <= p and b[0][0] == 0 and b[-1][1] == n
        assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
        sizes = [hi - lo for lo, hi in b]
        assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1


class TestParallelConfig:
    def test_negative(self):
        with pytest.raises(ValueError):
            sb.ParallelConfig(workers=-1)

    def test_threshold(self):
        cfg = sb.ParallelConfig(workers=8)
        assert cfg.effective_workers(100 * 100) == 1 and cfg.effective_workers(2048 * 2048) == 8


class TestCensus:
    def test_overlap_and_gap(self):
        c = sb.WriteCensus()
        c.record("rows/sum", 0, 3)
        c.record("rows/sum", 2, 5)
        with pytest.raises(AssertionError):
            c.assert_disjoint_cover("rows/sum", 5)
        c2 = sb.WriteCensus()
        c2.record("cols/sum", 0, 2)
        with pytest.raises(AssertionError):
            c2.assert_disjoint_cover("cols/sum", 4)


class TestApiValidation:
    """Errors raised before any device work (pkg/tests/test_api.py:11-37)."""

    def test_window_too_large(self):
        with pytest.raises(ValueError):
            sb.swa(np.ones((3, 3), dtype=np.uint8), 4, "sum")

    def test_unsupported_dtype(self):
        with pytest.raises(TypeError):
            sb.swa(np.ones((3, 3), dtype=np.int64), 2, "sum")

    def test_unknown_stat_and_method(self):
        arr = np.ones((3, 3), dtype=np.uint8)
        with pytest.raises(ValueError):
            sb.swa(arr, 2, "median")
        with pytest.raises(ValueError):
            sb.swa(arr, 2, "sum", method="gpu")

    def test_not_2d(self):
        with pytest.raises(ValueError):
            sb.swa(np.ones((3, 3, 3), dtype=np.uint8), 2)

    def test_multi_window_empty(self):
        with pytest.raises(ValueError):
            sb.multi_window(np.ones((3, 3), dtype=np.uint8), [], "sum")

    def test_multi_window_invalid_before_work(self):
        with pytest.raises(sb.InvalidWindowError):
            sb.multi_window(np.ones((8, 8), dtype=np.uint8), [2, 9], "sum")

    def test_pipeline_names(self):
        with pytest.raises(ValueError):
            api._engine.choose_pipeline("bogus", sb.ElemKind.U8, 3, 1)
