"""GPU parity of the one-pass table + window sweep (ssb_sat_build_swa, csrc/sat_sweep.cu).

The kernel writes the integral image and the stride-1 window sums/means in
one pass.  Its table must be bit-identical to ssb_sat_build's (and to the
oracle's restatement of build_sat, integral.py:109-116), and its outputs
bit-identical to the oracle's swa (integral.py:141-189, stats.py:35-56) and to
the two-kernel table pipeline (ssb_sat_build -> ssb_window_eval)."""

from __future__ import annotations

import zlib

import numpy as np
import pytest

from oracle import satsweep_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2410_16291_b200 import _lib, build_ext

    build_ext.build()
    _lib.load()
    import paper_2410_16291_b200 as mod

    return mod


@pytest.fixture(scope="module")
def dev():
    import torch

    return torch.device("cuda", 0)


def host(t, dt):
    from paper_2410_16291_b200 import _device

    return _device.to_host(t, dt)


def to_dev(a, dev):
    from paper_2410_16291_b200 import _device

    return _device.to_device(a, dev)


def raster(kind: str, rows: int, cols: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "u8":
        return rng.integers(0, 256, (rows, cols), dtype=np.uint8)
    if kind == "u8mask":
        return (rng.random((rows, cols)) < 0.05).astype(np.uint8)
    if kind == "u16":
        return rng.integers(0, 65536, (rows, cols), dtype=np.uint16)
    return rng.integers(-(2**31), 2**31, (rows, cols), dtype=np.int64).astype(np.int32)


def oracle_table(v: np.ndarray) -> np.ndarray:
    t = O.build_table(v)
    return t.view(np.uint64) if t.dtype == np.int64 else t


def two_kernel(sb, x, kind, rows, cols, w, stats, dev):
    from paper_2410_16291_b200 import _engine

    sat, sq, ld = _engine.build_tables(x, kind, rows, cols, dev, squared=False)
    outs = _engine.eval_tables(sat, sq, ld, kind, rows, cols, w, 1, stats, dev)
    return sat, ld, outs


def check_case(sb, dev, kind: str, rows: int, cols: int, w: int, seed: int, stats=("sum",), onepass=False):
    from paper_2410_16291_b200 import _engine
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    v = raster(kind, rows, cols, seed)
    ek = ElemKind.from_dtype(v.dtype)
    sk = tuple(StatKind.parse(s) for s in stats)
    assert _engine.sweep_supported(ek, w, 1, sk)
    x = to_dev(v, dev)
    sat, ld, outs = _engine.table_and_sweep(x, ek, rows, cols, w, sk, dev, onepass=onepass)
    got_t = host(sat[:, : cols + 1], np.uint64)
    np.testing.assert_array_equal(got_t, oracle_table(v), err_msg=f"table {kind} {rows}x{cols} w={w}")
    sat2, ld2, outs2 = two_kernel(sb, x, ek, rows, cols, w, sk, dev)
    assert np.array_equal(got_t, host(sat2[:, : cols + 1], np.uint64))
    for s, k in zip(stats, sk):
        ref = O.swa(v, w, s)
        dt = np.float64 if s == "mean" else (np.int64 if kind == "i32" else np.uint64)
        got = host(outs[k], dt)
        np.testing.assert_array_equal(got, ref, err_msg=f"{s} {kind} {rows}x{cols} w={w}")
        np.testing.assert_array_equal(got, host(outs2[k], dt))


@pytest.mark.parametrize("onepass", [False, True], ids=["build+fused", "onepass"])
@pytest.mark.parametrize("kind", ["u8", "u8mask", "u16", "i32"])
@pytest.mark.parametrize("shape,w", [((1, 1), 1), ((7, 5), 3), ((300, 517), 17), ((260, 1030), 256),
                                     ((257, 257), 257), ((600, 1600), 2), ((520, 2200), 255)])
def test_sweep_shapes(sb, dev, kind, shape, w, onepass):
    if kind == "u16" and w > 256:
        pytest.skip("u16 takes w <= 256 (u32 window sums)")
    check_case(sb, dev, kind, *shape, w, seed=zlib.crc32(f"{kind}{shape}{w}".encode()), onepass=onepass)


@pytest.mark.parametrize("onepass", [False, True], ids=["build+fused", "onepass"])
@pytest.mark.parametrize("kind", ["u8", "u16", "i32"])
def test_sweep_multi_segment(sb, dev, kind, onepass):
    """Rows span many sweep segments: every segment after the first warms its
    vertical sums up over the w rows above it (one-pass kernel)."""
    check_case(sb, dev, kind, 4500, 700, 200, seed=11, stats=("sum", "mean"), onepass=onepass)


@pytest.mark.parametrize("onepass", [False, True], ids=["build+fused", "onepass"])
@pytest.mark.parametrize("w", [1, 64, 256, 257])
def test_sweep_mean(sb, dev, w, onepass):
    check_case(sb, dev, "u8", 2300, 1100, w, seed=w, stats=("mean",), onepass=onepass)


def test_sweep_api(sb, dev):
    """swa_with_table returns build_sat's table and swa's result; swa(pipeline='table')
    routes here for eligible requests, with the reference's result dtype."""
    v = raster("u8", 1200, 900, 3)
    x = to_dev(v, dev)
    sat, res = sb.swa_with_table(sb.ImageGrid(x), sb.WindowSpec(100), sb.StatKind.SUM)
    np.testing.assert_array_equal(sat.table, oracle_table(v))
    np.testing.assert_array_equal(host(res.values, np.uint64), O.swa(v, 100, "sum"))
    hsat, hres = sb.swa_with_table(sb.ImageGrid(v), sb.WindowSpec(100), sb.StatKind.MEAN)
    assert hres.values.dtype == np.float64
    np.testing.assert_array_equal(hres.values, O.swa(v, 100, "mean"))
    assert sb.window_sum(hsat, 5, 7, 100) == O.swa(v, 100, "sum")[5, 7]
    np.testing.assert_array_equal(sb.swa(v, 100, "sum", pipeline="table"), O.swa(v, 100, "sum"))
    # ineligible requests (std, f32, wide windows) take build + sweep with the same contract
    f = np.random.default_rng(4).random((300, 400), dtype=np.float32)
    fsat, fres = sb.swa_with_table(sb.ImageGrid(f), sb.WindowSpec(20), sb.StatKind.STD)
    np.testing.assert_allclose(fres.values, O.swa(f, 20, "std"), rtol=1e-6, atol=1e-9)
    np.testing.assert_array_equal(fsat.table, O.build_table(f))
    wsat, wres = sb.swa_with_table(sb.ImageGrid(v), sb.WindowSpec(300), sb.StatKind.SUM)
    np.testing.assert_array_equal(wres.values, O.swa(v, 300, "sum"))


def test_sweep_c5_band(sb, dev, hashes):
    """A reference-hashed C5 band (rows [34000, 34512) of the w=256 result)."""
    from conftest import digest
    from paper_2410_16291_b200 import _engine, synthetic
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    lo, hi = 34000, 34512
    v = synthetic.c5(lo, hi + 255)
    x = to_dev(v, dev)
    import torch

    sat2, _, _ = two_kernel(sb, x, ElemKind.U8, v.shape[0], v.shape[1], 256, (StatKind.SUM,), dev)
    for onepass in (False, True):
        sat, ld, outs = _engine.table_and_sweep(x, ElemKind.U8, v.shape[0], v.shape[1], 256, (StatKind.SUM,), dev,
                                                onepass=onepass)
        assert digest(host(outs[StatKind.SUM], np.uint64)) == hashes[f"C5_sum_w256_rows{lo}_{hi}"]
        assert bool(torch.equal(sat[:, : v.shape[1] + 1], sat2[:, : v.shape[1] + 1]))


def test_sweep_concurrent_callers(sb, dev):
    """ssb_sat_build_swa forks its window kernel onto a per-thread side stream:
    threads calling it at once (each on its own torch stream, rasters >= 2^24 px so
    the fork/join path runs) get correct, independent tables and sums."""
    import threading

    import torch

    from paper_2410_16291_b200 import _engine
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    imgs = [raster("u8", 4200 + 16 * k, 4100, 40 + k) for k in range(3)]
    refs = [O.swa(v, 64, "sum") for v in imgs]
    tabs = [oracle_table(v)[-1] for v in imgs]  # last table row: the column totals
    errs = []

    def work(k):
        try:
            st = torch.cuda.Stream(dev)
            with torch.cuda.stream(st):
                x = to_dev(imgs[k], dev)
                for _ in range(2):
                    sat, _, outs = _engine.table_and_sweep(x, ElemKind.U8, *imgs[k].shape, 64, (StatKind.SUM,), dev)
                    st.synchronize()
                    np.testing.assert_array_equal(host(outs[StatKind.SUM], np.uint64), refs[k])
                    np.testing.assert_array_equal(host(sat[-1, : imgs[k].shape[1] + 1], np.uint64), tabs[k])
        except Exception as exc:  # pragma: no cover
            errs.append(exc)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


@pytest.mark.parametrize("case", range(6))
def test_sweep_fork_join_fuzz(sb, dev, case):
    """Seeded random rasters of >= 2^24 px (the fork/join path: table build on the
    caller's stream, fused windows on the side stream) in every eligible kind and a
    random window; table and sums vs the oracle."""
    from paper_2410_16291_b200 import _engine
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    rng = np.random.default_rng(1000 + case)
    kind = ["u8", "u8mask", "u16"][case % 3]
    rows, cols = int(rng.integers(2100, 5200)), int(rng.integers(3300, 8200))
    if rows * cols < 1 << 24:
        cols = (1 << 24) // rows + 1
    w = int(rng.integers(1, 129 if kind == "u16" else 257))
    stats = [("sum",), ("mean",), ("sum", "mean")][int(rng.integers(0, 3))]
    v = raster(kind, rows, cols, 2000 + case)
    x = to_dev(v, dev)
    sk = tuple(StatKind.parse(s) for s in stats)
    sat, _, outs = _engine.table_and_sweep(x, ElemKind.from_dtype(v.dtype), rows, cols, w, sk, dev)
    np.testing.assert_array_equal(host(sat[:, : cols + 1], np.uint64), oracle_table(v))
    for s, k in zip(stats, sk):
        np.testing.assert_array_equal(host(outs[k], np.float64 if s == "mean" else np.uint64), O.swa(v, w, s),
                                      err_msg=f"{kind} {rows}x{cols} w={w} {s}")


def test_sweep_host_bands(sb):
    """numpy in, numpy out (ssb_swa_host): bands of >= 2^24 px take the table + concurrent
    fused-windows path inside the banded H2D/compute/D2H pipeline; sums and means equal the
    oracle's, and the caller's array is untouched."""
    v = raster("u8", 9000, 9000, 77)
    before = v.copy()
    got = sb.swa_stats(v, 256, ("sum", "mean"), pipeline="table")
    assert got["sum"].dtype == np.uint64 and got["mean"].dtype == np.float64
    np.testing.assert_array_equal(got["sum"], O.swa(v, 256, "sum"))
    np.testing.assert_array_equal(got["mean"], O.swa(v, 256, "mean"))
    np.testing.assert_array_equal(v, before)


@pytest.mark.parametrize("case", range(12))
def test_onepass_fuzz(sb, dev, case):
    """Seeded random shapes, kinds, windows and stats through the one-pass kernel
    (ssb_sat_build_swa_onepass): strips partly outside the image, segments with and
    without warm-up, odd and even windows, unaligned output rows; table and windows
    vs the oracle."""
    from paper_2410_16291_b200 import _engine
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    rng = np.random.default_rng(5000 + case)
    kind = ["u8", "u8mask", "u16", "i32"][case % 4]
    rows, cols = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
    if case >= 10:  # a couple of large ones: one-wave tiling, long segments
        rows, cols = int(rng.integers(5000, 9000)), int(rng.integers(3000, 6000))
    wmax = min(rows, cols, 256 if kind == "u16" else 257)
    w = int(rng.integers(1, wmax + 1))
    stats = [("sum",), ("mean",), ("sum", "mean")][int(rng.integers(0, 3))]
    v = raster(kind, rows, cols, 6000 + case)
    x = to_dev(v, dev)
    sk = tuple(StatKind.parse(s) for s in stats)
    sat, _, outs = _engine.table_and_sweep(x, ElemKind.from_dtype(v.dtype), rows, cols, w, sk, dev, onepass=True)
    np.testing.assert_array_equal(host(sat[:, : cols + 1], np.uint64), oracle_table(v))
    for s, k in zip(stats, sk):
        dt = np.float64 if s == "mean" else (np.int64 if kind == "i32" else np.uint64)
        np.testing.assert_array_equal(host(outs[k], dt), O.swa(v, w, s), err_msg=f"{kind} {rows}x{cols} w={w} {s}")
