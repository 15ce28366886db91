"""GPU parity of ssb_swa_host's narrow wire format (uint32 sums over PCIe, widened
into the caller's uint64 array by the library's host threads): the same bits as
the straight 64-bit copy and as the CPU oracle (api.py:28-55 returns uint64),
for contiguous and pitched outputs, one and many bands (slot-ring reuse),
sums above 2^31 (zero- not sign-extended) and windows whose sums do not fit."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from oracle import satsweep_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2410_16291_b200 import _lib, build_ext

    build_ext.build()
    handle = _lib.load()
    yield handle
    handle.ssb_host_wire(0)
    handle.ssb_host_release()


def host_sum(lib, img, w, *, band_rows=0, out_ld=None, pipeline=None, mean=False):
    from paper_2410_16291_b200 import _lib

    rows, cols = img.shape
    out_r, out_c = rows - w + 1, cols - w + 1
    ld = out_ld or out_c
    out = np.full((out_r, ld), 0xDEADBEEFDEADBEEF, dtype=np.uint64)
    avg = np.full((out_r, ld), np.nan) if mean else None
    code = {np.dtype(np.uint8): _lib.U8, np.dtype(np.uint16): _lib.U16}[img.dtype]
    vp = lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = lib.ssb_swa_host(vp(img), code, rows, cols, cols, w, 1, _lib.SUM | (_lib.MEAN if mean else 0), vp(out), vp(avg),
                          None, ld, _lib.PIPE_TABLE if pipeline is None else pipeline, 0, band_rows)
    _lib.check(rc, "ssb_swa_host")
    h2d, d2h = ctypes.c_int64(), ctypes.c_int64()
    lib.ssb_host_last_copy_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
    assert (out[:, out_c:] == 0xDEADBEEFDEADBEEF).all(), "pitch padding was written"
    return out[:, :out_c], (None if avg is None else avg[:, :out_c]), h2d.value, d2h.value


@pytest.mark.parametrize("band_rows", [0, 300])
@pytest.mark.parametrize("pitched", [False, True])
def test_narrow_wire_matches_wide_and_oracle_u8(lib, band_rows, pitched):
    from paper_2410_16291_b200 import _lib

    rng = np.random.default_rng(1610)
    img = rng.integers(0, 256, size=(2300, 2411), dtype=np.uint8)
    w = 37
    n = (2300 - w + 1) * (2411 - w + 1)
    ld = 2411 - w + 1 + (5 if pitched else 0)
    ref = O.swa(img, w, "sum")
    for pipe in (_lib.PIPE_TABLE, _lib.PIPE_FUSED):
        lib.ssb_host_wire(0)
        got, _, h2d, d2h = host_sum(lib, img, w, band_rows=band_rows, out_ld=ld, pipeline=pipe)
        assert np.array_equal(got, ref)
        bands = 1 if band_rows == 0 else -(-(2300 - w + 1) // band_rows)  # every band uploads its own w - 1 extra rows
        assert h2d == (2300 - w + 1 + bands * (w - 1)) * 2411
        assert d2h == 4 * n, "the sums must cross PCIe as uint32"
        lib.ssb_host_wire(64)
        wide, _, _, d2h = host_sum(lib, img, w, band_rows=band_rows, out_ld=ld, pipeline=pipe)
        assert np.array_equal(wide, ref) and d2h == 8 * n
    assert lib.ssb_host_wire(0) == 64


def test_narrow_wire_zero_extends_u16_near_2_32(lib):
    """w=256 on saturated uint16: sums up to 256^2 * 65535 = 4,294,901,760 (> 2^31, < 2^32)."""
    lib.ssb_host_wire(0)
    rng = np.random.default_rng(7)
    img = rng.integers(60000, 65536, size=(2300, 2310), dtype=np.uint16)
    img[400:1200, 300:1500] = 65535
    got, _, _, d2h = host_sum(lib, img, 256, band_rows=500)
    ref = O.swa(img, 256, "sum")
    assert got.max() == 256 * 256 * 65535 and np.array_equal(got, ref)
    assert d2h == 4 * got.size


def test_sums_that_do_not_fit_stay_64_bit(lib):
    lib.ssb_host_wire(0)
    img = np.full((2400, 2400), 65535, dtype=np.uint16)
    got, _, _, d2h = host_sum(lib, img, 257, band_rows=700)  # 257^2 * 65535 >= 2^32
    assert d2h == 8 * got.size and (got == 257 * 257 * 65535).all()


def test_narrow_sum_with_wide_mean(lib):
    """SUM narrowed, MEAN copied straight (float64), both from the same bands."""
    lib.ssb_host_wire(0)
    rng = np.random.default_rng(3)
    img = (rng.random((2200, 2300)) < 0.3).astype(np.uint8)
    got, avg, _, d2h = host_sum(lib, img, 50, band_rows=256, mean=True)
    assert np.array_equal(got, O.swa(img, 50, "sum"))
    assert np.array_equal(avg, O.swa(img, 50, "mean"))
    assert d2h == 10 * got.size  # sums <= 2500: uint16 on the wire; means float64


def test_uint16_wire_per_band(lib):
    """A band whose largest sum is below 2^16 leaves as uint16, the others as uint32 (decided per band
    from the device-computed maximum); ssb_host_wire(32) keeps every band at uint32."""
    rng = np.random.default_rng(5)
    img = (rng.random((2600, 2500)) < 0.2).astype(np.uint8)
    img[1500:1900, 700:1400] = 255  # sums far above 65535 in the bands that see this block
    w, br = 40, 400
    ref = O.swa(img, w, "sum")
    out_r, out_c = ref.shape
    lib.ssb_host_wire(0)
    got, _, _, d2h = host_sum(lib, img, w, band_rows=br)
    assert np.array_equal(got, ref)
    expect = sum((min(out_r, lo + br) - lo) * out_c * (2 if ref[lo:lo + br].max() < 65536 else 4)
                 for lo in range(0, out_r, br))
    assert 2 * ref.size < expect < 4 * ref.size and d2h == expect
    # exactly 65535 still fits (one zero in every 256 x 256 window), 65536 does not
    edge = np.ones((2304, 2304), dtype=np.uint8)
    edge[::256, ::256] = 0
    got, _, _, d2h = host_sum(lib, edge, 256, band_rows=600)
    assert (got == 65535).all() and d2h == 2 * got.size
    one = np.ones((2400, 2400), dtype=np.uint8)
    got, _, _, d2h = host_sum(lib, one, 256, band_rows=500)  # every sum == 65536: one above uint16
    assert (got == 65536).all() and d2h == 4 * got.size
    one[::7, ::5] = 0
    got, _, _, d2h = host_sum(lib, one, 255, band_rows=500)  # <= 65025
    assert np.array_equal(got, O.swa(one, 255, "sum")) and d2h == 2 * got.size
    assert lib.ssb_host_wire(32) == 0
    got, _, _, d2h = host_sum(lib, img, w, band_rows=br)
    assert np.array_equal(got, ref) and d2h == 4 * ref.size
    assert lib.ssb_host_wire(0) == 32


def test_public_api_host_arrays(lib):
    """swa(numpy) -> numpy uint64 through the narrow wire equals the oracle; repeated calls reuse the ring."""
    import paper_2410_16291_b200 as sb

    lib.ssb_host_wire(0)
    rng = np.random.default_rng(11)
    img = (rng.random((2500, 2600)) < 0.05).astype(np.uint8)
    ref = O.swa(img, 64, "sum")
    for _ in range(3):
        got = sb.swa(img, 64, "sum")
        assert got.dtype == np.uint64 and np.array_equal(got, ref)


def test_two_concurrent_calls_share_the_cores(lib):
    """swa(numpy, devices=[0, 0]): two ssb_swa_host calls at once, each narrow, each with its own ring."""
    import paper_2410_16291_b200 as sb

    lib.ssb_host_wire(0)
    rng = np.random.default_rng(12)
    img = rng.integers(0, 256, size=(3700, 2600), dtype=np.uint8)
    got = sb.swa(img, 64, "sum", devices=[0, 0])
    assert np.array_equal(got, O.swa(img, 64, "sum"))
    assert lib.ssb_host_threads(-1) == 0, "the per-call thread share must be restored"


def test_sums_to_host_and_multi_window(lib):
    """ssb_sums_to_host (device sums -> host uint64 through the narrow wire) against a plain copy, for
    bounds on either side of 2^32 and 2^16, and multi_window(numpy) through it against the oracle."""
    import torch

    import paper_2410_16291_b200 as sb

    lib.ssb_host_wire(0)
    rng = np.random.default_rng(44)
    h2d, d2h = ctypes.c_int64(), ctypes.c_int64()
    for rows, cols, hi in ((2500, 2301, 60000), (2500, 2301, 3_000_000_000), (33, 40, 100), (4097, 1025, 70000), (9001, 4000, 60000)):
        vals = rng.integers(0, hi, size=(rows, cols), dtype=np.uint64)
        dev = torch.from_numpy(vals.view(np.int64)).cuda()
        for bound in (hi, 0, 2**40):
            for ld in (cols, cols + 3):
                out = np.full((rows, ld), 7, dtype=np.uint64)
                rc = lib.ssb_sums_to_host(dev.data_ptr(), rows, cols, bound, out.ctypes.data, ld,
                                          torch.cuda.current_stream().cuda_stream)
                assert rc == 0
                assert np.array_equal(out[:, :cols], vals) and (out[:, cols:] == 7).all()
                lib.ssb_host_last_copy_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
                narrow = bound == hi and rows * cols >= 1 << 22
                width = 8 if not narrow else (2 if hi <= 65536 else 4)
                assert d2h.value == rows * cols * width, (rows, cols, hi, bound, d2h.value)
    img = (rng.random((2600, 2500)) < 0.1).astype(np.uint8)
    ws = [25, 60, 300]
    for pipe in ("auto", "table", "fused"):
        got = sb.multi_window(img, ws, "sum", pipeline=pipe)
        for g, w in zip(got, ws):
            assert g.dtype == np.uint64 and np.array_equal(g, O.swa(img, w, "sum"))
    got = sb.multi_window(img, ws, "mean")  # float64 results: through the ring as they are
    for g, w in zip(got, ws):
        assert g.dtype == np.float64 and np.array_equal(g, O.swa(img, w, "mean"))


def test_pageable_float_results_take_the_ring(lib):
    """float64 mean / std bound for pageable arrays go through the pinned ring in 8-byte chunks (copied,
    not widened): bit-identical to the straight copy, same bytes over PCIe, pitched or not, several bands."""
    from paper_2410_16291_b200 import _lib

    rng = np.random.default_rng(8)
    img = rng.lognormal(0.0, 1.0, size=(2300, 2400)).astype(np.float32)
    w = 33
    out_r, out_c = 2300 - w + 1, 2400 - w + 1
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    res = {}
    for bits in (0, 64):
        lib.ssb_host_wire(bits)
        for ld, br in ((out_c, 0), (out_c + 3, 500)):
            mean = np.full((out_r, ld), -1.0)
            std = np.full((out_r, ld), -1.0)
            rc = lib.ssb_swa_host(vp(img), _lib.F32, 2300, 2400, 2400, w, 1, _lib.MEAN | _lib.STD, None, vp(mean), vp(std),
                                  ld, _lib.PIPE_FUSED, 0, br)
            _lib.check(rc, "ssb_swa_host")
            h2d, d2h = ctypes.c_int64(), ctypes.c_int64()
            lib.ssb_host_last_copy_bytes(ctypes.byref(h2d), ctypes.byref(d2h))
            assert d2h.value == 16 * out_r * out_c
            assert (mean[:, out_c:] == -1.0).all() and (std[:, out_c:] == -1.0).all()
            res[bits, ld] = (mean[:, :out_c].copy(), std[:, :out_c].copy())
    lib.ssb_host_wire(0)
    for ld in (out_c, out_c + 3):
        assert np.array_equal(res[0, ld][0], res[64, ld][0]) and np.array_equal(res[0, ld][1], res[64, ld][1])
    np.testing.assert_allclose(res[0, out_c][0], O.swa(img, w, "mean"), rtol=1e-6)
    np.testing.assert_allclose(res[0, out_c][1], O.swa(img, w, "std"), rtol=1e-6, atol=1e-9)
