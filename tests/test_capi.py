"""The C-ABI shared library loads and exports every symbol include/satsweep_b200.h
declares; argument validation works without a GPU (no compute calls here)."""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import REPO
from paper_2410_16291_b200 import _lib, build_ext

HEADER = REPO / "include" / "satsweep_b200.h"


def declared_symbols() -> list[str]:
    return sorted(set(re.findall(r"\b(ssb_\w+)\s*\(", HEADER.read_text())))


@pytest.fixture(scope="module")
def lib():
    build_ext.build()
    return _lib.load()


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_every_symbol_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version(lib):
    assert lib.ssb_abi_version() == 1


def test_workspace_and_plan(lib):
    ws = lib.ssb_sat_workspace_bytes(_lib.U8, 70000, 85000, 0)
    assert 0 < ws < 512 * 2**20  # carry vectors are ~1/50 of the table
    info = (ctypes.c_int64 * 4)()
    assert lib.ssb_sat_plan(_lib.U8, 70000, 85000, 0, info) == 0
    tw, sr, nj, nk = list(info)
    assert tw == 512 and nj * tw >= 85001 and nk * sr >= 70001
    assert lib.ssb_sat_workspace_bytes(99, 10, 10, 0) == -1


def test_validation_without_device(lib):
    # window larger than the grid: rejected before any CUDA call
    rc = lib.ssb_window_eval(None, None, _lib.U8, 4, 4, 6, 5, 1, _lib.SUM, None, None, None, 1, None)
    assert rc == _lib.EINVAL and b"exceeds grid dims" in lib.ssb_last_error()
    rc = lib.ssb_window_fused(None, _lib.I32, 8, 8, 8, 3, _lib.STD, None, None, None, 6, None, 0, None)
    assert rc == _lib.EUNSUPPORTED
    rc = lib.ssb_window_sum_at(None, 0, 4, 4, 6, 3, 0, 2, None, None)
    assert rc == _lib.EINVAL and b"does not lie within" in lib.ssb_last_error()
    rc = lib.ssb_window_eval_multi(None, None, _lib.U8, 8, 8, 10, 0, None, _lib.SUM, None, None, None, None, None)
    assert rc == _lib.EINVAL
    with pytest.raises(_lib.InvalidWindowError):
        _lib.check(lib.ssb_window_eval(None, None, _lib.U8, 4, 4, 6, 0, 1, _lib.SUM, None, None, None, 1, None))


def test_table_and_windows_contract(lib):
    """ssb_sat_build_swa's request matrix (integer rasters, sum/mean, w <= 257, u16 sums in
    32 bits) and its validation, all without a device."""
    S = _lib.load().ssb_sat_swa_supported
    assert S(_lib.U8, 1, _lib.SUM) == 1 and S(_lib.U8, 257, _lib.SUM | _lib.MEAN) == 1
    assert S(_lib.U8, 258, _lib.SUM) == 0
    assert S(_lib.U16, 256, _lib.SUM) == 1 and S(_lib.U16, 257, _lib.SUM) == 0
    assert S(_lib.I32, 200, _lib.MEAN) == 1
    assert S(_lib.F32, 10, _lib.SUM) == 0 and S(_lib.U8, 10, _lib.STD) == 0 and S(99, 10, _lib.SUM) == 0
    assert lib.ssb_sat_swa_workspace_bytes(_lib.U8, 70000, 85000) >= lib.ssb_sat_workspace_bytes(_lib.U8, 70000,
                                                                                                 85000, 0)
    assert lib.ssb_sat_swa_workspace_bytes(_lib.F32, 10, 10) == -1
    info = (ctypes.c_int64 * 4)()
    assert lib.ssb_sat_swa_plan(_lib.U8, 70000, 85000, 256, info) == 0
    nj_w, sr, nk, m = list(info)
    assert nj_w * 1024 >= 85001 and sr * nk >= 70001 and m >= 1
    for fn in (lib.ssb_sat_build_swa, lib.ssb_sat_build_swa_onepass):
        rc = fn(None, _lib.F32, 8, 8, 8, None, 10, 3, _lib.SUM, None, None, 6, None, 0, None)
        assert rc == _lib.EUNSUPPORTED
        rc = fn(None, _lib.U8, 8, 8, 8, None, 10, 9, _lib.SUM, None, None, 6, None, 0, None)
        assert rc == _lib.EINVAL and b"exceeds grid dims" in lib.ssb_last_error()


@pytest.mark.parametrize("rows,w,n", [(100, 7, 4), (9, 9, 3), (12, 11, 3), (70000, 256, 8), (5, 1, 8), (61, 9, 2)])
def test_sharded_plan_matches_host_geometry(lib, rows, w, n):
    """ssb_sharded_plan (pure host) == shard.py's geometry (the reference's partition
    rule over output rows, parallel.py:80-90): owned rows partition [0, rows);
    the needed rows are the band plus its (w-1)-row halo."""
    from paper_2410_16291_b200 import shard

    buf = (ctypes.c_int64 * (7 * n))()
    assert lib.ssb_sharded_plan(rows, 40 if w <= 40 else w, w, n, buf) == 0
    v = list(buf)
    own = shard.window_input_bands(rows, w, 1, n)
    need = shard.window_needed_rows(rows, w, 1, n)
    out = shard.output_partition(rows - w + 1, n)
    for g in range(n):
        own_lo, own_hi, need_lo, need_hi, out_lo, out_hi, cap = v[7 * g:7 * g + 7]
        assert (own_lo, own_hi) == own[g]
        assert (out_lo, out_hi) == out[g]
        if out_hi > out_lo:
            assert (need_lo, need_hi) == need[g]
            assert cap >= need_hi - own_lo
        assert cap >= own_hi - own_lo


def test_sharded_validation_without_device(lib):
    assert lib.ssb_sharded_plan(10, 10, 11, 2, (ctypes.c_int64 * 14)()) == _lib.EINVAL
    assert lib.ssb_sharded_workspace_bytes(_lib.U8, 10, 10, 3, 2, 5, 1) == -1
    assert lib.ssb_band_carry(None, 1, 10, 10, 0, None, None) == _lib.EINVAL


def test_host_widen_and_wire_settings(lib):
    """The host half of ssb_swa_host's narrow wire (host_widen.cpp) needs no device:
    zero-extension of uint16 / uint32 into uint64 at every alignment and length, and
    the wire / thread settings round-trip."""
    import numpy as np

    rng = np.random.default_rng(16)
    for bits, dt in ((16, np.uint16), (32, np.uint32)):
        src = rng.integers(0, 2**bits, size=5000, dtype=np.uint64).astype(dt)
        src[:4] = [0, 2**bits - 1, 2**(bits - 1), 1]  # the top bit must not sign-extend
        for off_s, off_d, n in ((0, 0, 5000), (1, 0, 4097), (3, 1, 1023), (2, 3, 7), (5, 2, 0), (0, 1, 1), (7, 5, 64)):
            dst = np.full(off_d + n + 9, 0xA5A5A5A5A5A5A5A5, dtype=np.uint64)
            s = np.ascontiguousarray(src[off_s:off_s + n])
            rc = lib.ssb_host_widen(s.ctypes.data_as(ctypes.c_void_p), bits, ctypes.c_void_p(dst.ctypes.data + 8 * off_d), n)
            assert rc == 0
            assert np.array_equal(dst[off_d:off_d + n], s.astype(np.uint64))
            assert (dst[:off_d] == 0xA5A5A5A5A5A5A5A5).all() and (dst[off_d + n:] == 0xA5A5A5A5A5A5A5A5).all()
    one = np.zeros(1, np.uint64)
    assert lib.ssb_host_widen(one.ctypes.data_as(ctypes.c_void_p), 8, one.ctypes.data_as(ctypes.c_void_p), 1) == _lib.EINVAL
    assert lib.ssb_host_wire(-1) == 0 and lib.ssb_host_wire(32) == 0 and lib.ssb_host_wire(7) == 32
    assert lib.ssb_host_wire(64) == 32 and lib.ssb_host_wire(0) == 64 and lib.ssb_host_wire(-1) == 0
    assert lib.ssb_host_threads(-1) == 0 and lib.ssb_host_threads(5) == 0 and lib.ssb_host_threads(0) == 5
