"""GPU tests of the sharded paths on ONE device.

* ``shard.CudaBackend`` driven band by band for G in {2, 4, 8} emulated row
  bands: ssb_sat_prepare's band column totals, ssb_band_carry (the exclusive
  scan over bands), ssb_sat_finish with the carry row, and the fused windows on
  band + halo -- the CUDA half of the multi-rank step (shard.py), with the
  collectives replaced by stacking the bands' vectors on the one device.
  Concatenated tables and windows must equal the oracle's whole-image results
  (integral.py:109-116, :141-163; parallel.py:80-134).
* ``ssb_sharded_swa`` (single process, several devices) with the same device
  listed several times, so its peer-copy halo exchange and totals gather run
  as device-local copies.
* the public ``swa(..., devices=...)`` for host and device rasters.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import random_values
from oracle import satsweep_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch

    assert torch.cuda.is_available()
    from paper_2410_16291_b200 import _lib, build_ext

    build_ext.build()
    _lib.load()
    import paper_2410_16291_b200 as mod

    return mod


def _img(kind, shape, seed):
    rng = np.random.default_rng(seed)
    if kind == "i32":
        return rng.integers(-(2**20), 2**20, size=shape, dtype=np.int64).astype(np.int32)
    return random_values(rng, *shape, kind)


def _close(kind, got, ref, rtol=1e-9):
    if kind == "f32":
        np.testing.assert_allclose(got, ref, rtol=rtol, atol=0)
    else:
        np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("kind", ["u8", "u16", "i32", "f32"])
def test_cuda_backend_emulated_bands(sb, G, kind):
    import torch

    from paper_2410_16291_b200 import shard
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    rows, cols, w = 1203, 2050, 37
    img = _img(kind, (rows, cols), G * 31 + len(kind))
    ek = ElemKind.from_dtype(img.dtype)
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(img.view(np.int16) if kind == "u16" else img).to(dev)
    if kind == "u16":
        x = x.view(torch.uint16)
    owned = shard.window_input_bands(rows, w, 1, G)
    need = shard.window_needed_rows(rows, w, 1, G)
    outp = shard.output_partition(rows - w + 1, G)
    backends = [shard.CudaBackend(dev) for _ in range(G)]
    # every band in its own buffer, as on separate ranks (TMA staging needs 16-byte aligned rows)
    own_x = [x[a:b].clone() for a, b in owned]
    need_x = [x[a:b].clone() for a, b in need]
    states, tots = [], []
    for g, (a, b) in enumerate(owned):
        st = backends[g].band_totals(own_x[g], ek, False)
        states.append(st)
        tots.append(st["tot"].clone())
    gathered = torch.stack(tots)  # the all-gather, on one device
    stats = (StatKind.SUM, StatKind.MEAN) if kind != "f32" else (StatKind.SUM, StatKind.STD)
    tables, outs = [], {s: [] for s in stats}
    for g, (a, b) in enumerate(owned):
        carry = backends[g].carry(gathered, g) if g > 0 else None
        tab, ld = backends[g].finish(own_x[g], ek, states[g], carry, None, False)
        tables.append(tab[: b - a + (1 if g == G - 1 else 0)].clone())
        lo, hi = outp[g]
        if hi > lo:
            res = backends[g].window(need_x[g], ek, w, 1, stats, "fused")
            for s in stats:
                outs[s].append(res[s].clone())
    torch.cuda.synchronize()
    acc = np.float64 if kind == "f32" else (np.int64 if kind == "i32" else np.uint64)
    full = np.concatenate([t.cpu().numpy().view(acc)[:, : cols + 1] for t in tables])
    _close(kind, full, O.build_table(img), rtol=1e-12)
    for s in stats:
        got = torch.cat(outs[s]).cpu().numpy()
        ref = O.swa(img, w, s.value)
        if ref.dtype == np.uint64:
            got = got.view(np.uint64)
        _close(kind, got, ref, rtol=1e-6)


@pytest.mark.parametrize("ndev", [1, 2, 3, 8])
@pytest.mark.parametrize("kind", ["u8", "f32"])
def test_sharded_swa_same_device_repeated(sb, ndev, kind):
    """ssb_sharded_swa over devs = [0] * ndev: global table + windows == oracle."""
    import torch

    from paper_2410_16291_b200 import multidev
    from paper_2410_16291_b200.grid import ImageGrid, StatKind

    rows, cols, w = 777, 1501, 64
    img = _img(kind, (rows, cols), ndev)
    x = torch.from_numpy(img).to("cuda:0")
    stats = [StatKind.SUM, StatKind.MEAN] + ([StatKind.STD] if kind == "f32" else [])
    res, table = multidev.swa_device(ImageGrid(x), w, stats, [0] * ndev, with_table=True)
    torch.cuda.synchronize()
    _close(kind, table.to_host(), O.build_table(img), rtol=1e-12)
    for s in stats:
        got = res[s].cpu().numpy()
        ref = O.swa(img, w, s.value)
        if ref.dtype == np.uint64:
            got = got.view(np.uint64)
        _close(kind, got, ref, rtol=1e-6)


def test_sharded_tiny_bands(sb):
    """More devices than output rows: empty bands still own rows / pass their totals on."""
    import torch

    from paper_2410_16291_b200 import multidev
    from paper_2410_16291_b200.grid import ImageGrid, StatKind

    img = _img("u8", (40, 300), 5)
    x = torch.from_numpy(img).to("cuda:0")
    res, table = multidev.swa_device(ImageGrid(x), 38, [StatKind.SUM], [0] * 5, with_table=True)
    np.testing.assert_array_equal(res[StatKind.SUM].cpu().numpy().view(np.uint64), O.swa(img, 38, "sum"))
    np.testing.assert_array_equal(table.to_host(), O.build_table(img))


@pytest.mark.parametrize("devices", [[0], [0, 0], "all"])
def test_public_swa_devices(sb, devices):
    """swa(..., devices=...) -- host rasters (banded ssb_swa_host per device) and CUDA rasters."""
    import torch

    img = _img("u16", (901, 1333), 9)
    for stride in (1, 3):
        got = sb.swa(img, 21, "std", stride=stride, devices=devices)
        np.testing.assert_array_equal(got, O.swa(img, 21, "std", stride))
    d = torch.from_numpy(img.view(np.int16)).to("cuda:0").view(torch.uint16)
    got = sb.swa(d, 21, "mean", devices=devices)
    np.testing.assert_array_equal(got.cpu().numpy(), O.swa(img, 21, "mean"))
    st = sb.swa_stats(img, 21, ("sum", "mean"), devices=devices)
    np.testing.assert_array_equal(st["sum"], O.swa(img, 21, "sum"))


def test_build_sat_devices(sb):
    import torch

    from paper_2410_16291_b200 import multidev
    from paper_2410_16291_b200.grid import ImageGrid

    img = _img("u8", (1000, 3000), 3)
    t = multidev.build_sat_devices(ImageGrid(torch.from_numpy(img).to("cuda:0")), [0, 0, 0, 0])
    np.testing.assert_array_equal(t.to_host(), O.build_table(img))


def test_sharded_swa_validation(sb):
    import ctypes

    from paper_2410_16291_b200 import _lib

    lib = _lib.load()
    P = ctypes.c_void_p
    devs = (ctypes.c_int * 1)(0)
    one = (P * 1)(None)
    assert lib.ssb_sharded_swa(1, devs, _lib.U8, 10, 10, 11, _lib.SUM, one, None, 12, one, None, None, 1, None, None,
                               one) == _lib.EINVAL
    assert lib.ssb_sharded_swa(1, devs, 9, 10, 10, 3, _lib.SUM, one, None, 12, one, None, None, 8, None, None,
                               one) == _lib.EUNSUPPORTED


def test_swa_table_sharded_single_rank(sb):
    """bench.py's multi-GPU step (shard.swa_table_sharded with the CUDA backend)
    on one rank: the windows on the side stream and the table rows equal the
    oracle; a second call reuses every buffer."""
    import torch

    from paper_2410_16291_b200 import shard
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    img = _img("u8", (1500, 2100), 21)
    dev = torch.device("cuda", 0)
    storage, view = shard.band_storage(1500, 2100, 64, 1, torch.uint8, dev)
    view.copy_(torch.from_numpy(img))
    be = shard.CudaBackend(dev)
    for _ in range(2):
        wr, tr = shard.swa_table_sharded(view, 1500, 2100, ElemKind.U8, 64, (StatKind.SUM,), be, storage=storage)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(wr.values[StatKind.SUM].cpu().numpy().view(np.uint64), O.swa(img, 64, "sum"))
    assert tr.rows == (0, 1500)
    np.testing.assert_array_equal(tr.values["table"].cpu().numpy().view(np.uint64)[:, :2101], O.build_table(img))
