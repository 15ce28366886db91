"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Integer results bit-exact; F32 within rtol 1e-6
plus the reference's derived atol floor (conftest.assert_matches)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_matches, digest, random_values
from oracle import satsweep_oracle as O

pytestmark = pytest.mark.gpu

KINDS = ("u8", "u16", "f32")
PIPES = ("table", "fused")


@pytest.fixture(scope="module")
def sb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2410_16291_b200 import _lib, build_ext

    build_ext.build()
    _lib.load()
    import paper_2410_16291_b200 as mod

    return mod


def to_dev(a):
    import torch

    from paper_2410_16291_b200 import _device

    return _device.to_device(a, torch.device("cuda", 0))


def host(t, dtype):
    from paper_2410_16291_b200 import _device

    return _device.to_host(t, dtype)


# ---------------------------------------------------------------- tables
def test_hand_tables(sb, golden):
    img = sb.ImageGrid(golden["hand_in"])
    sat = sb.build_sat(img)
    assert sat.table.tolist() == [[0, 0, 0], [0, 1, 3], [0, 4, 10]]
    assert sat.accum_kind is sb.AccumKind.U64 and sat.source_dims == (2, 2)
    assert sb.build_sat(img, squared=True).table.tolist() == [[0, 0, 0], [0, 1, 5], [0, 10, 30]]
    assert sb.build_sat(sb.ImageGrid(np.zeros((4, 5), np.uint16))).table.tolist() == np.zeros((5, 6), int).tolist()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("sq", [False, True])
def test_random_tables(sb, golden, kind, sq):
    v = golden[f"rand_{kind}_in"]
    ref = golden[f"rand_{kind}_sat{'_sq' if sq else ''}"]
    got = sb.build_sat(sb.ImageGrid(v), squared=sq).table
    if kind == "f32":
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-9)
    else:
        np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("shape", [(1, 1), (1, 700), (700, 1), (33, 513), (513, 33), (1025, 1537), (3000, 2049)])
@pytest.mark.parametrize("kind", ["u8", "u16", "i32", "f32"])
def test_tables_vs_oracle_shapes(sb, shape, kind):
    rng = np.random.default_rng(hash((shape, kind)) % 2**32)
    if kind == "i32":
        v = rng.integers(-(2**31), 2**31, size=shape, dtype=np.int64).astype(np.int32)
    else:
        v = random_values(rng, *shape, kind)
    for sq in (False, True) if kind != "i32" else (False,):
        got = sb.build_sat(sb.ImageGrid(v), squared=sq).table
        ref = O.build_table(v, sq)
        if kind == "f32":
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-9 * max(1, shape[0] * shape[1]))
        elif ref.dtype == object:
            assert got.tolist() == ref.tolist()
        else:
            np.testing.assert_array_equal(got.view(ref.dtype), ref)


def test_zero_border_and_monotone(sb, rng):
    for kind in KINDS:
        v = random_values(rng, 31, 12, kind)
        for sq in (False, True):
            t = np.asarray(sb.build_sat(sb.ImageGrid(v), squared=sq).table, dtype=np.float64)
            assert (t[0] == 0).all() and (t[:, 0] == 0).all()
            assert (np.diff(t, axis=0) >= 0).all() and (np.diff(t, axis=1) >= 0).all()


def test_window_sum(sb, golden, rng):
    sat = sb.build_sat(sb.ImageGrid(golden["hand_in"]))
    assert sb.window_sum(sat, 0, 0, 2) == 10 and sb.window_sum(sat, 0, 1, 1) == 2
    for top, left, w in [(1, 0, 2), (0, 1, 2), (-1, 0, 1), (0, -1, 1), (0, 0, 3)]:
        with pytest.raises(sb.InvalidWindowError):
            sb.window_sum(sat, top, left, w)
    arr = rng.integers(0, 65536, size=(20, 20), dtype=np.uint16)
    s = sb.build_sat(sb.ImageGrid(arr))
    q = sb.build_sat(sb.ImageGrid(arr), squared=True)
    for top, left, w in [(0, 0, 20), (3, 5, 7), (12, 0, 8), (19, 19, 1)]:
        assert int(sb.window_sum(s, top, left, w)) == int(arr[top:top + w, left:left + w].astype(np.uint64).sum())
    for i in range(6):
        for j in range(7):
            assert sb.window_sum(q, i, j, 1) == int(arr[i, j]) ** 2


# ---------------------------------------------------------------- window statistics
@pytest.mark.parametrize("kind", KINDS)
def test_swa_golden_cases(sb, golden, kind):
    for ci, (r, c, w, s) in enumerate(golden["cases"].tolist()):
        v = golden[f"case{ci}_{kind}_in"]
        img = sb.ImageGrid(v)
        for stat in ("sum", "mean", "std"):
            ref = golden[f"case{ci}_{kind}_{stat}"]
            got = sb.swa_integral(img, sb.WindowSpec(w, s), sb.StatKind(stat)).values
            assert got.dtype == ref.dtype
            assert_matches(got, ref, v, stat, w)
            if s == 1:
                fused = sb.swa(v, w, stat, pipeline="fused")
                assert_matches(fused, ref, v, stat, w)


def test_wide_numerator_std(sb, golden):
    v = golden["wide_u16_in"]
    for pipe in PIPES:
        got = sb.swa(v, 300, "std", pipeline=pipe)
        np.testing.assert_array_equal(got, golden["wide_u16_std"])


def test_std_examples(sb):
    assert sb.swa(np.array([[0, 2], [0, 2]], np.uint8), 2, "std").tolist() == [[1.0]]
    arr = np.full((12, 12), 9, dtype=np.uint16)
    for w in (1, 3, 5):
        for pipe in PIPES:
            np.testing.assert_array_equal(sb.swa(arr, w, "std", pipeline=pipe), np.zeros((12 - w + 1,) * 2))


def _window_mean(x: np.ndarray, w: int) -> np.ndarray:
    t = np.zeros((x.shape[0] + 1, x.shape[1] + 1))
    t[1:, 1:] = x.cumsum(0).cumsum(1)
    return (t[w:, w:] - t[:-w, w:] - t[w:, :-w] + t[:-w, :-w]) / (w * w)


def test_float_std_edges(sb):
    """Float std's finalisation (the reference's mean = s/n, var = q/n - mean^2
    with correctly rounded divisions; sqrt from the rsqrt estimate of
    var + 2^-1000 and one Newton step): constant windows of exactly summable
    values give exactly 0 (not NaN, not a residue), as the reference does;
    every other case -- the smallest / largest float32 magnitudes, constant
    windows whose reference sums carry rounding noise, and windows whose
    one-pass variance cancels -- agrees with the reference within the rtol
    contract measured against the size of the terms, sqrt(mean(x^2)), plus
    the table arithmetic's own noise floor: the reference's one-pass formula
    over running sums (integral.py:141-163, stats.py:70-74) is accurate only
    to that scale, so a result at noise level is compared at noise level."""
    rng = np.random.default_rng(77)
    cases = [np.full((40, 70), v, dtype=np.float32) for v in (0.0, 1.0, 3.0e-38, 1.4e-45, 3.0e38 / 64, 1234.5678)]
    cases += [(1000.0 + rng.random((60, 90)) * 0.1).astype(np.float32),   # var / E[x^2] ~ 1e-8
              (rng.random((60, 90)) * 1e-30).astype(np.float32),
              (10.0 ** rng.uniform(-30, 30, (60, 90))).astype(np.float32)]
    for k, arr in enumerate(cases):
        # the table pipelines (the reference's and ours) difference running sums
        # of squares that reach sum(x^2): their var carries an absolute
        # rounding noise of ~eps * sum(x^2), so std agrees to sqrt of that
        noise = 8.0 * np.sqrt(np.finfo(np.float64).eps * (arr.astype(np.float64) ** 2).sum())
        for w in (1, 4, 9):
            ref = O.swa(arr, w, "std")
            scale = np.sqrt(np.maximum(_window_mean(arr.astype(np.float64) ** 2, w), 0.0))  # cumsum noise can dip < 0
            for pipe in PIPES:
                got = sb.swa(arr, w, "std", pipeline=pipe)
                assert np.isfinite(got).all() and (got >= 0).all(), (k, w, pipe)
                bad = np.abs(got - ref) > 1e-6 * scale + noise
                assert not bad.any(), (k, w, pipe, np.argwhere(bad)[:3].tolist(), got[bad][:3], ref[bad][:3], noise)
                if k < 2:  # 0.0 and 1.0: every window sum is exact -> std exactly 0
                    assert not got.any(), (k, w, pipe)


def test_multi_window(sb, golden):
    v = golden["mw_in"]
    for stat in ("sum", "mean", "std"):
        for w, got in zip((5, 50, 150), sb.multi_window(v, [5, 50, 150], stat)):
            np.testing.assert_array_equal(got, golden[f"mw_{stat}_{w}"])
    a, b = sb.multi_window(v, [7, 7], "sum")
    np.testing.assert_array_equal(a, b)


def test_acceptance_sweep(sb, hashes):
    """210 seeded images x 3 stats x 2 pipelines (pkg/tests/test_acceptance.py:37-74)."""
    rng = np.random.default_rng(20240817)
    for rec in hashes["acceptance"]:
        rows, cols = int(rng.integers(rec["w"], 257)), int(rng.integers(rec["w"], 257))
        assert (rows, cols) == (rec["rows"], rec["cols"])
        v = random_values(rng, rows, cols, rec["kind"])
        w, s = rec["w"], rec["stride"]
        for stat in ("sum", "mean", "std"):
            got = sb.swa(v, w, stat, stride=s, pipeline="table")
            if rec["kind"] == "f32":
                assert_matches(got, O.swa(v, w, stat, s), v, stat, w)
            else:
                assert digest(got) == rec[stat], rec
            if s == 1:
                fz = sb.swa(v, w, stat, pipeline="fused")
                if rec["kind"] == "f32":
                    assert_matches(fz, O.swa(v, w, stat, s), v, stat, w)
                else:
                    assert digest(fz) == rec[stat], rec


@pytest.mark.parametrize("pipe", PIPES)
def test_random_shapes_vs_oracle(sb, pipe):
    rng = np.random.default_rng(7777)
    for _ in range(40):
        kind = KINDS[int(rng.integers(0, 3))]
        rows, cols = int(rng.integers(1, 700)), int(rng.integers(1, 2200))
        w = int(rng.integers(1, min(rows, cols) + 1))
        v = random_values(rng, rows, cols, kind)
        for stat in ("sum", "mean", "std"):
            got = sb.swa(v, w, stat, pipeline=pipe)
            assert_matches(got, O.swa(v, w, stat), v, stat, w)


def test_int32_extension(sb):
    rng = np.random.default_rng(2)
    v = rng.integers(-(2**31), 2**31, size=(300, 400), dtype=np.int64).astype(np.int32)
    for pipe in PIPES:
        for stat in ("sum", "mean"):
            got = sb.swa(v, 17, stat, pipeline=pipe)
            ref = O.swa(v, 17, stat)
            assert got.dtype == ref.dtype
            np.testing.assert_array_equal(got, ref)
    with pytest.raises(TypeError):
        sb.swa(v, 3, "std")


def test_device_tensor_in_device_tensor_out(sb):
    rng = np.random.default_rng(9)
    v = random_values(rng, 257, 300, "u16")
    d = to_dev(v)
    for pipe in PIPES:
        out = sb.swa(d, 31, "mean", pipeline=pipe)
        assert out.is_cuda
        np.testing.assert_array_equal(host(out, np.float64), O.swa(v, 31, "mean"))
    res = sb.swa_stats(d, 31, ("sum", "mean", "std"))
    np.testing.assert_array_equal(host(res["sum"], np.uint64), O.swa(v, 31, "sum"))
    np.testing.assert_array_equal(host(res["std"], np.float64), O.swa(v, 31, "std"))


# ---------------------------------------------------------------- API contract
def test_api_contract(sb):
    import hashlib

    rng = np.random.default_rng(13)
    arr = rng.integers(0, 65536, size=(50, 50), dtype=np.uint16)
    before = hashlib.sha256(arr.tobytes()).hexdigest()
    for method in ("naive", "dp", "integral", "parallel"):
        sb.swa(arr, 7, "std", method)
    assert hashlib.sha256(arr.tobytes()).hexdigest() == before
    big = rng.integers(0, 256, size=(20, 40), dtype=np.uint8)
    view = big[:, ::2]
    np.testing.assert_array_equal(sb.swa(view, 3, "sum", "integral"), sb.swa(np.ascontiguousarray(view), 3))
    ones = np.ones((4, 4), dtype=np.uint8)
    out = sb.swa(ones, 1, "sum")
    assert out.dtype == np.uint64 and (out.base is None or out.base is not ones)
    out[0, 0] = 99
    assert ones[0, 0] == 1
    arr = rng.integers(0, 65536, size=(33, 29), dtype=np.uint16)
    res = [sb.swa(arr, 5, "sum", m, stride=2) for m in ("naive", "dp", "integral", "parallel")]
    for r in res[1:]:
        np.testing.assert_array_equal(res[0], r)


def test_nonfinite_rejected(sb):
    bad = np.ones((16, 16), dtype=np.float32)
    bad[3, 4] = np.nan
    for pipe in PIPES:
        with pytest.raises(sb.GridValidationError):
            sb.swa(bad, 3, "mean", pipeline=pipe)
    bad[3, 4] = np.inf
    with pytest.raises(sb.GridValidationError):
        sb.swa_stats(to_dev(bad), 3, ("sum",), pipeline="table")


def test_parallel_census_and_identity(sb, rng):
    census = sb.WriteCensus()
    v = random_values(rng, 41, 29, "u16")
    win = sb.WindowSpec(7, 2)
    cfg = sb.ParallelConfig(workers=4, min_parallel_elems=1, census=census)
    par = sb.swa_parallel(sb.ImageGrid(v), win, sb.StatKind.STD, cfg)
    np.testing.assert_array_equal(par.values, sb.swa_integral(sb.ImageGrid(v), win, sb.StatKind.STD).values)
    out_r, _ = sb.output_dims(41, 29, win)
    for phase, total in [("rows/sum", 41), ("cols/sum", 29), ("rows/sq", 41), ("cols/sq", 29),
                         ("query/sum", out_r), ("query/sq", out_r)]:
        census.assert_disjoint_cover(phase, total)


@pytest.mark.parametrize("kind,w,s,stat,shape", [("u8", 9, 1, "sum", (300, 517)), ("u8", 17, 1, "mean", (300, 517)),
                                                ("f32", 6, 1, "std", (300, 517)), ("f32", 6, 2, "std", (300, 517)),
                                                ("u16", 5, 3, "sum", (300, 517)),
                                                ("i32", 4, 1, "mean", (300, 517)),
                                                ("u8", 64, 1, "sum", (4100, 4100))])  # >= 2^24 px: fused windows
def test_device_census_exactly_once(sb, rng, kind, w, s, stat, shape):
    """The census is written by the kernels (one atomic per stored table entry /
    output position): every table row, column and output row is covered exactly
    once on every pipeline the parallel entry points take (parallel.py:35-51,
    pkg/tests/test_parallel.py:90-118)."""
    R, C = shape
    if kind == "i32":
        v = rng.integers(-1000, 1000, size=(R, C)).astype(np.int32)
    else:
        v = random_values(rng, R, C, kind)
    census = sb.WriteCensus()
    cfg = sb.ParallelConfig(census=census)
    win = sb.WindowSpec(w, s)
    sb.swa_parallel(sb.ImageGrid(v), win, sb.StatKind(stat), cfg)
    out_r, _ = sb.output_dims(R, C, win)
    # float windows of stride 1, w <= 256 take the fused kernel: no table phases
    table = not (kind == "f32" and s == 1 and w <= 256)
    phases = [("query/sum", out_r)] + ([("rows/sum", R), ("cols/sum", C)] if table else [])
    if stat == "std":
        phases += [("query/sq", out_r)] + ([("rows/sq", R), ("cols/sq", C)] if table else [])
    if not table:
        assert "rows/sum" not in census.ranges
    for phase, total in phases:
        census.assert_disjoint_cover(phase, total)
    c2 = sb.WriteCensus()
    sb.build_sat_parallel(sb.ImageGrid(v), False, sb.ParallelConfig(census=c2))
    c2.assert_disjoint_cover("rows/sum", R)
    c2.assert_disjoint_cover("cols/sum", C)


def test_device_census_sees_double_writes(sb, rng):
    """Two builds inside one census window store every entry twice: the check must fail."""
    import torch

    from paper_2410_16291_b200.parallel import _DeviceCensus

    v = random_values(rng, 64, 80, "u8")
    img = sb.ImageGrid(v)
    census = sb.WriteCensus()
    with _DeviceCensus(census, img) as dc:
        sb.build_sat(img)
        sb.build_sat(img)
    torch.cuda.synchronize()
    dc.record_table(["sum"])
    with pytest.raises(AssertionError):
        census.assert_disjoint_cover("rows/sum", 64)
    # and a multi-window sweep counts each window's rows in its own block
    from paper_2410_16291_b200 import _device, _engine, _lib
    import ctypes

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    x = to_dev(v)
    sat, _, ld = _engine.build_tables(x, sb.ElemKind.U8, 64, 80, dev, squared=False)
    ws = [5, 9]
    outs = [_device.empty((64 - w + 1, 80 - w + 1), np.uint64, dev, "o") for w in ws]
    cnt = torch.zeros(sum(64 - w + 1 for w in ws), dtype=torch.int64, device=dev)
    _lib.check(lib.ssb_census_enable(None, 0, None, 0, cnt.data_ptr(), cnt.numel()))
    arr = lambda t, vals: (t * 2)(*vals)  # noqa: E731
    _lib.check(lib.ssb_window_eval_multi(sat.data_ptr(), None, _lib.U8, 64, 80, ld, 2, arr(ctypes.c_int64, ws), _lib.SUM,
                                         arr(ctypes.c_void_p, [o.data_ptr() for o in outs]), None, None,
                                         arr(ctypes.c_int64, [80 - w + 1 for w in ws]), _device.stream_ptr(dev)))
    lib.ssb_census_disable()
    c = cnt.cpu().numpy()
    assert (c[:60] == 76).all() and (c[60:] == 72).all()


def test_host_streaming_bands(sb):
    """ssb_swa_host with several bands equals one-shot evaluation (offsets cancel per band)."""
    from paper_2410_16291_b200 import _engine

    rng = np.random.default_rng(21)
    for kind in KINDS:
        v = random_values(rng, 611, 333, kind)
        img = sb.ImageGrid(v)
        for pipe in PIPES:
            for stride in (1, 3) if pipe == "table" else (1,):
                one = _engine.run_host(img, 40, stride, [sb.StatKind.SUM, sb.StatKind.STD], pipe)
                many = _engine.run_host(img, 40, stride, [sb.StatKind.SUM, sb.StatKind.STD], pipe, band_rows=37)
                for k in one:
                    if kind == "f32":
                        np.testing.assert_allclose(many[k], one[k], rtol=1e-9, atol=1e-9)
                    else:
                        np.testing.assert_array_equal(many[k], one[k])


def test_reference_seams(sb, rng):
    """seams.builder / seams.sweep behind the reference's builder/sweep signatures
    (integral.py:166-189), driven like _sats_for_stat/_finalize_from_sats would."""
    from types import SimpleNamespace

    from paper_2410_16291_b200 import seams

    for kind in KINDS:
        v = random_values(rng, 97, 131, kind)
        img = SimpleNamespace(values=v, elem_kind=None)
        win = SimpleNamespace(w=9, stride=2)
        sat = seams.builder(img, False)
        np.testing.assert_array_equal(sat.table, O.build_table(v)) if kind != "f32" else \
            np.testing.assert_allclose(sat.table, O.build_table(v), rtol=1e-12)
        out_r, out_c = O.out_shape(97, 131, 9, 2)
        ref = O.corner_sums(O.build_table(v), 9, 2, out_r, out_c)
        for table in (sat, SimpleNamespace(table=O.build_table(v))):
            got = seams.sweep(table, win, out_r, out_c)
            if kind == "f32":
                np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-9)
            else:
                np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("shape,w,stride", [((1, 1), 1, 1), ((1, 4097), 1, 1), ((4097, 1), 1, 3), ((3, 70001), 3, 1),
                                            ((5000, 7), 7, 1), ((33, 33), 33, 1), ((257, 300), 256, 1),
                                            ((700, 701), 5, 9), ((4000, 3300), 3200, 1), ((300, 300), 17, 17)])
def test_edge_shapes(sb, shape, w, stride):
    """Degenerate and ragged shapes: 1-pixel images, single rows/columns, w = min dim,
    stride > w, windows wider than the fused path (table fallback)."""
    rng = np.random.default_rng(sum(shape) + w)
    for kind in ("u8", "u16", "f32"):
        v = random_values(rng, *shape, kind)
        for stat in ("sum", "std"):
            got = sb.swa(v, w, stat, stride=stride)
            assert_matches(got, O.swa(v, w, stat, stride), v, stat, w)


def test_unaligned_device_view(sb):
    """A row-slice view whose data pointer is not 16-byte aligned is handled (copied once)."""
    rng = np.random.default_rng(3)
    v = random_values(rng, 41, 37, "u8")
    d = to_dev(v)
    view = d[1:]  # offset 37 bytes
    assert view.data_ptr() % 16 != 0
    for pipe in PIPES:
        got = host(sb.swa(view, 5, "sum", pipeline=pipe), np.uint64)
        np.testing.assert_array_equal(got, O.swa(v[1:], 5, "sum"))


def test_capi_rejects_unaligned_raster(sb):
    from paper_2410_16291_b200 import _lib

    lib = _lib.load()
    d = to_dev(np.zeros((8, 40), np.uint8))
    rc = lib.ssb_window_fused(d.data_ptr() + 1, _lib.U8, 4, 40, 40, 3, _lib.SUM, d.data_ptr(), None, None, 38, None, 0,
                              None)
    assert rc == _lib.EINVAL and b"aligned" in lib.ssb_last_error()


def test_capi_table_writers_reject_pitch_2_mod_4(sb):
    """Table rows are written with 256-bit stores: a pitch of 2 mod 4 elements
    (cols + 1 rounded up to even, e.g. C5's 85,002) or a table that is not
    32-byte aligned is refused with SSB_EINVAL before any launch, and the
    context stays usable (no misaligned-address fault)."""
    import torch

    from paper_2410_16291_b200 import _device, _engine, _lib

    lib = _lib.load()
    R, C = 37, 85  # cols + 1 = 86 = 2 mod 4
    v = np.random.default_rng(11).integers(0, 256, (R, C), dtype=np.uint8)
    x = to_dev(v)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    bad_ld = C + 1
    assert bad_ld % 4 == 2
    sat = _device.empty(((R + 1) * 90,), np.uint64, dev, "t")
    wsb = max(int(lib.ssb_sat_workspace_bytes(_lib.U8, R, C, 0)), int(lib.ssb_sat_swa_workspace_bytes(_lib.U8, R, C)),
              int(lib.ssb_sat_lookback_workspace_bytes(_lib.U8, R, C, 0)))
    ws = _device.empty((wsb,), np.uint8, dev, "ws")
    out = _device.empty((R - 4, C - 4), np.uint64, dev, "o")
    calls = {
        "build": lambda ld, p: lib.ssb_sat_build(x.data_ptr(), _lib.U8, R, C, C, p, None, ld, None, None,
                                                 ws.data_ptr(), wsb, None, st),
        "finish": lambda ld, p: lib.ssb_sat_finish(x.data_ptr(), _lib.U8, R, C, C, p, None, ld, None, None,
                                                   ws.data_ptr(), wsb, st),
        "lookback": lambda ld, p: lib.ssb_sat_build_lookback(x.data_ptr(), _lib.U8, R, C, C, p, None, ld, None, None,
                                                             ws.data_ptr(), wsb, st),
        "swa": lambda ld, p: lib.ssb_sat_build_swa(x.data_ptr(), _lib.U8, R, C, C, p, ld, 5, _lib.SUM, out.data_ptr(),
                                                   None, C - 4, ws.data_ptr(), wsb, st),
    }
    for name, fn in calls.items():
        assert fn(bad_ld, sat.data_ptr()) == _lib.EINVAL, name
        assert b"multiple of 4" in lib.ssb_last_error(), name
        assert fn(88, sat.data_ptr() + 16) == _lib.EINVAL, name  # 16- but not 32-byte aligned
        assert b"32-byte" in lib.ssb_last_error(), name
    # the rounded pitch works and the context is healthy
    ld = _engine.sat_ld_for(C)
    assert ld % 4 == 0
    assert calls["build"](ld, sat.data_ptr()) == _lib.OK
    torch.cuda.synchronize()
    got = host(sat[: (R + 1) * ld].view(R + 1, ld), np.uint64)[:, : C + 1]
    np.testing.assert_array_equal(got, O.build_table(v))


def test_concurrent_threads(sb):
    """The facade is reentrant: concurrent callers get correct, independent results."""
    import threading

    rng = np.random.default_rng(8)
    imgs = [random_values(rng, 300 + 7 * k, 290, "u16") for k in range(6)]
    refs = [O.swa(v, 11, "mean") for v in imgs]
    errs = []

    def work(k):
        try:
            for _ in range(3):
                np.testing.assert_array_equal(sb.swa(imgs[k], 11, "mean", pipeline="table"), refs[k])
        except Exception as exc:  # pragma: no cover
            errs.append(exc)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


# ---------------------------------------------------------------- single-pass look-back build
@pytest.mark.parametrize("shape", [(1, 1), (1, 700), (700, 1), (129, 513), (127, 511), (1025, 1537), (3001, 4099)])
@pytest.mark.parametrize("kind", ["u8", "u16", "i32"])
def test_lookback_build_matches_oracle(sb, shape, kind):
    """ssb_sat_build_lookback (single pass, decoupled look-back) vs the oracle:
    plain, squared-only and both tables, with and without a carry row."""
    import torch

    from paper_2410_16291_b200 import _device, _engine, _lib

    lib = _lib.load()
    rng = np.random.default_rng(hash(("lb", shape, kind)) % 2**32)
    R, C = shape
    if kind == "i32":
        v = rng.integers(-(2**31), 2**31, size=shape, dtype=np.int64).astype(np.int32)
    else:
        v = random_values(rng, R, C, kind)
    code = {"u8": _lib.U8, "u16": _lib.U16, "i32": _lib.I32}[kind]
    x = to_dev(v)
    ld = _engine.sat_ld_for(C)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    carry_h = rng.integers(0, 2**63, size=C + 1, dtype=np.uint64)
    modes = [(True, False), (False, True), (True, True)] if kind != "i32" else [(True, False)]
    for plain, sq in modes:
        for with_carry in (False, True):
            sat = _device.empty((R + 1, ld), np.uint64, dev, "t") if plain else None
            sat_sq = _device.empty((R + 1, ld), np.uint64, dev, "t") if sq else None
            wsb = int(lib.ssb_sat_lookback_workspace_bytes(code, R, C, 1 if sq else 0))
            ws = _device.empty((wsb,), np.uint8, dev, "ws")
            carry = to_dev(carry_h.view(np.int64)) if with_carry else None
            ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
            _lib.check(lib.ssb_sat_build_lookback(x.data_ptr(), code, R, C, C, ptr(sat), ptr(sat_sq), ld, ptr(carry),
                                                  ptr(carry), ws.data_ptr(), wsb, st))
            torch.cuda.synchronize()
            for tab, squared in ((sat, False), (sat_sq, True)):
                if tab is None:
                    continue
                ref = O.build_table(v, squared).astype(np.uint64)
                if with_carry:
                    ref = ref + carry_h[None, :]  # wraps modulo 2^64 like the device table
                got = host(tab, np.uint64)[:, : C + 1]
                np.testing.assert_array_equal(got, ref)


def test_lookback_build_refuses_float(sb):
    from paper_2410_16291_b200 import _lib

    lib = _lib.load()
    rc = lib.ssb_sat_build_lookback(None, _lib.F32, 4, 4, 4, None, None, 6, None, None, None, 0, None)
    assert rc == _lib.EUNSUPPORTED


@pytest.mark.parametrize("kind", ["u8", "u16"])
def test_lookback_build_large_matches_two_pass(sb, kind):
    """12,000 x 30,001: thousands of tiles in flight, long look-back chains; bit-identical to the default build."""
    import torch

    from paper_2410_16291_b200 import _device, _engine, _lib

    lib = _lib.load()
    R, C = 12000, 30001
    rng = np.random.default_rng(7)
    v = rng.integers(0, 256 if kind == "u8" else 65536, size=(R, C), dtype=np.uint8 if kind == "u8" else np.uint16)
    code = _lib.U8 if kind == "u8" else _lib.U16
    x = to_dev(v)
    ld = _engine.sat_ld_for(C)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream().cuda_stream
    wsb = max(int(lib.ssb_sat_workspace_bytes(code, R, C, 0)), int(lib.ssb_sat_lookback_workspace_bytes(code, R, C, 0)))
    ws = _device.empty((wsb,), np.uint8, dev, "ws")
    a = _device.empty((R + 1, ld), np.uint64, dev, "t")
    b = _device.empty((R + 1, ld), np.uint64, dev, "t")
    _lib.check(lib.ssb_sat_build(x.data_ptr(), code, R, C, C, a.data_ptr(), None, ld, None, None, ws.data_ptr(), wsb,
                                 None, st))
    _lib.check(lib.ssb_sat_build_lookback(x.data_ptr(), code, R, C, C, b.data_ptr(), None, ld, None, None,
                                          ws.data_ptr(), wsb, st))
    torch.cuda.synchronize()
    assert torch.equal(a[:, : C + 1], b[:, : C + 1])


def test_division_by_n_is_ieee(sb):
    """The finalisation divides by n = w*w with a reciprocal multiply + FMA
    correction; it must give the IEEE quotient bit for bit (stats.py:55-74 divide
    with numpy's IEEE '/').  Integer window sums (every magnitude class, incl.
    > 2^53), random doubles and f32 sums, for w = 1..300 and a few huge n."""
    import torch

    from paper_2410_16291_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(99)
    ints = np.concatenate([np.arange(0, 200000, dtype=np.float64),
                           rng.integers(0, 2**62, 200000).astype(np.float64),
                           (rng.integers(0, 2**53, 200000)).astype(np.float64),
                           -rng.integers(0, 2**40, 100000).astype(np.float64)])
    floats = np.concatenate([rng.random(200000) * 10.0 ** rng.integers(-30, 30, 200000),
                             rng.lognormal(0, 1, 200000) * 4096.0])
    x = torch.from_numpy(np.concatenate([ints, floats])).to("cuda:0")
    bad = torch.zeros(1, dtype=torch.int64, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    ns = [w * w for w in range(1, 301)] + [10000, 4096, 65536 * 3 + 1, 3071 * 3071, 2**40 + 3]
    for n in ns:
        _lib.check(lib.ssb_selftest_division(x.data_ptr(), x.numel(), float(n), bad.data_ptr(), st))
    torch.cuda.synchronize()
    assert int(bad.item()) == 0


@pytest.mark.parametrize("w", [9, 64, 300])
def test_float_methods_agree_bitwise(sb, w):
    """Every entry point routes a float window the same way (the fused kernel
    for stride 1, w <= 256; the table otherwise), so swa / swa_integral /
    swa_parallel / multi_window agree bit for bit, as the reference's methods
    do (pkg/tests/test_api.py:68-79)."""
    rng = np.random.default_rng(w)
    v = rng.lognormal(0.0, 1.0, (700, 900)).astype(np.float32)
    img = sb.ImageGrid(v)
    for stat in ("sum", "mean", "std"):
        a = sb.swa(v, w, stat)
        b = sb.swa_integral(img, sb.WindowSpec(w), sb.StatKind(stat)).values
        c = sb.swa_parallel(img, sb.WindowSpec(w), sb.StatKind(stat)).values
        d = sb.multi_window(v, [5, w, 301], stat)[1]
        e = sb.swa(to_dev(v), w, stat).cpu().numpy()
        for other in (b, c, d, e):
            np.testing.assert_array_equal(a, other)
        np.testing.assert_allclose(a, O.swa(v, w, stat), rtol=1e-6, atol=0)
