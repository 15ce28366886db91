"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  scripts/sanitize.sh runs it
under each tool; results are checked against the oracle so a run is also a
functional check."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2410_16291_b200 as sb  # noqa: E402
from oracle import satsweep_oracle as O  # noqa: E402
from paper_2410_16291_b200 import _device, _engine, _lib, multidev  # noqa: E402
from paper_2410_16291_b200.grid import ElemKind, ImageGrid, StatKind  # noqa: E402

big = "--big" in sys.argv


def check(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f" or b.dtype.kind == "f":
        np.testing.assert_allclose(a.astype(np.float64), b.astype(np.float64), rtol=1e-6, atol=1e-9)
    else:
        np.testing.assert_array_equal(a.view(np.uint64) if a.dtype == np.int64 and b.dtype == np.uint64 else a, b)


def main():
    rng = np.random.default_rng(1)
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    imgs = {
        "u8": rng.integers(0, 256, (203, 1100), dtype=np.uint8),
        "u16": rng.integers(0, 65536, (150, 700), dtype=np.uint16),
        "i32": rng.integers(-1000, 1000, (130, 600)).astype(np.int32),
        "f32": rng.random((140, 650), dtype=np.float32),
    }
    for k, v in imgs.items():
        x = torch.from_numpy(v.view(np.int16) if k == "u16" else v).to(dev)
        if k == "u16":
            x = x.view(torch.uint16)
        for sq in ((False, True) if k != "i32" else (False,)):
            check(sb.build_sat(ImageGrid(x), sq).table, O.build_table(v, sq))  # reduce-then-scan build
        stats = ("sum", "mean") + (("std",) if k != "i32" else ())
        for pipe in ("table", "fused"):
            res = sb.swa_stats(x, 13, stats, pipeline=pipe)  # corner sweep / fused strip kernels
            for st in stats:
                check(_device.to_host(res[st], _engine.result_dtype(ElemKind.from_dtype(v.dtype), StatKind(st))),
                      O.swa(v, 13, st))
        res = sb.swa_stats(x, 7, ("sum",), stride=3, pipeline="table")  # strided corner kernel
        check(_device.to_host(res["sum"], _engine.result_dtype(ElemKind.from_dtype(v.dtype), StatKind.SUM)),
              O.swa(v, 7, "sum", 3))
        outs = sb.multi_window(x, [5, 9, 20], "sum")  # multi-window TMA sweep
        for w, o in zip((5, 9, 20), outs):
            check(_device.to_host(o, _engine.result_dtype(ElemKind.from_dtype(v.dtype), StatKind.SUM)),
                  O.swa(v, w, "sum"))
        if k != "f32":  # single-pass look-back build and the one-pass table+windows kernel
            R, C = v.shape
            code = ElemKind.from_dtype(v.dtype).abi_code
            ld = _engine.sat_ld_for(C)
            t = _device.empty((R + 1, ld), np.uint64, dev, "t")
            wsb = int(lib.ssb_sat_lookback_workspace_bytes(code, R, C, 0))
            ws = _device.empty((wsb,), np.uint8, dev, "ws")
            _lib.check(lib.ssb_sat_build_lookback(x.data_ptr(), code, R, C, C, t.data_ptr(), None, ld, None, None,
                                                  ws.data_ptr(), wsb, _device.stream_ptr(dev)))
            check(_device.to_host(t, np.uint64)[:, : C + 1], O.build_table(v).astype(np.uint64))
            sat, _, outs = _engine.table_and_sweep(x, ElemKind.from_dtype(v.dtype), R, C, 13, (StatKind.SUM,), dev,
                                                   onepass=True)
            check(_device.to_host(outs[StatKind.SUM], np.uint64), O.swa(v, 13, "sum").astype(np.uint64))
    # multi-device orchestration on one device (peer copies, totals gather, carry kernel)
    v = imgs["u8"]
    res, table = multidev.swa_device(ImageGrid(torch.from_numpy(v).to(dev)), 11, [StatKind.SUM], [0, 0, 0],
                                     with_table=True)
    check(res[StatKind.SUM].cpu().numpy(), O.swa(v, 11, "sum").astype(np.uint64))
    check(table.to_host(), O.build_table(v))
    # host streaming path
    check(sb.swa(v, 11, "mean"), O.swa(v, 11, "mean"))
    if big:  # >= 2^24 px: the concurrent table build + fused windows of ssb_sat_build_swa
        vb = (rng.random((4200, 4100)) < 0.3).astype(np.uint8)
        xb = torch.from_numpy(vb).to(dev)
        sat, _, outs = _engine.table_and_sweep(xb, ElemKind.U8, 4200, 4100, 256, (StatKind.SUM,), dev)
        check(_device.to_host(outs[StatKind.SUM], np.uint64)[:50], O.swa(vb[:305], 256, "sum"))
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
