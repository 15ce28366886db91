"""The persistent column-strip sweep (sat_strip.cu): the integral image and the
window sums of ssb_sat_build_swa for uint8 rasters at least 42,624 columns wide
(w <= 256, sums, 8-byte aligned rows).  Tables and windows against the oracle
(integral.py:109-116, :141-163), ragged last strips and row steps, w from 1 to
256, R == w, and the concurrent pair (SSB_SWA_PATH=pair) as a second opinion."""

from __future__ import annotations

import numpy as np
import pytest

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


@pytest.mark.parametrize("R,C,w,p", [(300, 50000, 256, 1.0), (271, 43008, 17, 1.0), (33, 85000, 33, 0.5),
                                     (256, 45000, 256, 1.0), (517, 60000, 1, 1.0), (100, 46000, 100, 0.02),
                                     (1040, 44000, 255, 1.0)])
def test_strip_sweep_matches_oracle(sb, R, C, w, p):
    import torch

    from paper_2410_16291_b200 import _engine, _lib
    from paper_2410_16291_b200.grid import ElemKind, StatKind

    rng = np.random.default_rng(R * 7 + w)
    if p < 1.0:
        img = (rng.random((R, C)) < p).astype(np.uint8)
    else:
        img = rng.integers(0, 256, (R, C), dtype=np.uint8)
    lib = _lib.load()
    ld = _engine.sat_ld_for(C)
    assert lib.ssb_sat_swa_supported(_lib.U8, w, _lib.SUM) == 1
    x = torch.from_numpy(img).to("cuda:0")
    sat, ld2, outs = _engine.table_and_sweep(x, ElemKind.U8, R, C, w, (StatKind.SUM,), torch.device("cuda", 0))
    torch.cuda.synchronize()
    assert ld2 == ld
    np.testing.assert_array_equal(sat.cpu().numpy().view(np.uint64)[:, : C + 1], O.build_table(img))
    np.testing.assert_array_equal(outs[StatKind.SUM].cpu().numpy().view(np.uint64), O.swa(img, w, "sum"))


def test_strip_census(sb):
    """Every table entry and every output position stored exactly once by the strip sweep."""
    rng = np.random.default_rng(5)
    v = rng.integers(0, 256, (70, 43008), dtype=np.uint8)
    census = sb.WriteCensus()
    win = sb.WindowSpec(9)
    sb.swa_parallel(sb.ImageGrid(v), win, sb.StatKind.SUM, sb.ParallelConfig(census=census))
    for phase, total in [("rows/sum", 70), ("cols/sum", 43008), ("query/sum", 62)]:
        census.assert_disjoint_cover(phase, total)
