"""Seeded randomized parity sweep of the public API against the oracle (-m gpu).

Each case draws a shape, dtype, window(s), stride, statistic and pipeline and
compares the device result with the CPU oracle: integer results bit-exact,
float results within rtol 1e-6 (north_star) plus the reference's atol floor.
Host (numpy) and device (CUDA tensor) inputs are both exercised, as are
multi-window sets with more windows than one kernel launch takes (8).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_matches, random_values
from oracle import satsweep_oracle as O

pytestmark = pytest.mark.gpu

N_CASES = 200


@pytest.fixture(scope="module")
def sb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2410_16291_b200 as mod
    from paper_2410_16291_b200 import _lib, build_ext

    build_ext.build()
    _lib.load()
    return mod


def _case(i):
    rng = np.random.default_rng(1_000_003 * (i + 1))
    kind = ("u8", "u16", "f32")[i % 3]
    rows = int(rng.integers(1, 700))
    cols = int(rng.integers(1, 900))
    w = int(rng.integers(1, min(rows, cols) + 1))
    stride = 1 if rng.random() < 0.6 else int(rng.integers(1, 2 * w + 2))
    stat = ("sum", "mean", "std")[int(rng.integers(0, 3))]
    pipeline = ("auto", "table", "fused")[int(rng.integers(0, 3))]
    on_device = bool(rng.random() < 0.5)
    v = random_values(rng, rows, cols, kind)
    return v, w, stride, stat, pipeline, on_device


def _to_host(x, dtype):
    if hasattr(x, "is_cuda"):
        from paper_2410_16291_b200 import _device

        return _device.to_host(x, dtype)
    return x


@pytest.mark.parametrize("i", range(N_CASES))
def test_swa_random(sb, i):
    v, w, stride, stat, pipeline, on_device = _case(i)
    if pipeline == "fused" and stride != 1:
        pipeline = "table"
    x = v
    if on_device:
        import torch

        from paper_2410_16291_b200 import _device

        x = _device.to_device(v, torch.device("cuda", 0))
    got = sb.swa(x, w, stat, stride=stride, pipeline=pipeline)
    ref = O.swa(v, w, stat, stride)
    got = _to_host(got, ref.dtype)
    assert got.shape == ref.shape and got.dtype == ref.dtype
    assert_matches(got, ref, v, stat, w)


@pytest.mark.parametrize("i", range(40))
def test_multi_window_random(sb, i):
    rng = np.random.default_rng(7919 * (i + 1))
    kind = ("u8", "u16", "f32")[i % 3]
    rows, cols = int(rng.integers(40, 600)), int(rng.integers(40, 800))
    n = int(rng.integers(1, 12))  # beyond 8 windows the C ABI groups the launches
    ws = [int(t) for t in rng.integers(1, min(rows, cols) + 1, size=n)]
    stat = ("sum", "mean", "std")[i % 3]
    v = random_values(rng, rows, cols, kind)
    got = sb.multi_window(v, ws, stat)
    ref = O.multi_window(v, ws, stat)
    assert len(got) == len(ref)
    for g, r, w in zip(got, ref, ws):
        assert_matches(g, r, v, stat, w)
