"""Shared test helpers.

Markers: ``gpu`` tests need a B200 and the built libsatsweep_b200.so; they must
fail (not skip) when the library is missing on a GPU box.  Everything else runs
on the CPU.  The oracle (oracle/) is the checker; golden vectors under
tests/golden/ pin the oracle to the reference implementation.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"
EPS = float(np.finfo(np.float64).eps)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built shared library")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN / "golden.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def hashes():
    return json.loads((GOLDEN / "hashes.json").read_text())


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(0xC0FFEE)


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(f"{a.dtype.str}{a.shape}".encode())
    h.update(a.tobytes())
    return h.hexdigest()


def random_values(rng, rows, cols, kind: str):
    """Same draws as the reference tests' random_grid (pkg/tests/conftest.py:15-20)."""
    if kind in ("u8", "u16"):
        dt = np.uint8 if kind == "u8" else np.uint16
        return rng.integers(0, int(np.iinfo(dt).max) + 1, size=(rows, cols), dtype=dt)
    return rng.random(size=(rows, cols), dtype=np.float32)


def stat_atol(stat: str, values: np.ndarray, w: int) -> float:
    """Absolute noise floor for f64-accumulated F32 paths (pkg/tests/conftest.py:23-43)."""
    if values.dtype.kind in "ui":
        return 0.0
    scale = max(1.0, float(np.abs(values).max()))
    rc = values.shape[0] * values.shape[1]
    if stat == "sum":
        return 4.0 * rc * EPS * scale
    if stat == "mean":
        return 4.0 * rc * EPS * scale / (w * w)
    return float(np.sqrt(8.0 * rc * EPS)) * scale


def assert_matches(actual, expected, values: np.ndarray, stat: str, w: int, rtol: float | None = None) -> None:
    """Exact for integer inputs (sum, mean and std are bit-exact on this path); rtol + atol for F32.

    F32 tolerance: rtol 1e-6 (BASELINE north_star, fp64 accumulation) plus the
    reference's derived atol floor."""
    actual = np.asarray(actual)
    expected = np.asarray(expected)
    assert actual.shape == expected.shape
    if values.dtype.kind in "ui":
        if stat == "sum":
            assert actual.dtype.kind in "ui" and expected.dtype.kind in "ui"
            np.testing.assert_array_equal(actual.view(np.uint64), expected.astype(np.uint64, copy=False))
        else:
            assert actual.dtype == np.float64
            np.testing.assert_array_equal(actual, expected)
        return
    np.testing.assert_allclose(actual.astype(np.float64), expected.astype(np.float64),
                               rtol=1e-6 if rtol is None else rtol, atol=stat_atol(stat, values, w))
