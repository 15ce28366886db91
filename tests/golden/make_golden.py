"""Generate the golden vectors that pin the oracle and the GPU path.

Runs the REFERENCE implementation (`satsweep`, imported from
/root/reference/pkg/src) -- only possible in the survey/build container,
never on the GPU box -- and writes:

  golden.npz    small inputs/outputs (hand tables, random tables, swa cases)
  hashes.json   sha256 of reference outputs too large to commit (C1..C5 and
                the acceptance-style 210-image sweep), plus sampled rows of
                the float configs for tolerance checks

Usage:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import satsweep as ss  # noqa: E402  (the reference)

from paper_2410_16291_b200 import synthetic  # noqa: E402

KINDS = (ss.ElemKind.U8, ss.ElemKind.U16, ss.ElemKind.F32)


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(f"{a.dtype.str}{a.shape}".encode())
    h.update(a.tobytes())
    return h.hexdigest()


def random_values(rng, rows, cols, kind):
    """Same draws as the reference tests' random_grid (tests/conftest.py:15-20)."""
    if kind.is_integer:
        return rng.integers(0, int(kind.max_value) + 1, size=(rows, cols), dtype=kind.dtype)
    return rng.random(size=(rows, cols), dtype=np.float32)


def small(out: dict) -> None:
    rng = np.random.default_rng(0xC0FFEE)
    hand = np.array([[1, 2], [3, 4]], dtype=np.uint8)
    out["hand_in"] = hand
    out["hand_sat"] = ss.build_sat(ss.ImageGrid(hand)).table.astype(np.uint64)
    out["hand_sat_sq"] = ss.build_sat(ss.ImageGrid(hand), squared=True).table.astype(np.uint64)
    for kind in KINDS:
        v = random_values(rng, 17, 23, kind)
        out[f"rand_{kind.value}_in"] = v
        for sq in (False, True):
            t = ss.build_sat(ss.ImageGrid(v), squared=sq).table
            out[f"rand_{kind.value}_sat{'_sq' if sq else ''}"] = t
    cases = [(8, 8, 1, 1), (40, 25, 3, 1), (64, 64, 16, 16), (80, 61, 50, 1), (50, 50, 50, 1),
             (33, 29, 5, 2), (61, 44, 9, 4), (37, 53, 7, 3)]
    for kind in KINDS:
        for ci, (r, c, w, s) in enumerate(cases):
            v = random_values(rng, r, c, kind)
            out[f"case{ci}_{kind.value}_in"] = v
            for stat in ss.StatKind:
                res = ss.swa_integral(ss.ImageGrid(v), ss.WindowSpec(w, s), stat).values
                out[f"case{ci}_{kind.value}_{stat.value}"] = res
    out["cases"] = np.array(cases, dtype=np.int64)
    # wide-numerator std (tests/test_integral.py:165-174)
    v = random_values(rng, 310, 305, ss.ElemKind.U16)
    out["wide_u16_in"] = v
    out["wide_u16_std"] = ss.swa_integral(ss.ImageGrid(v), ss.WindowSpec(300), ss.StatKind.STD).values
    # max-value u16 squared peak (erratum: SPEC.md:194; value from tests/test_integral.py:64-73)
    out["peak_u16_sq"] = np.array([9 * 65535**2], dtype=np.uint64)
    # constant and tiny std examples
    out["std_example"] = ss.swa(np.array([[0, 2], [0, 2]], dtype=np.uint8), 2, "std")
    # multi-window (all stats, small enough to store)
    v = ss.generate("random", 200, 220, ss.ElemKind.U16, seed=2024).values
    out["mw_in"] = v
    for stat in ("sum", "mean", "std"):
        for w, r in zip((5, 50, 150), ss.multi_window(v, [5, 50, 150], stat)):
            out[f"mw_{stat}_{w}"] = r


def acceptance_sweep(hashes: dict) -> None:
    """Hashes of the reference on the acceptance-style sweep (tests/test_acceptance.py:37-74)."""
    rng = np.random.default_rng(20240817)
    windows = (1, 2, 3, 16, 50)
    recs = []
    checked = 0
    while checked < 210:
        for kind in KINDS:
            w = int(windows[checked % len(windows)])
            stride = 1 if (checked // len(windows)) % 2 == 0 else w
            rows = int(rng.integers(w, 257))
            cols = int(rng.integers(w, 257))
            v = random_values(rng, rows, cols, kind)
            rec = {"kind": kind.value, "rows": rows, "cols": cols, "w": w, "stride": stride}
            for stat in ss.StatKind:
                rec[stat.value] = digest(ss.swa_integral(ss.ImageGrid(v), ss.WindowSpec(w, stride), stat).values)
            recs.append(rec)
            checked += 1
    hashes["acceptance"] = recs


def big(hashes: dict, out: dict) -> None:
    t0 = time.time()
    x = synthetic.c1()
    hashes["C1_sum_w50"] = digest(ss.swa(x, 50, "sum"))
    x = synthetic.c2()
    assert 0 <= x.min() and x.max() <= 65535
    x16 = x.astype(np.uint16)
    hashes["C2_sum_w100"] = digest(ss.swa(x16, 100, "sum"))
    hashes["C2_mean_w100"] = digest(ss.swa(x16, 100, "mean"))
    print("C1/C2", time.time() - t0, flush=True)
    x = synthetic.c4()
    rows_pick = np.array([0, 1234, 9999, 19936], dtype=np.int64)
    out["C4_rows"] = rows_pick
    for stat in ("mean", "std"):
        r = ss.swa(x, 64, stat)
        hashes[f"C4_{stat}_w64"] = digest(r)
        out[f"C4_{stat}_rows"] = r[rows_pick]
        del r
    del x
    print("C4", time.time() - t0, flush=True)
    x = synthetic.c3()
    for w in (25, 50, 100, 200, 400):
        hashes[f"C3_sum_w{w}"] = digest(ss.swa(x, w, "sum"))
    del x
    print("C3", time.time() - t0, flush=True)
    w = 256
    for lo, hi in ((0, 2048), (34000, 34512), (69745 - 512, 69745)):
        band = synthetic.c5(lo, hi + w - 1)
        hashes[f"C5_sum_w256_rows{lo}_{hi}"] = digest(ss.swa(band, w, "sum"))
    print("C5 bands", time.time() - t0, flush=True)


def main() -> None:
    out: dict = {}
    hashes: dict = {"reference": "satsweep " + ss.__version__, "numpy": np.__version__}
    small(out)
    acceptance_sweep(hashes)
    if "--big" in sys.argv:
        big(hashes, out)
    else:
        old = HERE / "hashes.json"
        if old.exists():  # keep previously generated big-config hashes
            prev = json.loads(old.read_text())
            for k, v in prev.items():
                if k.startswith("C"):
                    hashes[k] = v
            prevz = HERE / "golden.npz"
            if prevz.exists():
                with np.load(prevz, allow_pickle=False) as z:
                    for k in z.files:
                        if k.startswith("C4_"):
                            out[k] = z[k]
    np.savez_compressed(HERE / "golden.npz", **out)
    (HERE / "hashes.json").write_text(json.dumps(hashes, indent=1, sort_keys=True))
    print("wrote", HERE / "golden.npz", HERE / "hashes.json")


if __name__ == "__main__":
    main()
