"""Golden outcomes of the reference's file readers (pkg/src/satsweep/imgio.py).

Builds a fixed list of PGM and raw+sidecar files -- valid ones, and one per
error branch of read_pgm / read_sidecar / read_raw / read_raw_result -- runs
the REFERENCE readers on them (only possible in the build container), and
writes imgio_cases.json: the file bytes (base64) plus the outcome, either
(dtype, shape, sha256 of the values) or (exception class, message,
byte_offset).  tests/test_imgio.py replays the cases against the drop-in.

Usage:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_imgio_golden.py
"""

from __future__ import annotations

import base64
import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import satsweep as ss  # noqa: E402  (the reference)
from satsweep import imgio  # noqa: E402


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def pgm_cases() -> list[tuple[str, bytes]]:
    rng = np.random.default_rng(2410)
    u8 = rng.integers(0, 256, size=(7, 13), dtype=np.uint8)
    u16 = rng.integers(0, 65536, size=(5, 9), dtype=np.uint16)
    odd = rng.integers(0, 256, size=(3, 1001), dtype=np.uint8)
    be = u16.astype(">u2").tobytes()
    return [
        ("u8_plain", b"P5\n13 7\n255\n" + u8.tobytes()),
        ("u8_maxval_1", b"P5 13 7 1\n" + (u8 & 1).tobytes()),
        ("u8_comments", b"P5\n# made by hand\n13 # width\n7\n#c\n255\t" + u8.tobytes()),
        ("u8_trailing_bytes", b"P5\n13 7\n255\n" + u8.tobytes() + b"extra"),
        ("u8_leading_zeros", b"P5\n0013 007\n0255\n" + u8.tobytes()),
        ("u8_ragged_wide", b"P5\n1001 3\n200\n" + odd.tobytes()),
        ("u16_plain", b"P5\n9 5\n65535\n" + be),
        ("u16_maxval_256", b"P5\n9 5\n256\r" + be),
        ("bad_magic", b"P2\n13 7\n255\n" + u8.tobytes()),
        ("bad_magic_short", b"P"),
        ("empty_file", b""),
        ("only_magic", b"P5"),
        ("comment_to_eof", b"P5\n# never ends"),
        ("bad_width", b"P5\n1x3 7\n255\n" + u8.tobytes()),
        ("bad_height", b"P5\n13 -7\n255\n" + u8.tobytes()),
        ("bad_maxval", b"P5\n13 7\n25a\n" + u8.tobytes()),
        ("zero_width", b"P5\n0 7\n255\n"),
        ("zero_height", b"P5\n13 0\n255\n"),
        ("maxval_zero", b"P5\n13 7\n0\n" + u8.tobytes()),
        ("maxval_big", b"P5\n13 7\n65536\n" + u8.tobytes()),
        ("maxval_huge", b"P5\n13 7\n99999999999999999999999\n" + u8.tobytes()),
        ("no_ws_after_maxval", b"P5\n13 7\n255"),
        ("comment_after_maxval", b"P5\n13 7\n255#x\n" + u8.tobytes()),
        ("truncated_u8", b"P5\n13 7\n255\n" + u8.tobytes()[:-1]),
        ("truncated_u16", b"P5\n9 5\n65535\n" + be[:-3]),
        ("truncated_empty_payload", b"P5\n13 7\n255\n"),
        ("huge_dims_truncated", b"P5\n123456789012 98765432109\n255\n" + b"\0" * 10),
    ]


def raw_cases() -> list[tuple[str, str, bytes, str]]:
    """(name, reader, raw bytes, sidecar text)"""
    rng = np.random.default_rng(16291)
    u8 = rng.integers(0, 256, size=(6, 11), dtype=np.uint8)
    u16 = rng.integers(0, 65536, size=(4, 5), dtype=np.uint16)
    f32 = rng.random((3, 7), dtype=np.float32)
    u64 = rng.integers(0, 2**63, size=(2, 3), dtype=np.uint64)
    f64 = rng.random((5, 2))

    def side(rows, cols, dtype, endian="little"):
        return json.dumps({"rows": rows, "cols": cols, "dtype": dtype, "endianness": endian}) + "\n"

    bad_f32 = f32.copy()
    bad_f32[1, 2] = np.inf
    return [
        ("raw_u8", "read_raw", u8.tobytes(), side(6, 11, "u8")),
        ("raw_u16", "read_raw", u16.astype("<u2").tobytes(), side(4, 5, "u16")),
        ("raw_f32", "read_raw", f32.astype("<f4").tobytes(), side(3, 7, "f32")),
        ("raw_f32_inf", "read_raw", bad_f32.astype("<f4").tobytes(), side(3, 7, "f32")),
        ("raw_short", "read_raw", u8.tobytes()[:-1], side(6, 11, "u8")),
        ("raw_long", "read_raw", u8.tobytes() + b"\0", side(6, 11, "u8")),
        ("raw_result_dtype", "read_raw", u64.tobytes(), side(2, 3, "u64")),
        ("raw_bad_json", "read_raw", u8.tobytes(), "{rows: 6"),
        ("raw_extra_key", "read_raw", u8.tobytes(), json.dumps({"rows": 6, "cols": 11, "dtype": "u8",
                                                                "endianness": "little", "x": 1})),
        ("raw_missing_key", "read_raw", u8.tobytes(), json.dumps({"rows": 6, "cols": 11, "dtype": "u8"})),
        ("raw_not_object", "read_raw", u8.tobytes(), "[1, 2]"),
        ("raw_big_endian", "read_raw", u8.tobytes(), side(6, 11, "u8", "big")),
        ("raw_unknown_dtype", "read_raw", u8.tobytes(), side(6, 11, "i8")),
        ("raw_zero_rows", "read_raw", b"", side(0, 11, "u8")),
        ("res_u64", "read_raw_result", u64.astype("<u8").tobytes(), side(2, 3, "u64")),
        ("res_f64", "read_raw_result", f64.astype("<f8").tobytes(), side(5, 2, "f64")),
        ("res_image_dtype", "read_raw_result", u8.tobytes(), side(6, 11, "u8")),
        ("res_short", "read_raw_result", u64.tobytes()[:-8], side(2, 3, "u64")),
    ]


def outcome(fn):
    try:
        v = fn()
    except Exception as exc:  # noqa: BLE001 - recording the reference's behaviour
        return {"error": type(exc).__name__, "message": str(exc), "byte_offset": getattr(exc, "byte_offset", None)}
    a = v.values if isinstance(v, ss.ImageGrid) else v
    return {"dtype": a.dtype.str, "shape": list(a.shape), "sha256": digest(a)}


def main():
    cases = []
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        for name, data in pgm_cases():
            p = td / f"{name}.pgm"
            p.write_bytes(data)
            cases.append({"name": name, "reader": "read_pgm", "file": base64.b64encode(data).decode(),
                          "outcome": outcome(lambda: imgio.read_pgm(p))})
        for name, reader, data, side_text in raw_cases():
            rp, sp = td / f"{name}.raw", td / f"{name}.json"
            rp.write_bytes(data)
            sp.write_text(side_text, encoding="utf-8")
            fn = getattr(imgio, reader)
            cases.append({"name": name, "reader": reader, "file": base64.b64encode(data).decode(),
                          "sidecar": side_text, "outcome": outcome(lambda: fn(rp, sp))})
    (HERE / "imgio_cases.json").write_text(json.dumps(cases, indent=1) + "\n")
    print(f"{len(cases)} cases -> {HERE / 'imgio_cases.json'}")


if __name__ == "__main__":
    main()
