"""ctypes binding of libsatsweep_b200.so (the C ABI in include/satsweep_b200.h).

The library is the only compute path: if it is missing or no CUDA device is
present, calls fail loudly -- there is no CPU fallback.  ctypes releases the
GIL for the duration of every foreign call, so concurrent callers from
several threads run concurrently, as the reference's numpy kernels did
(pkg/src/satsweep/api.py:1-9).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import GridValidationError, InvalidWindowError, ResourceLimitError, SatsweepError

LIB_PATH = Path(os.environ["SSB_LIB"]) if os.environ.get("SSB_LIB") else (
    Path(__file__).resolve().parent / "libsatsweep_b200.so")  # SSB_LIB: tuning builds only

# status codes / enums (include/satsweep_b200.h)
OK, EINVAL, ECUDA, ENOMEM, EUNSUPPORTED, ENONFINITE = 0, 1, 2, 3, 4, 5
U8, U16, I32, F32 = 0, 1, 2, 3
SUM, MEAN, STD = 1, 2, 4
PIPE_TABLE, PIPE_FUSED = 0, 1

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_SIGS = {
    "ssb_abi_version": (_int, []),
    "ssb_last_error": (ctypes.c_char_p, []),
    "ssb_launch_count": (_i64, []),
    "ssb_window_fused_max_w": (_i64, []),
    "ssb_sat_workspace_bytes": (_i64, [_int, _i64, _i64, _int]),
    "ssb_sat_plan": (_int, [_int, _i64, _i64, _int, ctypes.POINTER(_i64)]),
    "ssb_sat_prepare": (_int, [_vp, _int, _i64, _i64, _i64, _int, _vp, _i64, _vp, _vp, _vp, _vp]),
    "ssb_sat_finish": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp]),
    "ssb_sat_build": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp]),
    "ssb_sat_lookback_workspace_bytes": (_i64, [_int, _i64, _i64, _int]),
    "ssb_sat_build_lookback": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp]),
    "ssb_sat_swa_supported": (_int, [_int, _i64, _int]),
    "ssb_sat_swa_workspace_bytes": (_i64, [_int, _i64, _i64]),
    "ssb_sat_swa_plan": (_int, [_int, _i64, _i64, _i64, ctypes.POINTER(_i64)]),
    "ssb_sat_build_swa": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _i64, _i64, _int, _vp, _vp, _i64, _vp, _i64, _vp]),
    "ssb_sat_build_swa_onepass": (
        _int, [_vp, _int, _i64, _i64, _i64, _vp, _i64, _i64, _int, _vp, _vp, _i64, _vp, _i64, _vp]),
    "ssb_window_eval": (_int, [_vp, _vp, _int, _i64, _i64, _i64, _i64, _i64, _int, _vp, _vp, _vp, _i64, _vp]),
    "ssb_window_eval_multi": (
        _int,
        [_vp, _vp, _int, _i64, _i64, _i64, _int, ctypes.POINTER(_i64), _int, ctypes.POINTER(_vp),
         ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_i64), _vp],
    ),
    "ssb_window_fused": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _int, _vp, _vp, _vp, _i64, _vp, _int, _vp]),
    "ssb_window_sum_at": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp]),
    "ssb_swa_host": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _int, _vp, _vp, _vp, _i64, _int, _int, _i64]),
    "ssb_sharded_plan": (_int, [_i64, _i64, _i64, _int, ctypes.POINTER(_i64)]),
    "ssb_sharded_workspace_bytes": (_i64, [_int, _i64, _i64, _i64, _int, _int, _int]),
    "ssb_sharded_swa": (
        _int,
        [_int, ctypes.POINTER(_int), _int, _i64, _i64, _i64, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64,
         ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, ctypes.POINTER(_vp),
         ctypes.POINTER(_i64), ctypes.POINTER(_vp)],
    ),
    "ssb_band_carry": (_int, [_vp, _int, _i64, _i64, _int, _vp, _vp]),
    "ssb_selftest_division": (_int, [_vp, _i64, ctypes.c_double, _vp, _vp]),
    "ssb_census_enable": (_int, [_vp, _i64, _vp, _i64, _vp, _i64]),
    "ssb_census_disable": (_int, []),
    "ssb_host_release": (_int, []),
    "ssb_host_wire": (_int, [_int]),
    "ssb_host_threads": (_int, [_int]),
    "ssb_host_widen": (_int, [_vp, _int, _vp, _i64]),
    "ssb_sums_to_host": (_int, [_vp, _i64, _i64, ctypes.c_uint64, _vp, _i64, _vp]),
    "ssb_host_last_copy_bytes": (None, [ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "ssb_file_to_device": (_int, [ctypes.c_char_p, _i64, _i64, _vp, _int, _vp]),
    "ssb_device_to_file": (_int, [ctypes.c_char_p, _i64, _vp, _i64, _int, _vp]),
    "ssb_f32_nonfinite": (_int, [_vp, _i64, _vp, _vp]),
}
EXPORTS = tuple(_SIGS)


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise SatsweepError(
                    f"{LIB_PATH.name} is not built; run `python -m paper_2410_16291_b200.build_ext` "
                    "(there is no CPU fallback)"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                if os.environ.get("SSB_LIB") and not hasattr(lib, name):
                    continue  # older tuning build without this entry point
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.ssb_abi_version() != 1:
                raise SatsweepError("libsatsweep_b200 ABI version mismatch")
            _lib = lib
    return _lib


def check(rc: int, what: str = "", required_bytes: int = 0) -> None:
    """Map a status code onto the reference's exception types."""
    if rc == OK:
        return
    msg = load().ssb_last_error().decode(errors="replace")
    if rc == EINVAL:
        if "window" in msg or "stride" in msg or "region" in msg:
            raise InvalidWindowError(msg)
        raise ValueError(msg)
    if rc == ENOMEM:
        raise ResourceLimitError(required_bytes, what or msg)
    if rc == EUNSUPPORTED:
        raise TypeError(msg)
    if rc == ENONFINITE:
        raise GridValidationError(msg)
    raise SatsweepError(f"{what}: {msg}" if what else msg)


def launch_count() -> int:
    return int(load().ssb_launch_count())
