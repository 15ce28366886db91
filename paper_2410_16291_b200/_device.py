"""Device plumbing: torch owns device memory and streams; the kernels are ours.

torch is used only for allocation, the current stream and host<->device copies
of small objects; every computation on the hot path is a launch inside
libsatsweep_b200.so.
"""

from __future__ import annotations

import numpy as np

from .errors import ResourceLimitError, SatsweepError


def torch():
    import torch as _t

    return _t


def require_cuda() -> None:
    t = torch()
    if not t.cuda.is_available():
        raise SatsweepError("no CUDA device is available; satsweep-b200 has no CPU fallback")


def current_device():
    require_cuda()
    t = torch()
    return t.device("cuda", t.cuda.current_device())


def stream_ptr(device=None) -> int:
    t = torch()
    return int(t.cuda.current_stream(device).cuda_stream)


# storage dtypes: kernels only see raw pointers; uint64 results travel as int64
# storage (bit-identical views on the host side).
def storage_dtype(np_dtype: np.dtype):
    t = torch()
    return {
        np.dtype(np.uint8): t.uint8,
        np.dtype(np.uint16): t.uint16,
        np.dtype(np.int32): t.int32,
        np.dtype(np.float32): t.float32,
        np.dtype(np.uint64): t.int64,
        np.dtype(np.int64): t.int64,
        np.dtype(np.float64): t.float64,
    }[np.dtype(np_dtype)]


_TOTAL: dict = {}


def total_memory(device) -> int:
    """Device capacity, cached: cudaMemGetInfo can stall the host for tens of
    milliseconds, so it stays off the per-call path."""
    t = torch()
    idx = t.device(device).index
    idx = t.cuda.current_device() if idx is None else idx
    if idx not in _TOTAL:
        _TOTAL[idx] = int(t.cuda.get_device_properties(idx).total_memory)
    return _TOTAL[idx]


def empty(shape, np_dtype, device, what: str):
    """Device allocation that raises ResourceLimitError (integral.py:76-83) on failure."""
    t = torch()
    nbytes = int(np.prod(shape, dtype=object)) * np.dtype(np_dtype).itemsize
    if nbytes > total_memory(device):
        raise ResourceLimitError(nbytes, what)
    try:
        return t.empty(tuple(int(s) for s in shape), dtype=storage_dtype(np_dtype), device=device)
    except (t.cuda.OutOfMemoryError, RuntimeError) as exc:  # pragma: no cover - device dependent
        if isinstance(exc, t.cuda.OutOfMemoryError) or "out of memory" in str(exc):
            raise ResourceLimitError(nbytes, what) from None
        raise


def to_device(arr: np.ndarray, device):
    """Host raster -> device tensor (one copy)."""
    import warnings

    t = torch()
    with warnings.catch_warnings():  # read-only views are only read here
        warnings.simplefilter("ignore", UserWarning)
        src = t.from_numpy(np.ascontiguousarray(arr).view(_view_np(arr.dtype)))
    return src.to(device)


def _view_np(dt):
    dt = np.dtype(dt)
    return {np.dtype(np.uint64): np.int64}.get(dt, dt)


def to_host(tensor, np_dtype: np.dtype) -> np.ndarray:
    """Device tensor -> fresh host numpy array of the requested dtype (bit view)."""
    return tensor.cpu().numpy().view(np.dtype(np_dtype))


def sums_to_host(tensor, max_sum: int) -> np.ndarray:
    """Device uint64 window sums -> fresh host uint64 array through ssb_sums_to_host: when
    ``max_sum`` (a bound on every sum, w * w * the kind's largest pixel) is below 2**32 the
    sums cross PCIe as uint32 / uint16 and the library's host threads widen them (the same
    wire as ssb_swa_host); otherwise, and for small grids, a straight 64-bit copy."""
    from . import _lib

    if tensor.dim() != 2 or not tensor.is_contiguous() or tensor.element_size() != 8:
        return to_host(tensor, np.uint64)
    rows, cols = (int(v) for v in tensor.shape)
    out = np.empty((rows, cols), dtype=np.uint64)
    if rows == 0 or cols == 0:
        return out
    with torch().cuda.device(tensor.device):
        rc = _lib.load().ssb_sums_to_host(tensor.data_ptr(), rows, cols, max(0, min(int(max_sum), 2**64 - 1)),
                                          out.ctypes.data, cols, stream_ptr(tensor.device))
    _lib.check(rc, "result read-back")
    return out


def as_np_view(tensor, np_dtype):
    """Device tensor with a different logical dtype (e.g. int64 storage read as uint64) -- host copy."""
    return to_host(tensor, np_dtype)
