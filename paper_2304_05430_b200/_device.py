"""Device plumbing: PyTorch owns device memory and streams; the kernels see
raw pointers through the C ABI.

Every helper raises if CUDA is unavailable -- the product path never falls
back to the CPU.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _lib

_torch = None
_ws_lock = threading.Lock()
_ws_cache: dict = {}


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


_cuda_ok = False


def require_cuda():
    global _cuda_ok
    t = torch()
    if _cuda_ok:  # checked once per process (is_available costs ~4 us per call)
        return t
    if not t.cuda.is_available():
        raise _lib.LibraryError("paper_2304_05430_b200 needs a CUDA device (B200, sm_100a); none is visible")
    _lib.load()
    _cuda_ok = True
    return t


def device():
    return require_cuda().device("cuda", torch().cuda.current_device())


def stream_ptr() -> int:
    return require_cuda().cuda.current_stream().cuda_stream


def ptr(x) -> int | None:
    return None if x is None else x.data_ptr()


def to_dev(a, dtype=None):
    """Upload a numpy array (or pass a CUDA tensor through)."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        out = a if a.is_cuda else a.cuda()
        return out if dtype is None else out.to(dtype)
    arr = np.ascontiguousarray(a)
    ten = t.from_numpy(arr)
    if dtype is not None:
        ten = ten.to(dtype)
    return ten.to(device(), non_blocking=False)


def empty(n, dtype):
    t = require_cuda()
    return t.empty(int(n), dtype=dtype, device=device())


def zeros(n, dtype):
    t = require_cuda()
    return t.zeros(int(n), dtype=dtype, device=device())


def workspace(nbytes: int, key: str = "default"):
    """A per-(thread, stream, key) reusable uint8 workspace of >= nbytes."""
    t = require_cuda()
    k = (threading.get_ident(), stream_ptr(), key)
    with _ws_lock:
        buf = _ws_cache.get(k)
        if buf is None or buf.numel() < nbytes:
            buf = t.empty(max(int(nbytes), 256), dtype=t.uint8, device=device())
            _ws_cache[k] = buf
    return buf


def real_dtype(precision: str):
    t = torch()
    if precision == "fp64":
        return t.float64
    if precision in ("fp32", "tf32", "fp32_cuda"):  # tf32: tensor-core scoring, fp32 storage;
        # fp32_cuda: the fp32 CUDA-core kernels even where a tensor-core fp32 path exists
        return t.float32
    raise ValueError(f"precision must be 'fp32', 'tf32', 'fp32_cuda' or 'fp64', got {precision!r}")
