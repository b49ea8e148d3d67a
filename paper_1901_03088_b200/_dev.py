"""Device plumbing (PyTorch is used for memory, streams and copies only)."""
from __future__ import annotations

import contextlib
import os
import threading

import numpy as np

_ws_lock = threading.Lock()
_ws_cache: dict = {}


_TORCH_OK = None


def torch():
    """The torch module, once a CUDA device is known to be present (checked
    on the first call: the availability query is slow and cannot change)."""
    global _TORCH_OK
    if _TORCH_OK is None:
        import torch as _t

        if not _t.cuda.is_available():
            raise RuntimeError("paper_1901_03088_b200 needs a CUDA device (B200); "
                               "there is no CPU path")
        _TORCH_OK = _t
    return _TORCH_OK


def is_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


def to_device(x, dtype=None, device=None):
    """numpy / sequence / tensor → contiguous CUDA tensor (no copy if already there)."""
    t = torch()
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    if is_tensor(x):
        y = x
        if dtype is not None and y.dtype != dtype:
            y = y.to(dtype)
        if y.device.type != "cuda":
            y = y.to(dev, non_blocking=True)
        return y.contiguous()
    a = np.ascontiguousarray(x)
    y = t.from_numpy(a)
    if dtype is not None and y.dtype != dtype:
        y = y.to(dtype)
    return y.to(dev, non_blocking=False)


def workspace(nbytes: int, device=None, stream: int | None = None):
    """Cached byte buffer for the repair list, one per (device, thread,
    stream): launches in flight on different streams (the streamed strips,
    the pipelined batch chunks) must not share a repair list."""
    t = torch()
    dev = device if device is not None else t._C._cuda_getDevice()
    if stream is None:
        from . import _lib

        stream = _lib.stream_handle()
    key = (int(dev), threading.get_ident(), int(stream))
    with _ws_lock:
        buf = _ws_cache.pop(key, None)
        if buf is None or buf.numel() < nbytes:
            with t.cuda.stream(t.cuda.ExternalStream(int(stream))) if stream else _null():
                buf = t.empty(int(nbytes), dtype=t.uint8, device=dev)
        _ws_cache[key] = buf            # most recently used last
        if len(_ws_cache) > 64:         # bound the cache (callers with transient streams);
            _ws_cache.pop(next(iter(_ws_cache)))   # freed into its own stream's pool: safe
    return buf


class _null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def f64_array(x, n, name):
    a = np.asarray(x, dtype=np.float64).ravel()
    if a.size != n:
        raise ValueError(f"{name} must have {n} entries, got {a.size}")
    return np.ascontiguousarray(a)


_rb = threading.local()


def readback(x) -> np.ndarray:
    """Small CUDA tensor → numpy through a reusable pinned buffer written by a
    kernel (libspcn spcn_readback), synchronising only the current stream —
    not queued behind large copies other streams have on the copy engine."""
    import ctypes

    from . import _lib

    t = torch()
    x = x.contiguous()
    nbytes = x.numel() * x.element_size()
    buf = getattr(_rb, "buf", None)
    if buf is None or buf.numel() < max(nbytes, 4):
        buf = t.empty(max(4096, 2 * nbytes), dtype=t.uint8, pin_memory=True)
        _rb.buf = buf
    L = _lib.lib()
    if not getattr(L, "_spcn_rb_declared", False):
        _lib.declare("spcn_readback", ctypes.c_int, [_lib.P, _lib.P, _lib.I64, _lib.P])
        L._spcn_rb_declared = True
    _lib.check(L.spcn_readback(_lib.ptr(x), _lib.ptr(buf), nbytes, _lib.stream_handle()),
               "readback")
    t.cuda.current_stream().synchronize()
    return buf[:nbytes].view(x.dtype).reshape(x.shape).numpy().copy()


class fast_stream:
    """``torch.cuda.stream(s)`` for a stream on the current device without the
    Python-level device-index checks (~30 us per use, three uses per
    normalize(image, image) call); another device takes torch's own."""

    __slots__ = ("s", "prev", "ctx")

    def __init__(self, s):
        self.s = s
        self.prev = self.ctx = None

    def __enter__(self):
        C = torch()._C
        s = self.s
        if s.device_index != C._cuda_getDevice():
            self.ctx = torch().cuda.stream(s)
            return self.ctx.__enter__()
        self.prev = C._cuda_getCurrentStream(s.device_index)
        C._cuda_setStream(stream_id=s.stream_id, device_index=s.device_index,
                          device_type=s.device_type)
        return s

    def __exit__(self, *exc):
        if self.ctx is not None:
            return self.ctx.__exit__(*exc)
        p = self.prev
        torch()._C._cuda_setStream(stream_id=p[0], device_index=p[1], device_type=p[2])
        return False


_NVTX = os.environ.get("SPCN_NVTX", "") not in ("", "0")


def nvtx(label: str):
    """NVTX range around a pass (SPCN_NVTX=1: visible in nsys/ncu timelines;
    otherwise a no-op context)."""
    if not _NVTX:
        return contextlib.nullcontext()
    import torch as _t

    return _t.cuda.nvtx.range(label)
