"""Device plumbing (PyTorch is used for memory, streams and copies only)."""
from __future__ import annotations

import threading

import numpy as np

_ws_lock = threading.Lock()
_ws_cache: dict = {}


def torch():
    import torch as _t

    if not _t.cuda.is_available():
        raise RuntimeError("paper_1901_03088_b200 needs a CUDA device (B200); there is no CPU path")
    return _t


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


def workspace(nbytes: int, device=None):
    """Per-(device, thread) cached byte buffer for the repair list."""
    t = torch()
    dev = device if device is not None else t.cuda.current_device()
    key = (int(dev), threading.get_ident())
    with _ws_lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = t.empty(int(nbytes), dtype=t.uint8, device=dev)
            _ws_cache[key] = buf
    return buf


def f64_array(x, n, name):
    a = np.asarray(x, dtype=np.float64).ravel()
    if a.size != n:
        raise ValueError(f"{name} must have {n} entries, got {a.size}")
    return np.ascontiguousarray(a)
