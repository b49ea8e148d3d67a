"""Device order statistics (libspcn radix select) for CUDA tensors.

Exact: the k-th smallest value is found by counting fp64 bit patterns, so
results equal ``np.sort(x)[k]`` bit for bit.
"""
from __future__ import annotations

import numpy as np

from . import _dev, _lib
from .errors import StainAbsentError

_QBYTES = 32  # sizeof(SelQuery)


def _sig():
    L = _lib.lib()
    if not getattr(L, "_spcn_stats_declared", False):
        P, I64, I32, DBL = _lib.P, _lib.I64, _lib.I32, _lib.DBL
        _lib.declare("spcn_select_kth", _lib.ctypes.c_int, [P, P, P, P, I32, P, P, P])
        _lib.declare("spcn_percentile_segments", _lib.ctypes.c_int,
                     [P, I64, P, I32, DBL, P, P, P, P, P])
        L._spcn_stats_declared = True
    return L


def select_kth(values, ks):
    """k-th smallest entries (0-based ranks ``ks``) of a 1-D CUDA float64 tensor."""
    t = _dev.torch()
    L = _sig()
    v = values.reshape(-1).to(t.float64).contiguous()
    ks = np.asarray(ks, dtype=np.int64).ravel()
    n = v.numel()
    if np.any(ks < 0) or np.any(ks >= n):
        raise ValueError("rank out of range")
    nq = ks.size
    b = t.zeros(nq, dtype=t.int64, device=v.device)
    e = t.full((nq,), n, dtype=t.int64, device=v.device)
    k = t.from_numpy(ks).to(v.device)
    q = t.empty(nq * _QBYTES, dtype=t.uint8, device=v.device)
    out = t.empty(nq, dtype=t.float64, device=v.device)
    _lib.check(L.spcn_select_kth(_lib.ptr(v), _lib.ptr(b), _lib.ptr(e), _lib.ptr(k), nq,
                                 _lib.ptr(q), _lib.ptr(out), _lib.stream_handle()), "select_kth")
    return out


def percentile_device(values, p: float) -> float:
    """order_stats.percentile for a CUDA tensor (src/order_stats.py:11-36)."""
    from .order_stats import interpolate

    n = values.numel()
    if n == 0:
        raise ValueError("percentile of an empty collection")
    if not 0.0 <= p <= 100.0:
        raise ValueError(f"percentile p must be in [0, 100], got {p}")
    rank = (p / 100.0) * (n - 1)
    lo, hi = int(np.floor(rank)), int(np.ceil(rank))
    vals = select_kth(values, [lo, hi]).cpu().numpy()
    return interpolate(vals[0], vals[1], rank)


def segment_percentiles(h, seg_offsets, p: float = 99.0):
    """Per-segment, per-stain percentile of a (2, total) CUDA float64 density
    tensor.  Returns (values (nseg, 2) CUDA tensor, absent (nseg, 2) CUDA int32)."""
    t = _dev.torch()
    L = _sig()
    total = h.shape[1]
    seg = seg_offsets if _dev.is_tensor(seg_offsets) else t.as_tensor(
        np.asarray(seg_offsets, dtype=np.int64), device=h.device)
    nseg = seg.numel() - 1
    q = t.empty(6 * nseg * _QBYTES, dtype=t.uint8, device=h.device)
    sel = t.empty(6 * nseg, dtype=t.float64, device=h.device)
    out = t.empty((nseg, 2), dtype=t.float64, device=h.device)
    absent = t.empty((nseg, 2), dtype=t.int32, device=h.device)
    _lib.check(L.spcn_percentile_segments(_lib.ptr(h), total, _lib.ptr(seg), nseg, float(p),
                                          _lib.ptr(q), _lib.ptr(sel), _lib.ptr(out),
                                          _lib.ptr(absent), _lib.stream_handle()),
               "percentile_segments")
    return out, absent


def stain_stats_device(h, sample_count=None):
    """stain_stats pooled mode (src/normalize.py:83-100) on a CUDA (2, N) tensor."""
    from .normalize import _STAIN_NAMES, StainStats

    hh = h.to(_dev.torch().float64).contiguous()
    n = hh.shape[1]
    vals, absent = segment_percentiles(hh, [0, n], 99.0)
    vals, absent = vals.cpu().numpy()[0], absent.cpu().numpy()[0]
    for j in range(2):
        if absent[j]:
            raise StainAbsentError(f"stain absent: no {_STAIN_NAMES[j]} density observed")
    p99 = np.asarray(vals, dtype=np.float64)
    if not np.all(np.isfinite(p99)) or np.any(p99 < 0):
        raise ValueError(f"p99 must be finite and non-negative, got {p99}")
    return StainStats(p99=p99, sample_count=int(sample_count) if sample_count is not None else n)
