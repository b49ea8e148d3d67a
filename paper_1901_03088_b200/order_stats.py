"""Order statistics — the single percentile definition of src/order_stats.py:1-47.

``percentile(values, p)`` = linear interpolation between closest ranks with
zero-based rank ``p/100*(n-1)``.  Host arrays are answered on the host (these
are ≤100 k-element scalars of the fit, not the per-pixel path); CUDA tensors
go through the device radix select (``stats.select_kth``) so no device data
is copied back for a sort.
"""
from __future__ import annotations

import math

import numpy as np

from . import _dev


def _check_p(p: float) -> None:
    if not 0.0 <= p <= 100.0:
        raise ValueError(f"percentile p must be in [0, 100], got {p}")


def interpolate(lo_val: float, hi_val: float, rank: float) -> float:
    """a[lo] + (a[hi] - a[lo]) * frac, in float64 (src/order_stats.py:36)."""
    lo = math.floor(rank)
    frac = rank - lo
    return float(np.float64(lo_val) + (np.float64(hi_val) - np.float64(lo_val)) * np.float64(frac))


def percentile(values, p: float) -> float:
    """src/order_stats.py:11-36."""
    if _dev.is_tensor(values) and values.is_cuda:
        from . import stats

        return stats.percentile_device(values, p)
    a = np.sort(np.asarray(values, dtype=np.float64).ravel())
    if a.size == 0:
        raise ValueError("percentile of an empty collection")
    _check_p(p)
    rank = (p / 100.0) * (a.size - 1)
    return interpolate(a[int(math.floor(rank))], a[int(math.ceil(rank))], rank)


def median(values) -> float:
    """src/order_stats.py:39-47."""
    a = np.sort(np.asarray(values, dtype=np.float64).ravel())
    if a.size == 0:
        raise ValueError("median of an empty collection")
    mid = a.size // 2
    if a.size % 2 == 1:
        return float(a[mid])
    return float((a[mid - 1] + a[mid]) / 2.0)


def percentile_from_counts(counts, p: float) -> float:
    """Exact percentile of a multiset of small integers given as a histogram.

    ``counts[v]`` = multiplicity of value v.  Identical to ``percentile`` of
    the expanded multiset (order statistics of integers are exact; the
    interpolation is the same float64 expression).  Used for i0 from the
    per-channel 256-bin bright-pixel counts the sampling kernel produces.
    """
    c = np.asarray(counts, dtype=np.int64).ravel()
    n = int(c.sum())
    if n == 0:
        raise ValueError("percentile of an empty collection")
    _check_p(p)
    rank = (p / 100.0) * (n - 1)
    cum = np.cumsum(c)
    lo_idx, hi_idx = int(math.floor(rank)), int(math.ceil(rank))
    lo_val = int(np.searchsorted(cum, lo_idx, side="right"))
    hi_val = int(np.searchsorted(cum, hi_idx, side="right"))
    return interpolate(float(lo_val), float(hi_val), rank)
