"""Beer-Lambert transforms and background estimation (src/optics.py:1-110).

The forward transform is evaluated through a 256-entry per-channel table
built with the reference's own expression ``ln(i0 / clip(i, 1, i0))``
(src/optics.py:92-94) on the 0..255 ramp: for 8-bit input the table is
bit-identical to the reference's elementwise ufuncs, and it is what every
device kernel consumes.
"""
from __future__ import annotations

import warnings

import numpy as np

from . import _dev, _lib
from .order_stats import percentile_from_counts

WHITE_THRESHOLD = 220          # src/optics.py:22
SAMPLE_CAP = 100_000           # src/optics.py:25
_BRIGHT_PERCENTILE = 80.0      # src/optics.py:28


class BackgroundEstimateWarning(UserWarning):
    """A channel had no bright pixels; its maximum fell back to 255."""


def od_table(i0) -> np.ndarray:
    """(3, 256) float64 OD table for per-channel background ``i0``."""
    i0 = np.asarray(i0, dtype=np.float64)
    if i0.shape != (3,):
        raise ValueError("i0 must have 3 entries")
    if np.any(i0 < 1.0):
        raise ValueError("i0 components must be >= 1")
    ramp = np.repeat(np.arange(256, dtype=np.float64)[:, None], 3, axis=1)
    np.clip(ramp, 1.0, i0, out=ramp)
    return np.ascontiguousarray(np.log(i0 / ramp).T)


def i0_from_counts(counts) -> np.ndarray:
    """Per-channel 80th percentile from (3, 256) bright-value counts
    (src/optics.py:35-68, exact order statistics of u8 values)."""
    counts = np.asarray(counts, dtype=np.int64).reshape(3, 256)
    i0 = np.empty(3, dtype=np.float64)
    names = ("red", "green", "blue")
    for c in range(3):
        if counts[c].sum() == 0:
            warnings.warn(
                f"no pixels brighter than the white threshold in the {names[c]} "
                "channel; falling back to 255", BackgroundEstimateWarning, stacklevel=3)
            i0[c] = 255.0
        else:
            i0[c] = percentile_from_counts(counts[c], _BRIGHT_PERCENTILE)
    return i0


def estimate_max_intensity(bright_samples) -> np.ndarray:
    """src/optics.py:35-68 for three per-channel pools of 8-bit values."""
    if len(bright_samples) != 3:
        raise ValueError("expected three per-channel collections")
    counts = np.zeros((3, 256), dtype=np.int64)
    for c, s in enumerate(bright_samples):
        a = np.asarray(s, dtype=np.float64).ravel()
        if a.size and (np.any(a != np.round(a)) or a.min() < 0 or a.max() > 255):
            # non-8-bit pools: plain sort (host, small)
            from .order_stats import percentile

            counts = None
            break
        counts[c] = np.bincount(a.astype(np.int64), minlength=256)[:256]
    if counts is not None:
        return i0_from_counts(counts)
    from .order_stats import percentile

    out = np.empty(3)
    for c, s in enumerate(bright_samples):
        a = np.asarray(s, dtype=np.float64).ravel()
        if a.size == 0:
            warnings.warn("no bright pixels; falling back to 255", BackgroundEstimateWarning,
                          stacklevel=2)
            out[c] = 255.0
        else:
            out[c] = percentile(a, _BRIGHT_PERCENTILE)
    return out


def beer_lambert(pixels, i0):
    """src/optics.py:71-94 on the device.  u8 (..., 3) in, float64 (..., 3) out.

    numpy in → numpy out; CUDA tensor in → CUDA tensor out.
    """
    i0 = np.asarray(i0, dtype=np.float64)
    table = od_table(i0)
    t = _dev.torch()
    host = not _dev.is_tensor(pixels)
    x = pixels if not host else np.asarray(pixels)
    if host and x.dtype != np.uint8:
        if np.any(x != np.round(x)) or x.min() < 0 or x.max() > 255:
            raise TypeError("beer_lambert on the device takes 8-bit pixels")
        x = x.astype(np.uint8)
    dx = _dev.to_device(x, dtype=t.uint8)
    shape = tuple(dx.shape)
    if shape[-1] != 3:
        raise ValueError("pixels must have a trailing channel axis of 3")
    n = dx.numel() // 3
    od = t.empty((3, n), dtype=t.float64, device=dx.device)
    L = _lib.lib()
    _lib.check(L.spcn_beer_lambert(_lib.ptr(dx), _lib.ptr(od), n, i0.ctypes.data,
                                   table.ctypes.data, _lib.stream_handle()), "beer_lambert")
    out = od.t().reshape(shape)
    return out.cpu().numpy() if host else out.contiguous()


def inverse_beer_lambert(od, i0):
    """src/optics.py:97-110 on the device: float64 (..., 3) → u8 (..., 3)."""
    i0 = _dev.f64_array(i0, 3, "i0")
    t = _dev.torch()
    host = not _dev.is_tensor(od)
    d = _dev.to_device(od, dtype=t.float64)
    shape = tuple(d.shape)
    n = d.numel() // 3
    out = t.empty(shape, dtype=t.uint8, device=d.device)
    _lib.check(_lib.lib().spcn_inverse_beer_lambert(_lib.ptr(d), _lib.ptr(out), n, i0.ctypes.data,
                                                    _lib.stream_handle()), "inverse_beer_lambert")
    return out.cpu().numpy() if host else out
