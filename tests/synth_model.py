"""NumPy restatement of the on-device synthetic generator ``k_render``
(paper_1901_03088_b200/csrc/synth.cu:27-65) — test infrastructure only.

``k_render`` draws its random numbers from a counter-based hash of
(seed, pixel index) instead of the reference renderer's PCG64 stream
(src/synthetic.py:69-121), so its bytes differ from the reference's while the
generative model must not.  This module recomputes, for any pixel window, the
tissue mask and the stain densities the kernel used, so that tests can check
the rendered bytes against the model (od = W_ref h, pixel = floor(i0 e^-od +
0.5)) and a fit against the generator's own densities, as the reference does
for its renderer (tests/test_pipeline.py:80-91).
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def _mix64(z):
    z = z + _M1
    z = (z ^ (z >> np.uint64(30))) * _M2
    z = (z ^ (z >> np.uint64(27))) * _M3
    return z ^ (z >> np.uint64(31))


def _u01(x32):
    return (x32 >> np.uint64(8)).astype(np.float64) * (1.0 / 16777216.0)


def densities(width, height, seed, rows=None, tissue_fraction=0.6, layout="scatter",
              dense=False):
    """(h (2, n) float64, tissue (n,) bool) of the rows ``rows`` = (row0, nrows)
    of a width x height k_render slide (all rows by default)."""
    row0, nrows = rows if rows is not None else (0, height)
    with np.errstate(over="ignore"):
        y = np.arange(row0, row0 + nrows, dtype=np.uint64)[:, None]
        x = np.arange(width, dtype=np.uint64)[None, :]
        n = (y * np.uint64(width) + x).ravel()
        r0 = _mix64(np.uint64(seed) ^ _mix64(n))
        r1 = _mix64(r0)
    lo, hi = np.uint64(0xFFFFFFFF), np.uint64(32)
    ut, uk = _u01(r0 & lo), _u01(r0 >> hi)
    ua, ub = _u01(r1 & lo), _u01(r1 >> hi)
    tf = float(np.float32(tissue_fraction))
    if layout == "scatter":
        tissue = ut < tf
    else:
        side = int(np.rint(np.sqrt(tf * width * height)))
        bx, by = (width - side) // 2, (height - side) // 2
        yy = (row0 + np.arange(nrows))[:, None]
        xx = np.arange(width)[None, :]
        tissue = ((xx >= bx) & (xx < bx + side) & (yy >= by) & (yy < by + side)).ravel()
    f32 = lambda v: float(np.float32(v))      # noqa: E731  (the kernel compares in fp32)
    h = np.zeros((2, n.size))
    if dense:
        h[0] = 0.65 + 1.35 * ua
        h[1] = np.where(uk < f32(0.3), 0.0, 1.2 * ub)
    else:
        m0, m1 = 0.2 + 1.8 * ua, 0.2 + 1.8 * ub
        only_h, only_e = uk < f32(0.4), (uk >= f32(0.4)) & (uk < f32(0.8))
        both = ~(only_h | only_e)
        h[0] = np.where(only_h, m0, np.where(both, 0.7 * m0, 0.0))
        h[1] = np.where(only_e, m1, np.where(both, 0.7 * m1, 0.0))
    h[:, ~tissue] = 0.0
    return h, tissue


def pixels(h, basis, i0=(255, 255, 255)):
    """The model's bytes for densities h: floor(i0 exp(-W h) + 0.5), clipped."""
    od = np.asarray(basis, dtype=np.float64) @ h
    v = np.floor(np.asarray(i0, dtype=np.float64)[:, None] * np.exp(-od) + 0.5)
    return np.clip(v, 0, 255).astype(np.uint8).T
