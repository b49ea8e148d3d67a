"""Synthetic H&E slides rendered on the device (measurement input, K8).

Same generative model as src/synthetic.py:26-121 (``render_slide``), with a
counter-based RNG so that any row band of a gigapixel slide can be rendered
independently on any GPU.  Parity tests use the reference's own renderer
(via the oracle fixtures); this generator feeds the benchmarks.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _dev, _lib
from .stain_sep import reference_basis


class SynthParamsC(ctypes.Structure):
    _fields_ = [("i0", ctypes.c_float * 3), ("basis", ctypes.c_float * 6),
                ("tissue_fraction", ctypes.c_float), ("layout", ctypes.c_int32),
                ("dense", ctypes.c_int32)]


def _sig():
    L = _lib.lib()
    if not getattr(L, "_spcn_synth_declared", False):
        P, I64 = _lib.P, _lib.I64
        _lib.declare("spcn_render_synthetic", ctypes.c_int,
                     [P, I64, I64, I64, I64, ctypes.c_uint64, ctypes.POINTER(SynthParamsC), P])
        L._spcn_synth_declared = True
    return L


def render_rows(out, width: int, height: int, row0: int, rows: int, seed: int, *,
                i0=(255, 255, 255), tissue_fraction: float = 0.6, layout: str = "scatter",
                dense: bool = False, stream=None):
    """Render rows [row0, row0+rows) into the CUDA uint8 tensor ``out`` (rows*width*3 bytes)."""
    L = _sig()
    p = SynthParamsC()
    p.i0[:] = [float(x) for x in i0]
    p.basis[:] = [float(x) for x in reference_basis().ravel()]
    p.tissue_fraction = float(tissue_fraction)
    if layout not in ("scatter", "block"):
        raise ValueError(f"unknown layout {layout!r}")
    p.layout = 0 if layout == "scatter" else 1
    p.dense = 1 if dense else 0
    _lib.check(L.spcn_render_synthetic(_lib.ptr(out), int(width), int(row0), int(rows),
                                       int(height), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                       ctypes.byref(p), _lib.stream_handle(stream)),
               "render_synthetic")
    return out


def render_slide(width: int, height: int, seed: int, *, i0=(255, 255, 255),
                 tissue_fraction: float = 0.6, layout: str = "scatter", dense: bool = False,
                 device=None):
    """A whole (height, width, 3) uint8 CUDA slide."""
    t = _dev.torch()
    out = t.empty((height, width, 3), dtype=t.uint8, device=device or "cuda")
    render_rows(out, width, height, 0, height, seed, i0=i0, tissue_fraction=tissue_fraction,
                layout=layout, dense=dense)
    return out


def tissue_fraction_of(pixels, threshold: int = 220) -> float:
    """Fraction of non-white pixels (any channel <= threshold) of a CUDA slide."""
    nw = (pixels <= threshold).any(dim=-1)
    return float(nw.float().mean().item()) if nw.numel() else float(np.nan)
