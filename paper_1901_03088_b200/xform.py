"""The per-pixel hot unit: ``process_strip`` ≙ src/pipeline.py:260-272.

``process_strip(pixels, src_i0, src_basis, code_lam, factors, tgt_basis,
tgt_i0)`` has the reference's signature and semantics (pure per pixel, any
chunking gives identical bytes) and runs one fused libspcn launch
(``spcn_xform_rgb8``).  ``XformPlan`` prepares the C parameter block once per
(source, target) pair so a whole-slide transform pays the host setup once.
"""
from __future__ import annotations

import ctypes

import numpy as np


from . import _dev, _lib
from .optics import od_table


CALIBRATE_INLINE = -1.0   # include/spcn.h SPCN_CALIBRATE_INLINE
CALIBRATE_DEVICE = -2.0   # include/spcn.h SPCN_CALIBRATE_DEVICE


class XformPlan:
    """Packed spcn_xform_params for one recoloring (host-side, reusable)."""

    def __init__(self, src_i0, src_basis, code_lam, factors, tgt_basis, tgt_i0,
                 precision: str = "exact", max_sweeps: int = 2000):
        if precision not in _lib.PREC:
            raise ValueError(f"precision must be one of {sorted(_lib.PREC)}")
        from .fitcore import od_table_cached

        i0b = _dev.f64_array(src_i0, 3, "src_i0")
        if (i0b < 1.0).any():
            od_table(i0b)                            # raises the reference's ValueError
        self.table = od_table_cached(i0b.tobytes())  # exact reference OD table (host numpy)
        p = _lib.XformParams()
        # the 21 leading doubles of spcn_xform_params in one numpy assignment
        np.frombuffer(p, dtype=np.float64, count=21)[:] = np.concatenate([
            i0b, _dev.f64_array(src_basis, 6, "src_basis"), [float(code_lam)],
            _dev.f64_array(factors, 2, "factors"), _dev.f64_array(tgt_basis, 6, "tgt_basis"),
            _dev.f64_array(tgt_i0, 3, "tgt_i0")])
        p.od_table = self.table.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        p.precision = _lib.PREC[precision]
        p.max_sweeps = int(max_sweeps)
        p.cert_alpha = 0.0
        self.params = p
        self.precision = precision
        self.alpha = None

    # Images at least this large amortise the ~0.5 ms exhaustive calibration.
    CALIBRATE_MIN_PIXELS = 1 << 24

    def calibrate(self, stream=None) -> float:
        """EXACT mode: replace the analytic per-pixel certification bound by the
        bound measured on all 2^24 colours (fewer fp64 repairs, same bytes)."""
        if self.alpha is None:
            L = _lib.lib()
            ws = _dev.workspace(64, stream=_lib.stream_handle(stream))
            out = ctypes.c_double(-1.0)
            _lib.check(L.spcn_xform_calibrate(ctypes.byref(self.params), _lib.ptr(ws), 64,
                                              ctypes.byref(out), _lib.stream_handle(stream)),
                       "xform_calibrate")
            self.alpha = float(out.value)
            self.params.cert_alpha = self.alpha if self.alpha > 0 else 0.0
        return self.alpha

    def maybe_calibrate(self, npix: int, stream=None, inline: bool = False) -> None:
        """Use the calibrated bound for large images.  inline=True leaves the
        calibration to the next run (on the device, no host round trip) —
        for a single launch over the whole image; many launches (streamed
        strips) should calibrate once up front instead."""
        if self.precision == "exact" and npix >= self.CALIBRATE_MIN_PIXELS:
            if inline:
                self.params.cert_alpha = CALIBRATE_INLINE
            else:
                self.calibrate(stream)

    def calibrate_shared(self, total_pixels: int, npix: int, part: int, nparts: int, reduce_max,
                         stream=None) -> None:
        """Multi-GPU calibration: this rank evaluates part `part` of `nparts`
        of the colours into the calibration word of the workspace the next
        run(npix) on this stream uses; reduce_max(int32 tensor) max-reduces the
        word across ranks (a collective: every rank must call this with the
        same total_pixels, which decides whether to calibrate at all)."""
        if not (self.precision == "exact" and total_pixels >= self.CALIBRATE_MIN_PIXELS):
            return
        L = _lib.lib()
        if not getattr(L, "_spcn_calpart_declared", False):
            _lib.declare("spcn_xform_calibrate_part", ctypes.c_int,
                         [ctypes.POINTER(_lib.XformParams), _lib.I32, _lib.I32, _lib.P, _lib.I64,
                          _lib.P])
            L._spcn_calpart_declared = True
        ws_bytes = int(L.spcn_xform_workspace_bytes(int(npix)))
        ws = _dev.workspace(ws_bytes, stream=_lib.stream_handle(stream))
        _lib.check(L.spcn_xform_calibrate_part(ctypes.byref(self.params), int(part), int(nparts),
                                               _lib.ptr(ws), ws_bytes, _lib.stream_handle(stream)),
                   "xform_calibrate_part")
        reduce_max(ws[8:12].view(_dev.torch().int32))
        self.params.cert_alpha = CALIBRATE_DEVICE

    def run(self, src, dst, npix: int, stream=None) -> None:
        """src/dst: CUDA uint8 tensors (or raw device pointers) holding npix RGB pixels."""
        L = _lib.lib()
        ws_bytes = int(L.spcn_xform_workspace_bytes(int(npix)))
        ws = _dev.workspace(ws_bytes, stream=_lib.stream_handle(stream))
        sp = src if isinstance(src, int) else _lib.ptr(src)
        dp = dst if isinstance(dst, int) else _lib.ptr(dst)
        _lib.check(L.spcn_xform_rgb8(sp, dp, int(npix), ctypes.byref(self.params), _lib.ptr(ws),
                                     ws_bytes, _lib.stream_handle(stream)), "xform_rgb8")

    def repair_count(self, stream=None) -> int:
        """Pixels sent to the fp64 repair path by the last EXACT run (synchronizes)."""
        L = _lib.lib()
        ws = _dev.workspace(16, stream=_lib.stream_handle(stream))
        out = ctypes.c_int64(0)
        _lib.check(L.spcn_xform_repair_count(_lib.ptr(ws), _lib.stream_handle(stream),
                                             ctypes.byref(out)), "repair_count")
        return int(out.value)


def process_strip(pixels, src_i0, src_basis, code_lam, factors, tgt_basis, tgt_i0,
                  precision: str = "exact", out=None):
    """Recolor one strip (src/pipeline.py:260-272).  numpy in → numpy out,
    CUDA tensor in → CUDA tensor out (``out`` may be given for the latter)."""
    t = _dev.torch()
    host = not _dev.is_tensor(pixels)
    src = _dev.to_device(pixels, dtype=t.uint8)
    if src.ndim != 3 or src.shape[2] != 3:
        raise ValueError("pixels must be (h, w, 3) uint8")
    dst = out if out is not None else t.empty_like(src)
    plan = XformPlan(src_i0, src_basis, code_lam, factors, tgt_basis, tgt_i0, precision)
    plan.run(src, dst, src.numel() // 3)
    return dst.cpu().numpy() if host else dst
