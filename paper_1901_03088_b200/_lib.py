"""ctypes binding of libspcn.so (the C ABI declared in include/spcn.h).

The library is the product path: there is no CPU fallback.  Loading fails
loudly when the .so is missing or when a call is made without a CUDA device.
"""
from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPCN_LIB_PATH") or os.path.join(_HERE, "libspcn.so")   # override: A/B tools

SPCN_OK = 0
SPCN_EINVAL = 1
SPCN_EBLANK = 2
SPCN_EINSUFFICIENT = 3
SPCN_ESTAIN_ABSENT = 4
SPCN_EDEGENERATE = 5
SPCN_ECUDA = 6
SPCN_ENCCL = 7

PREC = {"exact": 0, "fast": 1, "strict": 2}

# every symbol include/spcn.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "spcn_xform_workspace_bytes", "spcn_xform_rgb8", "spcn_xform_repair_count",
    "spcn_xform_calibrate", "spcn_xform_calibrate_part",
    "spcn_code_densities", "spcn_normalize_block", "spcn_beer_lambert",
    "spcn_inverse_beer_lambert", "spcn_sample_count", "spcn_sample_compact",
    "spcn_i0_from_hist", "spcn_od_tables", "spcn_snmf_batched", "spcn_code_samples",
    "spcn_percentile_segments", "spcn_code_table", "spcn_percentile_table",
    "spcn_select_kth", "spcn_render_synthetic",
    "spcn_batch_sizes", "spcn_batch_params", "spcn_xform_batch",
    "spcn_stats_hist", "spcn_stats_refine", "spcn_stats_table", "spcn_stats_table_scan",
    "spcn_stats_cube_classes", "spcn_stats_table_cube", "spcn_table_entries_hist",
    "spcn_table_entries_collect",
    "spcn_sample_visit",
    "spcn_readback", "spcn_last_error", "spcn_version", "spcn_launch_count", "spcn_xform_shape",
    "spcn_xform_timing_enable", "spcn_xform_timing", "spcn_stream_sync",
    "spcn_fit_sample_step", "spcn_fit_basis_step", "spcn_xform_rgb8_fitted",
    "spcn_xform_fitted_prepare", "spcn_xform_fitted_run", "spcn_visit_single",
)


class XformParams(ctypes.Structure):
    _fields_ = [
        ("src_i0", ctypes.c_double * 3),
        ("src_basis", ctypes.c_double * 6),
        ("code_lam", ctypes.c_double),
        ("factors", ctypes.c_double * 2),
        ("tgt_basis", ctypes.c_double * 6),
        ("tgt_i0", ctypes.c_double * 3),
        ("od_table", ctypes.POINTER(ctypes.c_double)),
        ("precision", ctypes.c_int32),
        ("max_sweeps", ctypes.c_int32),
        ("cert_alpha", ctypes.c_double),
    ]


class XformFitted(ctypes.Structure):
    """include/spcn.h spcn_xform_fitted (the device-built recolouring)."""
    _fields_ = [
        ("src_od_table", ctypes.c_void_p),
        ("src_fit", ctypes.c_void_p),
        ("tgt_basis", ctypes.c_double * 6),
        ("tgt_p99", ctypes.c_double * 2),
        ("tgt_i0", ctypes.c_double * 3),
        ("code_lam", ctypes.c_double),
        ("max_sweeps", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("tgt_fit", ctypes.c_void_p),
        ("tgt_i0_dev", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
DBL = ctypes.c_double
I32 = ctypes.c_int32
SZ = ctypes.c_size_t

_SIGS = {
    "spcn_xform_workspace_bytes": (SZ, [I64]),
    "spcn_xform_rgb8": (ctypes.c_int, [P, P, I64, ctypes.POINTER(XformParams), P, SZ, P]),
    "spcn_xform_rgb8_fitted": (ctypes.c_int, [P, P, I64, ctypes.POINTER(XformFitted), P, SZ, P,
                                              P]),
    "spcn_xform_fitted_prepare": (ctypes.c_int, [ctypes.POINTER(XformFitted), I32, I32, P, SZ, P,
                                                 P, P]),
    "spcn_xform_fitted_run": (ctypes.c_int, [P, P, I64, I32, P, SZ, P]),
    "spcn_xform_repair_count": (ctypes.c_int, [P, P, ctypes.POINTER(I64)]),
    "spcn_xform_calibrate": (ctypes.c_int, [ctypes.POINTER(XformParams), P, SZ,
                                            ctypes.POINTER(DBL), P]),
    "spcn_code_densities": (ctypes.c_int, [P, P, I64, P, DBL, I32, P]),
    "spcn_normalize_block": (ctypes.c_int, [P, P, I64, P, P, P, P]),
    "spcn_beer_lambert": (ctypes.c_int, [P, P, I64, P, P, P]),
    "spcn_inverse_beer_lambert": (ctypes.c_int, [P, P, I64, P, P]),
    "spcn_last_error": (ctypes.c_char_p, []),
    "spcn_version": (ctypes.c_char_p, []),
    "spcn_launch_count": (ctypes.c_uint64, []),
    "spcn_xform_shape": (ctypes.c_char_p, []),
    "spcn_xform_timing_enable": (ctypes.c_int, [I32]),
    "spcn_xform_timing": (ctypes.c_int, [ctypes.POINTER(I64), ctypes.POINTER(DBL)]),
    "spcn_stream_sync": (ctypes.c_int, [P]),
    "spcn_fit_sample_step": (ctypes.c_int, [P, P, I32, I32, I32, P, P, I32, I32, P, P, P, P, P,
                                            I64, P]),
    "spcn_fit_basis_step": (ctypes.c_int, [P, I64, P, P, P, P, P, P, P, DBL, I32, P, P, P, I32, P,
                                           I64, P]),
}


def lib():
    """Load libspcn.so once; raise if it is absent (no fallback path)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"libspcn.so not built ({LIB_PATH}); run "
                        "`python -m paper_1901_03088_b200._build` — there is no CPU fallback")
                h = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def declare(name, restype, argtypes):
    """Register the signature of an additional entry point (used by the fit/stats modules)."""
    fn = getattr(lib(), name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


_CODE_TO_EXC = {
    SPCN_EINVAL: ValueError,
    SPCN_EBLANK: errors.BlankSlideError,
    SPCN_EINSUFFICIENT: errors.InsufficientPixelsError,
    SPCN_ESTAIN_ABSENT: errors.StainAbsentError,
    SPCN_EDEGENERATE: errors.DegenerateStainError,
}


def check(rc: int, what: str = "") -> None:
    """Translate a libspcn status code into the reference's exception type."""
    if rc == SPCN_OK:
        return
    msg = lib().spcn_last_error().decode("utf-8", "replace")
    exc = _CODE_TO_EXC.get(rc)
    if exc is None:
        raise RuntimeError(f"{what}: libspcn error {rc}: {msg}")
    raise exc(msg)


_RAW_STREAM = None


def stream_handle(stream=None) -> int:
    """cudaStream_t (as int) of `stream`, else of the current stream.  The
    current stream is read through torch's raw C accessors: the Python-level
    torch.cuda.current_stream() costs ~15 us of device-index checks per call,
    paid a dozen times per fit."""
    global _RAW_STREAM
    if stream is not None:
        return int(stream.cuda_stream)
    if _RAW_STREAM is None:
        import torch

        C = torch._C
        if hasattr(C, "_cuda_getCurrentRawStream") and hasattr(C, "_cuda_getDevice"):
            _RAW_STREAM = lambda: C._cuda_getCurrentRawStream(C._cuda_getDevice())  # noqa: E731
        else:  # pragma: no cover - older torch
            _RAW_STREAM = lambda: int(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    return int(_RAW_STREAM())


def ptr(t) -> int:
    return int(t.data_ptr())
