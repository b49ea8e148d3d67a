"""The reference-side binding of INTEGRATION.md §2, as a maintainer would add
it to the reference package (``slidenorm/_spcn_backend.py``): plain ctypes on
libspcn.so, no import of this package.  The OD table comes from the caller
(the reference builds it with its own ``beer_lambert``; the tests pass the
oracle's restatement of it)."""
import ctypes
import os

import numpy as np
import torch

_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_1901_03088_b200", "libspcn.so")
L = ctypes.CDLL(_LIB)


class XformParams(ctypes.Structure):            # = spcn_xform_params, include/spcn.h
    _fields_ = [("src_i0", ctypes.c_double * 3), ("src_basis", ctypes.c_double * 6),
                ("code_lam", ctypes.c_double), ("factors", ctypes.c_double * 2),
                ("tgt_basis", ctypes.c_double * 6), ("tgt_i0", ctypes.c_double * 3),
                ("od_table", ctypes.POINTER(ctypes.c_double)),
                ("precision", ctypes.c_int32), ("max_sweeps", ctypes.c_int32),
                ("cert_alpha", ctypes.c_double)]


L.spcn_xform_rgb8.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                              ctypes.POINTER(XformParams), ctypes.c_void_p,
                              ctypes.c_size_t, ctypes.c_void_p]
L.spcn_xform_workspace_bytes.argtypes = [ctypes.c_int64]
L.spcn_xform_workspace_bytes.restype = ctypes.c_size_t
L.spcn_last_error.restype = ctypes.c_char_p


def process_strip_gpu(pixels, src_i0, src_basis, code_lam, factors, tgt_basis, tgt_i0, table):
    """_process_strip (src/pipeline.py:260) through spcn_xform_rgb8, EXACT."""
    table = np.ascontiguousarray(table, dtype=np.float64)
    p = XformParams()
    p.src_i0[:] = [float(v) for v in src_i0]
    p.src_basis[:] = [float(v) for v in np.ravel(src_basis)]
    p.code_lam = float(code_lam)
    p.factors[:] = [float(v) for v in factors]
    p.tgt_basis[:] = [float(v) for v in np.ravel(tgt_basis)]
    p.tgt_i0[:] = [float(v) for v in tgt_i0]
    p.od_table = table.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    p.precision, p.max_sweeps, p.cert_alpha = 0, 2000, 0.0
    src = torch.from_numpy(np.ascontiguousarray(pixels)).cuda()
    dst = torch.empty_like(src)
    n = src.numel() // 3
    ws = torch.empty(L.spcn_xform_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    rc = L.spcn_xform_rgb8(src.data_ptr(), dst.data_ptr(), n, ctypes.byref(p), ws.data_ptr(),
                           ws.numel(), torch.cuda.current_stream().cuda_stream)
    if rc:
        raise ValueError(L.spcn_last_error().decode())
    return dst.cpu().numpy()
