"""Device sparse-NMF stain-basis fit (src/stain_sep.py:239-336).

``fit_basis`` keeps the reference's signature.  The batched entry
(``snmf_batched``) is what ``fit`` / ``fit_batch`` use: every problem is a
sample of RGB8 pixels plus its OD table, solved by one thread-block cluster.
"""
from __future__ import annotations

import ctypes
import functools
import warnings

import numpy as np

from . import _dev, _lib
from .errors import InsufficientPixelsError


class SnmfCfgC(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("rel_tol", ctypes.c_double),
                ("w_init", ctypes.c_double * 6), ("max_outer", ctypes.c_int32),
                ("cluster", ctypes.c_int32)]


def _sig():
    L = _lib.lib()
    if not getattr(L, "_spcn_snmf_declared", False):
        P, I64, I32, DBL = _lib.P, _lib.I64, _lib.I32, _lib.DBL
        _lib.declare("spcn_snmf_batched", ctypes.c_int,
                     [P, P, P, I32, P, ctypes.POINTER(SnmfCfgC), P, I64, P, P, P, P])
        _lib.declare("spcn_code_samples", ctypes.c_int,
                     [P, P, I32, I64, P, P, DBL, I32, P, I64, P])
        _lib.declare("spcn_code_table", ctypes.c_int,
                     [P, P, I32, I64, P, P, DBL, I32, P, I64, P])
        _lib.declare("spcn_percentile_table", ctypes.c_int,
                     [P, I64, P, P, I32, DBL, P, P, P])
        L._spcn_snmf_declared = True
    return L


def initial_basis(seed: int) -> np.ndarray:
    """The reference initializer (src/stain_sep.py:271-274), evaluated with numpy."""
    return _initial_basis(int(seed)).copy()


@functools.lru_cache(maxsize=64)
def _initial_basis(seed: int) -> np.ndarray:    # a pure function of the seed
    from .stain_sep import reference_basis

    w = reference_basis() + np.random.default_rng(seed).uniform(0.0, 0.05, size=(3, 2))
    w = np.maximum(w, 0.0)
    w /= np.linalg.norm(w, axis=0)
    return w


def make_cfg(cfg, cluster: int) -> SnmfCfgC:
    c = SnmfCfgC()
    c.lam = float(cfg.lam)
    c.rel_tol = float(cfg.rel_tol)
    c.w_init[:] = [float(x) for x in initial_basis(cfg.seed).ravel()]
    c.max_outer = int(cfg.max_outer_iters)
    c.cluster = int(cluster)
    return c


class BatchFit:
    """Device results of ``snmf_batched`` (bases already ordered, on the host)."""

    def __init__(self, basis, history, info, table=None):
        self.basis = basis          # (P, 3, 2)
        self.history = history      # (P, max_outer+1), valid prefix = info[:, 3]
        self.info = info            # (P, 4): iterations, converged, flags, history length
        self.table = table          # colour-table scratch (batches) or None


def snmf_batched(samples, offsets, luts, cfg, cluster: int = 1, od=None) -> BatchFit:
    """Run the batched SNMF kernel.  samples: CUDA uint8 (total*3,), offsets: CUDA
    int64 (P+1,), luts: CUDA float64 (P, 3, 256); or od: CUDA float64 (3, total)."""
    t = _dev.torch()
    L = _sig()
    nprob = offsets.numel() - 1
    total = (od.shape[1] if od is not None else samples.numel() // 3)
    dev = offsets.device
    basis = t.empty((nprob, 6), dtype=t.float64, device=dev)
    hist = t.zeros((nprob, cfg.max_outer_iters + 1), dtype=t.float64, device=dev)
    info = t.zeros((nprob, 4), dtype=t.int32, device=dev)
    c = make_cfg(cfg, cluster)
    # colour-table scratch (keys | counts | per-problem sizes): RGB8 samples only
    scratch = (t.empty(total + nprob // 2 + 1, dtype=t.float64, device=dev)
               if od is None and samples is not None else None)
    _lib.check(L.spcn_snmf_batched(
        _lib.ptr(samples) if samples is not None else None,
        _lib.ptr(od) if od is not None else None, _lib.ptr(offsets), nprob,
        _lib.ptr(luts) if luts is not None else None, ctypes.byref(c),
        _lib.ptr(scratch) if scratch is not None else None, total,
        _lib.ptr(basis), _lib.ptr(hist), _lib.ptr(info), _lib.stream_handle()), "snmf_batched")
    return BatchFit(basis.reshape(nprob, 3, 2), hist, info,
                    table=scratch if cluster == 1 else None)


def code_samples(samples, offsets, luts, bases, lam, max_m, max_sweeps=2000):
    """Batched code_densities of fit samples → CUDA (2, total) float64."""
    t = _dev.torch()
    L = _sig()
    nprob = offsets.numel() - 1
    total = samples.numel() // 3
    h = t.empty((2, total), dtype=t.float64, device=samples.device)
    b = bases.reshape(nprob, 6).to(t.float64).contiguous()
    _lib.check(L.spcn_code_samples(_lib.ptr(samples), _lib.ptr(offsets), nprob, int(max_m),
                                   _lib.ptr(luts), _lib.ptr(b), float(lam), int(max_sweeps),
                                   _lib.ptr(h), total, _lib.stream_handle()), "code_samples")
    return h


# one slide's fit: clusters of 16 CTAs (non-portable), else 8; SPCN_SNMF_CLUSTER
# overrides (A/B measurements: the cluster size fixes the reduction order)
_BIG_CLUSTER = [int(__import__("os").environ.get("SPCN_SNMF_CLUSTER", "16"))]


def fit_slide(samples, offsets, luts, cfg, m: int, od=None) -> BatchFit:
    """snmf_batched for ONE slide's sample: a thread-block cluster of 16 CTAs
    (8 if the device cannot schedule 16) from 20 k samples, else one CTA.
    The cluster size fixes the reduction order, so every caller (single
    process, row-band ranks) uses this rule."""
    if m < 20_000:
        return snmf_batched(samples, offsets, luts, cfg, cluster=1, od=od)
    while True:
        try:
            return snmf_batched(samples, offsets, luts, cfg, cluster=_BIG_CLUSTER[0], od=od)
        except RuntimeError:
            if _BIG_CLUSTER[0] == 8:
                raise
            _BIG_CLUSTER[0] = 8      # 16-CTA clusters unavailable here


def code_table(table, offsets, luts, bases, lam, max_m, total, max_sweeps=2000):
    """code_samples over the colour table of ``snmf_batched`` (one fp64
    evaluation per distinct colour) → CUDA (2, total) float64, valid at the
    entry positions."""
    t = _dev.torch()
    L = _sig()
    nprob = offsets.numel() - 1
    h = t.empty((2, max(total, 1)), dtype=t.float64, device=offsets.device)
    b = bases.reshape(nprob, 6).to(t.float64).contiguous()
    _lib.check(L.spcn_code_table(_lib.ptr(table), _lib.ptr(offsets), nprob, int(max_m),
                                 _lib.ptr(luts), _lib.ptr(b), float(lam), int(max_sweeps),
                                 _lib.ptr(h), total, _lib.stream_handle()), "code_table")
    return h


def percentile_table(h, table, offsets, total, p=99.0):
    """Per-problem percentile of the colour-table densities (weighted) →
    (values (P, 2), absent (P, 2) int32) CUDA tensors."""
    t = _dev.torch()
    L = _sig()
    nprob = offsets.numel() - 1
    out = t.empty((nprob, 2), dtype=t.float64, device=offsets.device)
    absent = t.empty((nprob, 2), dtype=t.int32, device=offsets.device)
    _lib.check(L.spcn_percentile_table(_lib.ptr(h), total, _lib.ptr(table), _lib.ptr(offsets),
                                       nprob, float(p), _lib.ptr(out), _lib.ptr(absent),
                                       _lib.stream_handle()), "percentile_table")
    return out, absent


def warn_flags(m: int, flags: int, max_outer: int, stacklevel: int = 3) -> None:
    """The reference's StainDegeneracyWarning conditions (src/stain_sep.py:264-331)."""
    from .stain_sep import StainDegeneracyWarning

    if m < 1000:
        warnings.warn(f"only {m} OD samples; the stain basis may be unreliable",
                      StainDegeneracyWarning, stacklevel=stacklevel)
    if flags & 1:
        warnings.warn(f"stain basis fit did not converge within {max_outer} outer iterations; "
                      "returning the best iterate", StainDegeneracyWarning, stacklevel=stacklevel)
    if flags & 2:
        warnings.warn("one stain carries essentially no density; the slide may contain a single "
                      "stain and the basis may be degenerate", StainDegeneracyWarning,
                      stacklevel=stacklevel)


def fit_basis(od_sample, cfg):
    """src/stain_sep.py:239-336 for a (3, M) OD sample (numpy or CUDA tensor)."""
    from .stain_sep import SnmfFit

    t = _dev.torch()
    v = _dev.to_device(od_sample, dtype=t.float64)
    if v.ndim != 2 or v.shape[0] != 3:
        raise ValueError(f"od_sample must be 3xM, got {tuple(v.shape)}")
    m = v.shape[1]
    if m < 10:
        raise InsufficientPixelsError(f"insufficient pixels: need at least 10 OD samples, got {m}")
    offsets = t.tensor([0, m], dtype=t.int64, device=v.device)
    r = fit_slide(None, offsets, None, cfg, m, od=v.contiguous())
    info = r.info.cpu().numpy()[0]
    hist = r.history.cpu().numpy()[0][: int(info[3])]
    warn_flags(m, int(info[2]), cfg.max_outer_iters)
    return SnmfFit(basis=r.basis.cpu().numpy()[0], objective=[float(x) for x in hist],
                   converged=bool(info[1]), iterations=int(info[0]))
