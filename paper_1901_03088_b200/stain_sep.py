"""Stain basis utilities, per-pixel density coding and the sparse-NMF fit.

Mirrors src/stain_sep.py:1-336.  ``code_densities`` and ``fit_basis`` run on
the device (libspcn: k_code_densities, the batched SNMF kernel); the 3x2
basis bookkeeping (``reference_basis``, ``validate_basis``,
``order_stains``) is host arithmetic on six numbers.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib

REFERENCE_HEMATOXYLIN_OD = (0.650, 0.704, 0.286)   # src/stain_sep.py:34
REFERENCE_EOSIN_OD = (0.072, 0.990, 0.105)         # src/stain_sep.py:35
_UNIT_NORM_TOL = 1e-9                              # src/stain_sep.py:37


class StainDegeneracyWarning(UserWarning):
    """The fit looks degenerate: one stain is absent or the solver stalled."""


@dataclass(frozen=True)
class SnmfConfig:
    """Solver settings for :func:`fit_basis` (src/stain_sep.py:44-63)."""

    lam: float = 0.1
    max_outer_iters: int = 200
    rel_tol: float = 1e-6
    seed: int = 0

    def __post_init__(self):
        if self.lam < 0:
            raise ValueError("lam must be >= 0")
        if self.max_outer_iters < 1:
            raise ValueError("max_outer_iters must be >= 1")
        if self.rel_tol <= 0:
            raise ValueError("rel_tol must be > 0")


@dataclass
class SnmfFit:
    """Result of :func:`fit_basis` (src/stain_sep.py:66-80)."""

    basis: np.ndarray
    objective: list
    converged: bool
    iterations: int


def reference_basis() -> np.ndarray:
    """src/stain_sep.py:83-86."""
    w = np.array([REFERENCE_HEMATOXYLIN_OD, REFERENCE_EOSIN_OD], dtype=np.float64).T
    return w / np.linalg.norm(w, axis=0)


def validate_basis(w) -> np.ndarray:
    """src/stain_sep.py:89-101."""
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (3, 2):
        raise ValueError(f"stain basis must be 3x2, got {w.shape}")
    if not np.all(np.isfinite(w)):
        raise ValueError("stain basis contains non-finite entries")
    if np.any(w < 0):
        raise ValueError("stain basis entries must be non-negative")
    norms = np.linalg.norm(w, axis=0)
    if np.any(np.abs(norms - 1.0) > _UNIT_NORM_TOL):
        raise ValueError(f"stain basis columns must have unit L2 norm, got {norms}")
    return w


def order_stains(w):
    """src/stain_sep.py:104-116: larger red-minus-blue OD first."""
    w = validate_basis(w)
    rb = w[0] - w[2]
    if rb[1] > rb[0]:
        return np.ascontiguousarray(w[:, ::-1]), (1, 0)
    return w.copy(), (0, 1)


def code_densities(od, w, lam, max_sweeps: int = 2000):
    """src/stain_sep.py:168-201 on the device: (3, N) OD → (2, N) densities.

    Bit-identical to the reference (same operation order and the same bitwise
    CD fixed point).  numpy in → numpy out; CUDA tensor in → CUDA tensor out.
    """
    w = validate_basis(w)
    if lam < 0:
        raise ValueError("lam must be >= 0")
    t = _dev.torch()
    host = not _dev.is_tensor(od)
    v = _dev.to_device(od, dtype=t.float64)
    if v.ndim != 2 or v.shape[0] != 3:
        raise ValueError(f"od must be 3xN, got {tuple(v.shape)}")
    n = v.shape[1]
    h = t.empty((2, n), dtype=t.float64, device=v.device)
    wc = np.ascontiguousarray(w, dtype=np.float64)
    _lib.check(_lib.lib().spcn_code_densities(_lib.ptr(v), _lib.ptr(h), n, wc.ctypes.data,
                                              float(lam), int(max_sweeps), _lib.stream_handle()),
               "code_densities")
    return h.cpu().numpy() if host else h


def snmf_objective(v, w, h, lam) -> float:
    """``||V - WH||_F^2 + lam * sum(H)`` (src/stain_sep.py:204-207), host reference form."""
    resid = np.asarray(v) - np.asarray(w) @ np.asarray(h)
    return float(resid.ravel() @ resid.ravel() + lam * np.asarray(h).sum())


def fit_basis(od_sample, cfg: SnmfConfig = SnmfConfig()) -> SnmfFit:
    """src/stain_sep.py:239-336 on the device (batched SNMF kernel, batch of one)."""
    from . import snmf

    return snmf.fit_basis(od_sample, cfg)
