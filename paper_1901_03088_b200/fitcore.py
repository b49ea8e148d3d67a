"""Device fit core: reusable buffers and the fit tail shared by the
single-process fit (pipeline.fit) and the row-band-sharded fit
(distributed.RowBandGroup.fit) — src/pipeline.py:203-257.

A fit is launch-bound (≈ 0.2 ms of kernels), so the host side is kept to two
short round trips: one read after sampling (i0, which the host needs to build
the OD table with numpy's own ``log`` — the reference's table, bit for bit)
and one packed read of basis / SNMF info / p99 / absent flags at the end.
Everything else — device buffers, the seeded candidate list of a slide
geometry, the SNMF initial basis of a seed, the OD table of an i0 — is a pure
function of its key and is memoised per thread, so a fit allocates nothing
and runs no numpy beyond the table of a new i0.
"""
from __future__ import annotations

import ctypes
import threading
from functools import lru_cache

import numpy as np

from . import _dev, _lib, optics, snmf
from .errors import InsufficientPixelsError, StainAbsentError
from .normalize import FitParams, StainStats, config_hash

_STAIN_NAMES = ("hematoxylin", "eosin")
_QBYTES = 32        # sizeof(SelQuery), stats.py

# phase-1 arena (bytes): state i64[8] | offsets i64[2] | i0 f64[3] | empty i32[3] | pad | hist i32[768]
A_STATE, A_OFFS, A_I0, A_EMPTY, A_HIST, A_BYTES, A_READ = 0, 64, 80, 104, 128, 128 + 3072, 116
# phase-2 arena (bytes): basis f64[6] | p99 f64[2] | info i32[4] | absent i32[2]
B_BASIS, B_P99, B_INFO, B_ABSENT, B_BYTES = 0, 48, 64, 80, 88


@lru_cache(maxsize=64)
def od_table_cached(i0_bytes: bytes) -> np.ndarray:
    """optics.od_table of an i0 (memoised: a pure function of the 24 bytes)."""
    return optics.od_table(np.frombuffer(i0_bytes, dtype=np.float64))


@lru_cache(maxsize=32)
def snmf_cfg_cached(lam, rel_tol, max_outer, seed, cluster) -> snmf.SnmfCfgC:
    from .stain_sep import SnmfConfig

    return snmf.make_cfg(SnmfConfig(lam=lam, rel_tol=rel_tol, max_outer_iters=max_outer,
                                    seed=seed), cluster)


def snmf_cluster(m: int) -> int:
    """snmf.fit_slide's cluster rule (20 k samples → a 16-CTA cluster, else 1)."""
    return snmf._BIG_CLUSTER[0] if m >= 20_000 else 1


class FitBuffers:
    """Device + pinned buffers of fits with one (target_pixels, max_outer) on
    one device and stream (per thread: a fit is stream-ordered on the
    caller's stream, so consecutive fits reuse them safely)."""

    def __init__(self, device, target_pixels: int, max_outer: int):
        t = _dev.torch()
        self.device = device
        self.target = max(int(target_pixels), 1)
        self.arena_a = t.empty(A_BYTES, dtype=t.uint8, device=device)
        self.arena_b = t.empty(B_BYTES, dtype=t.uint8, device=device)
        self.sample = t.empty(3 * self.target, dtype=t.uint8, device=device)
        self.lut = t.empty((1, 3, 256), dtype=t.float64, device=device)
        self.history = t.empty(max_outer + 1, dtype=t.float64, device=device)
        self.h = t.empty(2 * self.target, dtype=t.float64, device=device)
        self.scratch = t.empty(self.target + 2, dtype=t.float64, device=device)
        self.q = t.empty(6 * _QBYTES, dtype=t.uint8, device=device)
        self.sel = t.empty(6, dtype=t.float64, device=device)
        self.pin_a = t.empty(256, dtype=t.uint8, pin_memory=True)
        self.pin_b = t.empty(256, dtype=t.uint8, pin_memory=True)
        self.pin_lut = t.empty(768, dtype=t.float64, pin_memory=True)
        self.pin_status = t.zeros(4, dtype=t.int32, pin_memory=True)   # device-built xform
        self.cand = {}          # (W, H, plan) -> candidate descriptors on the device
        # raw pointers / numpy views of the fixed buffers (ctypes arguments)
        self.arena_a_ptr, self.arena_b_ptr = _lib.ptr(self.arena_a), _lib.ptr(self.arena_b)
        self.sample_ptr, self.pin_a_ptr = _lib.ptr(self.sample), _lib.ptr(self.pin_a)
        self.lut_ptr = _lib.ptr(self.lut)
        self.offsets_ptr = self.arena_a_ptr + A_OFFS
        self.h_ptr, self.scratch_ptr = _lib.ptr(self.h), _lib.ptr(self.scratch)
        self.history_ptr, self.q_ptr = _lib.ptr(self.history), _lib.ptr(self.q)
        self.sel_ptr = _lib.ptr(self.sel)
        self.pin_b_ptr, self.pin_lut_ptr = _lib.ptr(self.pin_b), _lib.ptr(self.pin_lut)
        self.pin_a_np, self.pin_b_np = self.pin_a.numpy(), self.pin_b.numpy()
        self.pin_lut_np = self.pin_lut.numpy()
        self.pin_status_ptr, self.pin_status_np = _lib.ptr(self.pin_status), self.pin_status.numpy()

    def offsets(self):
        """[0, m] of the current sample (written by k_visit, or by the host)."""
        return self.arena_a[A_OFFS:A_I0].view(_dev.torch().int64)


_TLS = threading.local()


def buffers(device, target_pixels: int, max_outer: int, slot: int = 0) -> FitBuffers:
    """The thread's fit buffers for (device, current stream, sizes); `slot`
    gives a second set for a fit in flight beside another (target + source)."""
    t = _dev.torch()
    dev = t.device(device) if not isinstance(device, t.device) else device
    if dev.index is None:
        dev = t.device("cuda", t._C._cuda_getDevice())
    cache = getattr(_TLS, "bufs", None)
    if cache is None:
        cache = _TLS.bufs = {}
    key = (dev.index, _lib.stream_handle(), int(target_pixels), int(max_outer), int(slot))
    fb = cache.get(key)
    if fb is None:
        if len(cache) > 8:
            cache.clear()
        fb = cache[key] = FitBuffers(dev, target_pixels, max_outer)
    return fb


def cfg_fields(plan, cfg, code_lam, per_patch_stats):
    return {"lambda": cfg.lam, "code_lambda": code_lam, "rel_tol": cfg.rel_tol,
            "max_outer_iters": cfg.max_outer_iters, "snmf_seed": cfg.seed,
            "sample_seed": plan.seed, "white_threshold": plan.white_threshold,
            "sample_cap": plan.sample_cap, "target_pixels": plan.target_pixels,
            "max_patches": plan.max_patches, "patch_size": plan.patch_size,
            "background_fraction_cutoff": plan.background_fraction_cutoff,
            "per_patch_stats": per_patch_stats}


@lru_cache(maxsize=256)
def _provenance_hash(items: tuple) -> str:
    return config_hash(dict(items))


@lru_cache(maxsize=256)
def _config_hash_of(plan, cfg, code_lam, per_patch_stats, p99_mode) -> str:
    fields = cfg_fields(plan, cfg, code_lam, per_patch_stats)
    if p99_mode != "sample":
        fields["p99_mode"] = p99_mode
    return _provenance_hash(tuple(sorted((k, str(v)) for k, v in fields.items())))


def provenance(plan, cfg, code_lam, per_patch_stats, p99_mode, source_label) -> dict:
    """src/pipeline.py:241-256 (the hash memoised per configuration)."""
    return {"source": str(source_label),
            "config_hash": _config_hash_of(plan, cfg, float(code_lam), bool(per_patch_stats),
                                           p99_mode)}


def basis_enqueue(fb: FitBuffers, sample_flat, m: int, i0: np.ndarray, cfg, *, code_lam: float,
                  pooled: bool) -> None:
    """Stream-ordered: OD table upload -> SNMF -> densities (code_lam, into
    fb.h as (2, m) rows) -> pooled p99 (pooled=True) -> read-back of arena B
    into fb.pin_b.  sample_flat: CUDA uint8 (3m,) tensor or its device
    address.  The caller syncs the stream before parse_*."""
    if m < 10:
        raise InsufficientPixelsError(
            f"basis fit: insufficient pixels: need at least 10 OD samples, got {m}")
    L = _lib.lib()
    # the reference's OD table (numpy log) into the pinned staging buffer; the
    # previous fit's upload of it has completed (its read-back was waited for)
    fb.pin_lut_np[:] = od_table_cached(np.ascontiguousarray(i0, np.float64).tobytes()).reshape(-1)
    c = snmf_cfg_cached(float(cfg.lam), float(cfg.rel_tol), int(cfg.max_outer_iters),
                        int(cfg.seed), snmf_cluster(m))
    sp = sample_flat if isinstance(sample_flat, int) else _lib.ptr(sample_flat)
    # table upload -> SNMF -> densities -> pooled p99 -> read-back, one call
    _lib.check(L.spcn_fit_basis_step(sp, m, fb.offsets_ptr, fb.pin_lut_ptr, fb.lut_ptr,
                                     ctypes.byref(c), fb.scratch_ptr, fb.history_ptr,
                                     fb.arena_b_ptr, float(code_lam), 2000, fb.h_ptr, fb.q_ptr,
                                     fb.sel_ptr, 1 if pooled else 0, fb.pin_b_ptr, B_BYTES,
                                     _lib.stream_handle()), "fit_basis_step")


def parse_pooled(fb: FitBuffers, m: int, i0: np.ndarray, cfg, prov: dict,
                 stacklevel: int = 4) -> FitParams:
    """FitParams of a pooled-p99 fit from arena B (read back, stream synced),
    with the reference's warnings and errors (src/pipeline.py:228-257)."""
    raw = fb.pin_b_np[:B_BYTES].copy()
    basis = raw[B_BASIS:B_P99].view(np.float64).reshape(3, 2).copy()
    p99 = raw[B_P99:B_INFO].view(np.float64).copy()
    info = raw[B_INFO:B_ABSENT].view(np.int32)
    absent = raw[B_ABSENT:B_BYTES].view(np.int32)
    snmf.warn_flags(m, int(info[2]), cfg.max_outer_iters, stacklevel=stacklevel)
    for j in range(2):
        if absent[j]:
            raise StainAbsentError(f"density stats: stain absent: no {_STAIN_NAMES[j]} "
                                   "density observed")
    if not (np.isfinite(p99).all() and (p99 >= 0).all()):
        raise ValueError(f"density stats: p99 must be finite and non-negative, got {p99}")
    return FitParams(i0=np.asarray(i0, np.float64).copy(), basis=basis,
                     stats=StainStats(p99=p99, sample_count=m), provenance=prov)


def fit_tail(fb: FitBuffers, sample_flat, m: int, i0: np.ndarray, plan, cfg, *,
             code_lam: float, per_patch_stats: bool, p99_mode: str, used_counts,
             source_label: str = "", chunks=None, comm=None, stage=None) -> FitParams:
    """src/pipeline.py:222-257 from the sample on: OD table → SNMF basis →
    densities (code_lam) → p99 (pooled, per-patch median, or whole-slide),
    FitParams with the reference's warnings, errors and provenance.

    sample_flat: CUDA uint8 (3m,) RGB sample; i0: host (3,) background.
    chunks: whole-slide pass generator (global p99 mode); comm: collectives of
    a row-band group (global mode)."""
    stage = stage or (lambda label, fn, *a, **k: fn(*a, **k))
    pooled = p99_mode == "sample" and not per_patch_stats
    basis_enqueue(fb, sample_flat, m, i0, cfg, code_lam=code_lam, pooled=pooled)
    h = fb.h[:2 * m].view(2, m)
    _lib.check(_lib.lib().spcn_stream_sync(_lib.stream_handle()), "stream_sync")
    prov = provenance(plan, cfg, code_lam, per_patch_stats, p99_mode, source_label)
    if pooled:
        return parse_pooled(fb, m, i0, cfg, prov, stacklevel=5)
    raw = fb.pin_b_np[:B_ABSENT].copy()
    basis = raw[B_BASIS:B_P99].view(np.float64).reshape(3, 2).copy()
    snmf.warn_flags(m, int(raw[B_INFO:B_ABSENT].view(np.int32)[2]), cfg.max_outer_iters,
                    stacklevel=4)
    from .normalize import stain_stats

    if p99_mode == "global":
        from .global_stats import global_p99, sample_bracket

        guess = sample_bracket(h)              # the sampled densities seed the first level
        p99, nonwhite, _ = stage("density stats", global_p99, chunks, i0, basis, code_lam,
                                 plan.white_threshold, comm=comm, guess=guess)
        st = StainStats(p99=p99, sample_count=int(nonwhite))
    elif per_patch_stats:
        from . import stats as dstats

        counts = [v for v in used_counts if v > 0]
        seg = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        vals, _ = dstats.segment_percentiles(h, seg, 99.0)
        st = stage("density stats", stain_stats,
                   patch_p99s=[tuple(v) for v in vals.cpu().numpy()], sample_count=m)
    else:
        st = stage("density stats", stain_stats, h)
    return FitParams(i0=np.asarray(i0, np.float64).copy(), basis=basis, stats=st, provenance=prov)
