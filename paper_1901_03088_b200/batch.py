"""Batched normalisation: many images, each with its own fit, one target.

BASELINE configs[1] ("batch of 4096 synthetic 512x512 patches against one
fixed target basis").  Per item this is exactly the reference's
``_normalize_one`` (src/cli.py:220-244): fit(item) then transform(item)
against the target; failures are collected per item and do not stop the
batch, like ``cmd_batch`` (src/cli.py:270-301).  All items go through each
stage together: one sampling launch, one i0 launch, one SNMF launch (a CTA
per item), one coding launch, one p99 select launch, a device-side parameter
build and one persistent recolour launch (+ the fp64 repair launch).
"""
from __future__ import annotations

import ctypes
import os
import threading
import warnings
from dataclasses import dataclass

import numpy as np

from . import _dev, _lib, optics, snmf
from .errors import (BlankSlideError, DegenerateStainError, InsufficientPixelsError,
                     StainAbsentError)
from .normalize import FitParams, StainStats, config_hash
from .pipeline import PATCH_DT, TAKE_DT, SamplePlan, _cfg_fields, _lib_sample, _visit
from .stain_sep import SnmfConfig
from .xform import XformPlan

CHUNK = 4096
_ERR = {-_lib.SPCN_EBLANK: BlankSlideError, -_lib.SPCN_EINSUFFICIENT: InsufficientPixelsError,
        -_lib.SPCN_ESTAIN_ABSENT: StainAbsentError, -_lib.SPCN_EDEGENERATE: DegenerateStainError}
_MSG = {-_lib.SPCN_EBLANK: "sampling: blank slide: no non-white pixels found in any sampled patch",
        -_lib.SPCN_EINSUFFICIENT: "basis fit: insufficient pixels: need at least 10 OD samples",
        -_lib.SPCN_ESTAIN_ABSENT: "density stats: stain absent",
        -_lib.SPCN_EDEGENERATE: "degenerate stain density: p99 is zero for a stain"}


class BatchTargetC(ctypes.Structure):
    _fields_ = [("i0", ctypes.c_double * 3), ("basis", ctypes.c_double * 6),
                ("p99", ctypes.c_double * 2)]


def _sig():
    L = _lib.lib()
    if not getattr(L, "_spcn_batch_declared", False):
        P, I32, DBL = _lib.P, _lib.I32, _lib.DBL
        _lib.declare("spcn_batch_sizes", ctypes.c_int,
                     [ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)])
        _lib.declare("spcn_batch_params", ctypes.c_int,
                     [I32, P, P, P, P, ctypes.POINTER(BatchTargetC), DBL, I32, I32, P, P, P, P, P])
        _lib.declare("spcn_xform_batch", ctypes.c_int,
                     [P, P, I32, P, P, P, P, P, P, P, I32, P, _lib.SZ, P])
        L._spcn_batch_declared = True
    return L


@dataclass
class BatchFit:
    """Per-item fit results (device tensors) + host status."""

    i0: object          # (n, 3) float64 CUDA
    basis: object       # (n, 3, 2) float64 CUDA (ordered)
    p99: object         # (n, 2) float64 CUDA
    luts: object        # (n, 3, 256) float64 CUDA (exact reference OD tables)
    count: np.ndarray   # (n,) sampled pixels
    status: np.ndarray  # (n,) 0 = ok, <0 = -SPCN_E* error code
    provenance: dict
    iterations: np.ndarray = None   # (n,) SNMF outer iterations (SnmfFit.iterations)
    converged: np.ndarray = None    # (n,) SnmfFit.converged
    warn_flags: np.ndarray = None   # (n,) bit0 no convergence, bit1 one stain (warnings)

    def error(self, i):
        st = int(self.status[i])
        if st >= 0:
            return None
        return _ERR[st](_MSG[st])

    def params(self, i) -> FitParams:
        """FitParams of item i (raises the item's error, like fit() would)."""
        err = self.error(i)
        if err is not None:
            raise err
        return FitParams(i0=self.i0[i].cpu().numpy(), basis=self.basis[i].cpu().numpy(),
                         stats=StainStats(p99=self.p99[i].cpu().numpy(),
                                          sample_count=int(self.count[i])),
                         provenance=dict(self.provenance))


_OD_ROWS = threading.local()     # sorted i0 values seen, their OD rows (host + per device)


def _od_tables_exact(i0: np.ndarray, device, i0_dev=None):
    """(n, 3, 256) fp64 OD tables (CUDA) with the reference's numpy expression
    (src/optics.py:89-94), evaluated once per distinct i0 value on the host —
    i0 are order statistics of 8-bit pools, so there are few, and a row
    depends on the value only — and expanded to the items on the device.
    The rows are memoised per thread (a pure function of the value): a batch
    whose values were all seen before only looks its items up — on the device
    when i0_dev (the same values, CUDA) is given (a host binary search per
    value costs ~30 ns x 3n)."""
    t = _dev.torch()
    dev = t.device(device)
    key = dev.index if dev.index is not None else t._C._cuda_getDevice()
    st = _OD_ROWS.__dict__
    vals = st.get("vals")
    u = np.unique(i0)
    hit = False
    if vals is not None and vals.size:
        pos = np.searchsorted(vals, u)
        hit = bool(np.all(vals[np.minimum(pos, vals.size - 1)] == u))
    st["last_hit"] = hit
    if not hit or key not in st.get("dev_rows", {}):
        new = u if vals is None else np.union1d(vals, u)
        if new.size > 4096:                      # bound the memo
            new = u
        ramp = np.arange(256, dtype=np.float64)
        rows = np.log(new[:, None] / np.clip(ramp[None, :], 1.0, new[:, None]))
        st["vals"] = new
        st["dev_rows"] = {key: (t.from_numpy(rows).to(dev), t.from_numpy(new).to(dev))}
    rows_d, vals_d = st["dev_rows"][key]
    if i0_dev is not None:
        d_idx = t.searchsorted(vals_d, i0_dev.reshape(-1).to(t.float64)).reshape(i0.shape)
    else:
        d_idx = t.from_numpy(np.searchsorted(st["vals"], i0).astype(np.int64)).to(dev)
    return rows_d[d_idx].contiguous()


def _od_rows_device(dev):
    """(rows, values) of the OD-row memo on this device when the last batch's
    values were all in it (worth speculating on), else None."""
    t = _dev.torch()
    d = t.device(dev)
    key = d.index if d.index is not None else t._C._cuda_getDevice()
    st = _OD_ROWS.__dict__
    if os.environ.get("SPCN_BATCH_SPECULATE", "1") == "0" or not st.get("last_hit", False):
        return None
    return st.get("dev_rows", {}).get(key)


_GRIDS = threading.local()         # memoised patch grids (pure functions of their key)


def _batch_grid(n, H, W, plan, dev):
    """The seeded visit order (same for every item: same grid, same seed),
    the candidate rectangles, the chunk count and the device patch
    descriptors of an (n, H, W) batch; memoised per thread (a few keys)."""
    key = (n, H, W, plan.patch_size, plan.seed, plan.max_patches, str(dev))
    memo = _GRIDS.__dict__.setdefault("m", {})
    got = memo.get(key)
    if got is not None:
        return got
    t = _dev.torch()
    origins = [(x, y) for y in range(0, H, plan.patch_size) for x in range(0, W, plan.patch_size)]
    order = np.random.default_rng(plan.seed).permutation(len(origins))
    ncand = min(len(order), 10 * plan.max_patches)
    rects = [(origins[i][0], origins[i][1], min(plan.patch_size, W - origins[i][0]),
              min(plan.patch_size, H - origins[i][1])) for i in order[:ncand]]
    desc = np.zeros((n, ncand), dtype=PATCH_DT)
    for k, (x, y, w, h) in enumerate(rects):
        desc["base"][:, k] = np.arange(n, dtype=np.int64) * (H * W) + y * W + x
        desc["width"][:, k] = w
        desc["height"][:, k] = h
        desc["row_stride"][:, k] = W
    desc = desc.ravel()
    chunks = max(1, -(-max(w * h for (_, _, w, h) in rects) // CHUNK))
    d_desc = t.from_numpy(desc.view(np.uint8).copy()).to(dev)
    got = (order, ncand, rects, chunks, d_desc)
    if len(memo) < 8:   # (never evicted: a launch on another stream may still read one)
        memo[key] = got
    return got


def fit_batch(images, plan: SamplePlan = SamplePlan(), cfg: SnmfConfig = SnmfConfig(), *,
              code_lam: float = 0.0) -> BatchFit:
    """fit() of every image of a (n, H, W, 3) uint8 CUDA tensor, all on the device."""
    t = _dev.torch()
    L = _lib_sample()
    if images.ndim != 4 or images.shape[3] != 3 or str(images.dtype) != "torch.uint8":
        raise ValueError("images must be an (n, H, W, 3) uint8 tensor")
    imgs = images.contiguous() if images.is_cuda else images.cuda().contiguous()
    n, H, W = int(imgs.shape[0]), int(imgs.shape[1]), int(imgs.shape[2])
    dev = imgs.device
    order, ncand, rects, chunks, d_desc = _batch_grid(n, H, W, plan, dev)
    counts = t.empty((n * ncand, chunks, 4), dtype=t.int32, device=dev)
    thr = int(plan.white_threshold)
    _lib.check(L.spcn_sample_count(_lib.ptr(imgs), _lib.ptr(d_desc), n * ncand, chunks, thr,
                                   _lib.ptr(counts), _lib.stream_handle()), "sample_count")
    if ncand == 1:
        return _fit_batch_single_patch(imgs, n, rects[0], d_desc, counts, chunks, thr, plan, cfg,
                                       code_lam)
    tot = _dev.readback(counts.sum(dim=1)).astype(np.int64).reshape(n, ncand, 4)
    # the reference's visit loop per item
    take_nw = np.zeros((n, ncand), np.int64)
    take_b = np.zeros((n, ncand, 3), np.int64)
    collected = np.zeros(n, np.int64)
    for i in range(n):
        takes, _uc, coll, _, _ = _visit(plan, order[:ncand], rects,
                                        lambda k, i=i: tuple(int(v) for v in tot[i, k]))
        for (k, tnw, _base, tb) in takes:
            take_nw[i, k] = tnw
            take_b[i, k] = tb
        collected[i] = coll
    offsets = np.concatenate([[0], np.cumsum(collected)]).astype(np.int64)
    total = int(offsets[-1])
    base_in_item = np.cumsum(take_nw, axis=1) - take_nw
    tk = np.zeros((n, ncand), dtype=TAKE_DT)
    tk["take_nonwhite"] = take_nw
    tk["out_base"] = offsets[:-1, None] + base_in_item
    tk["take_bright"] = take_b
    tk["problem"] = np.arange(n, dtype=np.int32)[:, None]
    sample = t.empty((max(total, 1), 3), dtype=t.uint8, device=dev)
    d_tk = t.from_numpy(tk.ravel().view(np.uint8).copy()).to(dev)
    i0, ie = _compact_i0(imgs, n, ncand, d_desc, counts, chunks, thr, d_tk, sample, None)
    return _fit_batch_tail(n, sample, collected, offsets, i0, ie, cfg, plan, code_lam)


def _compact_i0(imgs, n, ncand, d_desc, counts, chunks, thr, d_tk, sample, extra, read=True):
    """Ordered compaction + bright histograms, i0 per item, and ONE read of
    (i0, empty flags[, extra]) — extra: a device int64 vector appended.
    read=False: no read; returns (i0, the device vector that would be read)."""
    t = _dev.torch()
    L = _lib_sample()
    dev = imgs.device
    hist = t.zeros((n, 3, 256), dtype=t.int32, device=dev)
    _lib.check(L.spcn_sample_compact(_lib.ptr(imgs), _lib.ptr(d_desc), n * ncand, chunks, thr,
                                     _lib.ptr(counts), _lib.ptr(d_tk), _lib.ptr(sample),
                                     _lib.ptr(hist), _lib.stream_handle()), "sample_compact")
    # background i0 per item (exact order statistic of the 8-bit pools)
    i0 = t.empty((n, 3), dtype=t.float64, device=dev)
    empty = t.empty((n, 3), dtype=t.int32, device=dev)
    _lib.check(L.spcn_i0_from_hist(_lib.ptr(hist), n, _lib.ptr(i0), _lib.ptr(empty),
                                   _lib.stream_handle()), "i0_from_hist")
    parts = [i0.reshape(-1), empty.reshape(-1).to(t.float64)]
    if extra is not None:
        parts.append(extra.to(t.float64))             # counts < 2^53: exact in f64
    v = t.cat(parts)
    return (i0, _dev.readback(v)) if read else (i0, v)   # one read


def _fit_batch_single_patch(imgs, n, rect, d_desc, counts, chunks, thr, plan, cfg, code_lam):
    """fit_batch for a one-candidate grid (every item is one patch, e.g. 512²
    tiles with patch_size 1000): the reference's visit rules
    (src/pipeline.py:156-184) reduce to per-item ones, evaluated on the device
    (spcn_visit_single), so the counts are never read back — the compaction
    follows the count pass directly.  When every OD-table row the batch could
    need is likely memoised (the rows of earlier batches on this device), the
    SNMF, coding and p99 are enqueued right behind the compaction with the
    rows looked up on the device, and ONE read at the end brings back i0, the
    take sizes, the statuses and a flag telling whether every i0 value was
    memoised; if one was not, the tail re-runs with the exact rows."""
    t = _dev.torch()
    dev = imgs.device
    npx = rect[2] * rect[3]
    min_frac = 1.0 - plan.background_fraction_cutoff
    tk = t.empty((n, 8), dtype=t.int32, device=dev)               # TAKE_DT rows (32 B)
    take_nw = t.empty(n, dtype=t.int64, device=dev)
    L = _lib_sample()
    _lib.check(L.spcn_visit_single(_lib.ptr(counts), n, int(counts.shape[1]), min_frac * npx,
                                   int(plan.target_pixels), int(plan.sample_cap), _lib.ptr(tk),
                                   _lib.ptr(take_nw), _lib.stream_handle()), "visit_single")
    # the sample at its largest (every item taking target_pixels): no read of
    # the totals before the compaction
    per_max = min(plan.target_pixels, npx)
    sample = t.empty((max(1, n * per_max), 3), dtype=t.uint8, device=dev)
    memo = _od_rows_device(dev)
    i0, v = _compact_i0(imgs, n, 1, d_desc, counts, chunks, thr, tk.view(-1).view(t.uint8),
                        sample, take_nw, read=memo is None)
    if memo is None:                                  # cold: rows from the host values first
        ie = v
        collected = ie[6 * n:].astype(np.int64)
        offsets = np.concatenate([[0], np.cumsum(collected)]).astype(np.int64)
        total = int(offsets[-1])
        luts = _od_tables_exact(ie[:3 * n].reshape(n, 3), dev, i0)
        d_off = t.from_numpy(offsets).to(dev)
        flat = sample.reshape(-1)[:3 * max(total, 1)]
        r, p99, absent = _fit_batch_launch(n, flat, d_off, luts, cfg, code_lam,
                                           int(collected.max(initial=0)), total)
        ai = _dev.readback(t.cat([absent.reshape(-1), r.info.reshape(-1)]))
        return _fit_batch_finish(n, collected, i0, ie[:6 * n], r, p99, ai, luts, cfg, plan,
                                 code_lam, stacklevel=3)
    # speculative: device offsets, memoised rows looked up on the device
    d_off = t.zeros(n + 1, dtype=t.int64, device=dev)
    t.cumsum(take_nw, 0, out=d_off[1:])
    rows_d, vals_d = memo
    idx = t.searchsorted(vals_d, i0.reshape(-1)).clamp_(max=vals_d.numel() - 1)
    miss = (vals_d[idx] != i0.reshape(-1)).any().to(t.float64).reshape(1)
    luts = rows_d[idx.reshape(n, 3)].contiguous()
    total_cap = n * per_max
    r, p99, absent = _fit_batch_launch(n, sample.reshape(-1), d_off, luts, cfg, code_lam,
                                       per_max, total_cap)
    allv = _dev.readback(t.cat([v, miss, absent.reshape(-1).to(t.float64),
                                r.info.reshape(-1).to(t.float64)]))
    ie = allv[:7 * n]
    collected = ie[6 * n:].astype(np.int64)
    rest = allv[7 * n:]
    if rest[0] != 0:                                   # an i0 value without a memoised row
        luts = _od_tables_exact(ie[:3 * n].reshape(n, 3), dev, i0)   # (clears last_hit)
        r, p99, absent = _fit_batch_launch(n, sample.reshape(-1), d_off, luts, cfg, code_lam,
                                           per_max, total_cap)
        ai = _dev.readback(t.cat([absent.reshape(-1), r.info.reshape(-1)]))
    else:
        ai = rest[1:].astype(np.int64)
    return _fit_batch_finish(n, collected, i0, ie[:6 * n], r, p99, ai, luts, cfg, plan,
                             code_lam, stacklevel=3)


def _fit_batch_launch(n, flat, d_off, luts, cfg, code_lam, mmax, total):
    """Enqueue the SNMF (over per-item colour tables), the densities of every
    distinct colour and the weighted p99.  `total` is the sample's length
    (the colour-table layout; entries past an item's offsets are not read)."""
    t = _dev.torch()
    r = snmf.snmf_batched(flat, d_off, luts, cfg, cluster=1)
    if r.table is not None and total > 0:
        # densities and p99 over the SNMF's colour table: one fp64 coding per
        # distinct colour, weighted exact select (same values as per sample)
        h = snmf.code_table(r.table, d_off, luts, r.basis, code_lam, mmax, total)
        p99, absent = snmf.percentile_table(h, r.table, d_off, total, 99.0)
    else:
        from . import stats as dstats

        h = snmf.code_samples(flat, d_off, luts, r.basis, code_lam, mmax)
        p99, absent = dstats.segment_percentiles(h, d_off, 99.0)
    if absent.dtype != t.int32:
        absent = absent.to(t.int32)
    return r, p99, absent


def _fit_batch_finish(n, collected, i0, ie, r, p99, ai, luts, cfg, plan, code_lam, stacklevel):
    """Statuses, warnings and the BatchFit from the host reads."""
    status = np.zeros(n, np.int32)
    status[collected == 0] = -_lib.SPCN_EBLANK
    status[(collected > 0) & (collected < 10)] = -_lib.SPCN_EINSUFFICIENT
    if ie[3 * n:6 * n].any():
        warnings.warn("some items had no pixels brighter than the white threshold in a "
                      "channel; their i0 fell back to 255", optics.BackgroundEstimateWarning,
                      stacklevel=stacklevel + 1)
    absent_h = ai[:2 * n].reshape(n, 2).any(axis=1)
    info = ai[2 * n:].reshape(n, -1)
    status[(status == 0) & absent_h] = -_lib.SPCN_ESTAIN_ABSENT
    prov = {"source": "", "config_hash": config_hash(_cfg_fields(plan, cfg, code_lam, False))}
    return BatchFit(i0=i0, basis=r.basis, p99=p99, luts=luts, count=collected, status=status,
                    provenance=prov, iterations=info[:, 0].copy(), converged=info[:, 1] != 0,
                    warn_flags=info[:, 2].copy())


def _fit_batch_tail(n, sample, collected, offsets, i0, ie, cfg, plan, code_lam, stacklevel=3):
    """From the sample and i0 on (host offsets): OD tables, SNMF, densities,
    p99, statuses."""
    t = _dev.torch()
    dev = sample.device
    total = int(offsets[-1])
    luts = _od_tables_exact(ie[:3 * n].reshape(n, 3), dev, i0)
    d_off = t.from_numpy(offsets).to(dev)
    flat = sample.reshape(-1)[:3 * max(total, 1)]
    r, p99, absent = _fit_batch_launch(n, flat, d_off, luts, cfg, code_lam,
                                       int(collected.max(initial=0)), total)
    ai = _dev.readback(t.cat([absent.reshape(-1), r.info.reshape(-1)]))   # one read
    return _fit_batch_finish(n, collected, i0, ie, r, p99, ai, luts, cfg, plan, code_lam,
                             stacklevel)


def transform_batch(images, fits: BatchFit, target: FitParams, out=None, *,
                    code_lam: float = 0.0, precision: str = "exact", max_sweeps: int = 2000):
    """Recolour every item against `target`.  Returns (out, errors) where
    errors[i] is None or the exception the reference would have raised."""
    t = _dev.torch()
    L = _sig()
    if precision not in _lib.PREC:
        raise ValueError(f"precision must be one of {sorted(_lib.PREC)}")
    imgs = images.contiguous()
    n = int(imgs.shape[0])
    per = int(imgs.shape[1]) * int(imgs.shape[2])
    dev = imgs.device
    out = out if out is not None else t.empty_like(imgs)
    fs_b, sp_b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    L.spcn_batch_sizes(ctypes.byref(fs_b), ctypes.byref(sp_b))
    fast = t.empty(n * fs_b.value, dtype=t.uint8, device=dev)
    strict = t.empty(n * sp_b.value, dtype=t.uint8, device=dev)
    flut = t.empty((n, 3, 256), dtype=t.float32, device=dev)
    status = t.from_numpy(fits.status.astype(np.int32)).to(dev)
    tg = BatchTargetC()
    tg.i0[:] = [float(x) for x in np.asarray(target.i0, dtype=np.float64)]
    tg.basis[:] = [float(x) for x in np.asarray(target.basis, dtype=np.float64).ravel()]
    tg.p99[:] = [float(x) for x in np.asarray(target.stats.p99, dtype=np.float64)]
    _lib.check(L.spcn_batch_params(n, _lib.ptr(fits.i0), _lib.ptr(fits.luts),
                                   _lib.ptr(fits.basis.contiguous()), _lib.ptr(fits.p99),
                                   ctypes.byref(tg), float(code_lam), int(max_sweeps),
                                   _lib.PREC[precision], _lib.ptr(fast), _lib.ptr(flut),
                                   _lib.ptr(strict), _lib.ptr(status), _lib.stream_handle()),
               "batch_params")
    if precision == "strict":
        status = t.where(status == 0, t.ones_like(status), status)
    status_h = _dev.readback(status)
    errors = [None] * n
    for i in np.flatnonzero(status_h < 0):
        errors[i] = _ERR[int(status_h[i])](_MSG[int(status_h[i])])
    if per % 16:
        # item boundaries not 16-pixel aligned: one aligned-head/tail launch per item
        for i in range(n):
            if status_h[i] < 0:
                continue
            fp = fits.params(i)
            fac = np.asarray(target.stats.p99, dtype=np.float64) / fp.stats.p99
            XformPlan(fp.i0, fp.basis, code_lam, fac, target.basis, target.i0,
                      precision=precision).run(imgs[i], out[i], per)
        return out, errors
    off = np.arange(n + 1, dtype=np.int64) * per
    d_off = t.from_numpy(off).to(dev)
    # items are small (no exhaustive calibration): the analytic bound can flag a
    # few % of pixels, so size the repair list for 1/8 of them (1 B/px)
    ws_bytes = max(int(_lib.lib().spcn_xform_workspace_bytes(n * per)),
                   16 + 8 * (65536 + n * per // 8))
    ws = _dev.workspace(ws_bytes)
    # (the host statuses skip the launches nothing needs; the read-back before
    # the launch also keeps normalize_batch_host's chunk pipeline flowing)
    _lib.check(L.spcn_xform_batch(_lib.ptr(imgs), _lib.ptr(out), n, off.ctypes.data,
                                  _lib.ptr(d_off), _lib.ptr(fast), status_h.ctypes.data,
                                  _lib.ptr(status), _lib.ptr(flut), _lib.ptr(strict),
                                  _lib.PREC[precision], _lib.ptr(ws), ws_bytes,
                                  _lib.stream_handle()), "xform_batch")
    return out, errors


def normalize_batch(images, target, *, plan: SamplePlan = SamplePlan(),
                    cfg: SnmfConfig = SnmfConfig(), code_lam: float = 0.0,
                    precision: str = "exact", out=None):
    """fit_batch + transform_batch: the batch equivalent of ``normalize``.
    ``target`` is a FitParams (e.g. a loaded profile)."""
    fits = fit_batch(images, plan, cfg, code_lam=code_lam)
    out, errors = transform_batch(images, fits, target, out, code_lam=code_lam,
                                  precision=precision)
    return out, errors, fits


_HOST_STREAMS = threading.local()
_SLICE_BYTES = 64 << 20


def _sliced_copy(dst, src, non_blocking):
    """dst.copy_(src) as <= 64 MB pieces: a copy engine serves its queue in
    order, so one 800 MB transfer would hold up the fit's small read-backs
    (issued from another stream) until it finished; between pieces they
    interleave."""
    per = max(1, _SLICE_BYTES // max(1, src[0].numel())) if src.shape[0] else 1
    for i in range(0, src.shape[0], per):
        dst[i:i + per].copy_(src[i:i + per], non_blocking=non_blocking)


def normalize_batch_host(images, target, out=None, *, chunk: int = 256, streams: int = 6,
                         plan: SamplePlan = SamplePlan(), cfg: SnmfConfig = SnmfConfig(),
                         code_lam: float = 0.0, precision: str = "exact"):
    """normalize_batch for a host-resident batch ((n, H, W, 3) uint8 numpy array
    or CPU tensor; pinned memory gives asynchronous copies): chunks of
    ``chunk`` items rotate over ``streams`` CUDA streams so the H2D copy of one
    chunk, the fit + recolour of another and the D2H copy of a third overlap —
    cmd_batch's loop over files (src/cli.py:270-301) as a pipeline.  Returns
    (out, errors) with errors in item order."""
    t = _dev.torch()
    host = images if _dev.is_tensor(images) else t.from_numpy(np.ascontiguousarray(images))
    if host.ndim != 4 or host.shape[3] != 3:
        raise ValueError("images must be an (n, H, W, 3) uint8 batch")
    n = int(host.shape[0])
    if out is None:
        out = t.empty(host.shape, dtype=t.uint8, pin_memory=host.is_pinned())
    elif not _dev.is_tensor(out):
        out = t.from_numpy(out)
    pinned = host.is_pinned() and out.is_pinned()
    starts = list(range(0, n, chunk))
    # streams persist per thread: the caching allocator keeps freed blocks per
    # stream, so fresh streams on every call would cudaMalloc (synchronously)
    # every buffer again and never reuse the cached ones
    pool = _HOST_STREAMS.__dict__.setdefault("streams", [])
    while len(pool) < max(2, streams):
        pool.append(t.cuda.Stream())
    slots = [dict(stream=pool[i], done=None, d_in=None) for i in range(max(2, streams))]

    def upload(k):                       # H2D of chunk k on its slot's stream
        slot = slots[k % len(slots)]
        if slot["done"] is not None:
            slot["done"].synchronize()   # the chunk that used this slot has left the GPU
        a, b = starts[k], min(n, starts[k] + chunk)
        with t.cuda.stream(slot["stream"]):
            d = t.empty(host[a:b].shape, dtype=t.uint8, device="cuda")
            _sliced_copy(d, host[a:b], pinned)
            slot["d_in"] = d

    errors = [None] * n
    ahead = max(1, min(int(os.environ.get("SPCN_BATCH_AHEAD", "2")), len(slots) - 2))
    for k in range(min(ahead, len(starts))):
        upload(k)
    for k, a in enumerate(starts):
        b = min(n, a + chunk)
        if k + ahead < len(starts):
            upload(k + ahead)            # later chunks' copies overlap this chunk's compute
        slot = slots[k % len(slots)]
        with t.cuda.stream(slot["stream"]):
            d_in = slot["d_in"]
            fits = fit_batch(d_in, plan, cfg, code_lam=code_lam)
            d_out, errs = transform_batch(d_in, fits, target, code_lam=code_lam,
                                          precision=precision)
            _sliced_copy(out[a:b], d_out, pinned)
            ev = t.cuda.Event()
            ev.record(slot["stream"])
        slot["done"] = ev
        errors[a:b] = errs
    for slot in slots:
        if slot["done"] is not None:
            slot["done"].synchronize()
    return out, errors
