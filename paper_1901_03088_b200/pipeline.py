"""Whole-slide orchestration on the device: sample → i0 → SNMF → p99 → transform.

Mirrors src/pipeline.py:1-345 (same functions, arguments, defaults, errors
and stage labels).  The per-pixel work is libspcn (CUDA); the host keeps the
reference's sequential control logic where it is O(patches): the seeded patch
visit order (numpy PCG64, identical to src/pipeline.py:138-142) and the
visit/stop rules (src/pipeline.py:156-184), replayed on per-patch counts the
GPU produced.
"""
from __future__ import annotations

import ctypes
import functools
import os
import time
import warnings
from collections import deque
from dataclasses import dataclass
import threading
from threading import Lock

import numpy as np

from . import _dev, _lib, optics
from .errors import BlankSlideError, DegenerateStainError, SlideNormError
from .image_io import (DEFAULT_STRIP_HEIGHT, ArraySource, ArrayWriter, DeviceSource, DeviceWriter,
                       PixelBlock, plan_strips)
from .normalize import FitParams, scale_factors
from .optics import SAMPLE_CAP, WHITE_THRESHOLD
from .stain_sep import SnmfConfig
from .xform import XformPlan

PATCH_DT = np.dtype([("base", "<i8"), ("width", "<i4"), ("height", "<i4"), ("row_stride", "<i8")])
TAKE_DT = np.dtype([("take_nonwhite", "<i8"), ("out_base", "<i8"), ("take_bright", "<i4", (3,)),
                    ("problem", "<i4")])
CHUNK = 4096  # SPCN_SAMPLE_CHUNK


@dataclass(frozen=True)
class SamplePlan:
    """How to gather the fitting sample from a slide (src/pipeline.py:39-59)."""

    max_patches: int = 20
    patch_size: int = 1000
    target_pixels: int = 100_000
    background_fraction_cutoff: float = 0.95
    seed: int = 0
    white_threshold: int = WHITE_THRESHOLD
    sample_cap: int = SAMPLE_CAP

    def __post_init__(self):
        if self.max_patches < 1:
            raise ValueError("max_patches must be >= 1")
        if self.target_pixels < 1:
            raise ValueError("target_pixels must be >= 1")
        if not 0.0 < self.background_fraction_cutoff <= 1.0:
            raise ValueError("background_fraction_cutoff must be in (0, 1]")
        if self.patch_size < 1:
            raise ValueError("patch_size must be >= 1")


@dataclass
class PixelSample:
    """Pixels gathered by :func:`sample_pixels` (src/pipeline.py:62-70)."""

    non_white: object              # (M, 3) uint8 (numpy from sample_pixels; CUDA inside fit)
    patch_counts: list
    bright: tuple                  # three 1-D arrays (sample_pixels) or None (device path)
    patches_visited: int = 0
    patches_used: int = 0
    bright_hist: np.ndarray = None  # (3, 256) counts of the bright pools


@dataclass
class RunStats:
    """Per-stage wall times and counters (src/pipeline.py:73-99)."""

    sampling_s: float = 0.0
    basis_fit_s: float = 0.0
    transform_s: float = 0.0
    total_s: float = 0.0
    sampled_pixels: int = 0
    transformed_pixels: int = 0
    patches: int = 0
    peak_strip_pixels: int = 0

    CSV_HEADER = "stage,seconds,pixels,patches"

    def csv_rows(self):
        return [("sampling", self.sampling_s, self.sampled_pixels, self.patches),
                ("basis_fit", self.basis_fit_s, self.sampled_pixels, self.patches),
                ("transform", self.transform_s, self.transformed_pixels, self.patches),
                ("total", self.total_s, self.transformed_pixels, self.patches)]

    def write_csv(self, fh):
        fh.write(self.CSV_HEADER + "\n")
        for stage, seconds, pixels, patches in self.csv_rows():
            fh.write(f"{stage},{seconds:.6f},{pixels},{patches}\n")


class BufferGauge:
    """Thread-safe gauge of pixels held in in-flight strip buffers (src/pipeline.py:102-118)."""

    def __init__(self):
        self._lock = Lock()
        self.current = 0
        self.peak = 0

    def add(self, pixels: int):
        with self._lock:
            self.current += pixels
            self.peak = max(self.peak, self.current)

    def release(self, pixels: int):
        with self._lock:
            self.current -= pixels


def _stage(label, fn, *args, **kwargs):
    """src/pipeline.py:121-125: prefix domain errors with the stage label."""
    try:
        return fn(*args, **kwargs)
    except SlideNormError as exc:
        raise type(exc)(f"{label}: {exc}") from exc


# ----------------------------------------------------------------------------- sampling
def _lib_sample():
    L = _lib.lib()
    if not getattr(L, "_spcn_sample_declared", False):
        P, I32 = _lib.P, _lib.I32
        _lib.declare("spcn_sample_count", _lib.ctypes.c_int, [P, P, I32, I32, I32, P, P])
        _lib.declare("spcn_sample_compact", _lib.ctypes.c_int, [P, P, I32, I32, I32, P, P, P, P, P])
        _lib.declare("spcn_i0_from_hist", _lib.ctypes.c_int, [P, I32, P, P, P])
        _lib.declare("spcn_od_tables", _lib.ctypes.c_int, [P, I32, P, P])
        _lib.declare("spcn_visit_single", _lib.ctypes.c_int,
                     [P, I32, I32, _lib.DBL, _lib.I64, _lib.I64, P, P, P])
        L._spcn_sample_declared = True
    return L


class _PatchImage:
    """Device view of the slide regions the sampler may visit.  A device slide
    is addressed in place; for a host slide only the regions of the batches
    the visit loop actually counts are uploaded (usually the first few of the
    10 x max_patches candidates)."""

    def __init__(self, slide, rects):
        self.rects = rects
        self.slide = slide
        self.device = isinstance(slide, DeviceSource)
        if self.device:
            width = slide.width
            self.img = slide.tensor
            self.desc = np.array([(y * width + x, w, h, width) for (x, y, w, h) in rects],
                                 dtype=PATCH_DT)

    def batch(self, lo, hi):
        """(device image, descriptors) of candidates [lo, hi)."""
        if self.device:
            return self.img, self.desc[lo:hi]
        desc, base = [], 0
        for (x, y, w, h) in self.rects[lo:hi]:
            desc.append((base, w, h, w))
            base += w * h
        arr = self.slide.array if isinstance(self.slide, ArraySource) else None

        def fill(stage):   # each region straight into the pinned buffer (one copy)
            off = 0
            for (x, y, w, h) in self.rects[lo:hi]:
                dst = stage[3 * off:3 * (off + w * h)].reshape(h, w, 3)
                _pcopy(dst, arr[y:y + h, x:x + w] if arr is not None else
                       self.slide.read_region(x, y, w, h).pixels)
                off += w * h

        return _STAGING.to_device_fill(max(3 * base, 3), fill), np.array(desc, dtype=PATCH_DT)


def _count(L, img, desc, thr):
    """Per-chunk counts for the patches `desc` of `img` → (n, chunks, 4)."""
    t = _dev.torch()
    npx = desc["width"].astype(np.int64) * desc["height"]
    chunks = int(max(1, -(-int(npx.max()) // CHUNK)))
    d = t.from_numpy(desc.view(np.uint8).copy()).cuda()
    out = t.empty((len(desc), chunks, 4), dtype=t.int32, device="cuda")
    _lib.check(L.spcn_sample_count(_lib.ptr(img), _lib.ptr(d), len(desc), chunks, thr,
                                   _lib.ptr(out), _lib.stream_handle()), "sample_count")
    return out, chunks


def _visit(plan, order, rects, counts_of):
    """Replay src/pipeline.py:156-184 on per-patch totals.  counts_of(i) → (nw, bR, bG, bB)."""
    limit = 10 * plan.max_patches
    min_frac = 1.0 - plan.background_fraction_cutoff
    collected = visited = used = 0
    bright_n = [0, 0, 0]
    takes, used_counts = [], []
    for k, idx in enumerate(order):
        if visited >= limit or used >= plan.max_patches:
            break
        if collected >= plan.target_pixels:
            break
        nw, b0, b1, b2 = counts_of(k)
        x, y, w, h = rects[k]
        visited += 1
        tb = [0, 0, 0]
        for c, bc in enumerate((b0, b1, b2)):
            if bright_n[c] < plan.sample_cap:
                tb[c] = int(min(bc, plan.sample_cap - bright_n[c]))
                bright_n[c] += tb[c]
        if nw < min_frac * (w * h):
            takes.append((k, 0, 0, tb))
            continue
        used += 1
        take = int(min(nw, plan.target_pixels - collected))
        takes.append((k, take, collected, tb))
        used_counts.append(take)
        collected += take
    return takes, used_counts, collected, visited, used


@functools.lru_cache(maxsize=32)
def _candidates(width: int, height: int, plan: SamplePlan):
    """The seeded visit order of the patch grid (src/pipeline.py:138-142):
    (order, ncand, rects of the first ncand candidates).  Memoised: a pure
    function of the geometry and the plan (callers do not modify it)."""
    ps = plan.patch_size
    ncols, nrows = -(-width // ps), -(-height // ps)
    order = np.random.default_rng(plan.seed).permutation(ncols * nrows)
    ncand = min(len(order), 10 * plan.max_patches)
    first = order[:ncand]
    xs, ys = (first % ncols) * ps, (first // ncols) * ps
    rects = [(int(x), int(y), int(min(ps, width - x)), int(min(ps, height - y)))
             for x, y in zip(xs, ys)]
    return order, ncand, rects


_VISIT_PLAN = None


def _visit_plan_type():
    global _VISIT_PLAN
    if _VISIT_PLAN is None:
        import ctypes

        class VisitPlan(ctypes.Structure):
            _fields_ = [("target_pixels", ctypes.c_int64), ("sample_cap", ctypes.c_int64),
                        ("max_patches", ctypes.c_int32), ("ncand", ctypes.c_int32),
                        ("background_cutoff", ctypes.c_double)]

        _VISIT_PLAN = VisitPlan
        P, I32 = _lib.P, _lib.I32
        _lib.declare("spcn_sample_visit", _lib.ctypes.c_int,
                     [P, I32, I32, I32, P, _lib.ctypes.POINTER(VisitPlan), P, P, P, P])
    return _VISIT_PLAN


_VISIT_BATCH_MAX = 1024   # candidates per k_visit launch (its totals live in shared memory)


def _resident_candidates(fb, slide: DeviceSource, plan: SamplePlan):
    """Candidate patches of a resident slide geometry on the device (memoised
    per (width, height, plan) in the fit buffers: a pure function of them)."""
    key = (slide.width, slide.height, plan)
    c = fb.cand.get(key)
    if c is None:
        t = _dev.torch()
        VisitPlan = _visit_plan_type()
        order, ncand, rects = _candidates(slide.width, slide.height, plan)
        W = slide.width
        desc = np.array([(y * W + x, w, h, W) for (x, y, w, h) in rects], dtype=PATCH_DT)
        dims = np.array([(w, h) for (_, _, w, h) in rects], dtype=np.int32)
        npx = dims[:, 0].astype(np.int64) * dims[:, 1]
        chunks = int(max(1, -(-int(npx.max()) // CHUNK)))
        batches, k0, n = [], 0, min(ncand, max(2, min(plan.max_patches, 8)))
        while k0 < ncand:
            n = min(n, ncand - k0, _VISIT_BATCH_MAX)
            batches.append((k0, n))
            k0 += n
            n *= 2
        c = dict(ncand=ncand, chunks=chunks, batches=batches,
                 desc=t.from_numpy(desc.view(np.uint8).copy()).to(fb.device),
                 dims=t.from_numpy(dims).to(fb.device),
                 takes=t.zeros(ncand * TAKE_DT.itemsize, dtype=t.uint8, device=fb.device),
                 counts=t.empty(max(n for _, n in batches) * chunks * 4, dtype=t.int32,
                                device=fb.device),
                 vp=VisitPlan(plan.target_pixels, plan.sample_cap, plan.max_patches, ncand,
                              float(plan.background_fraction_cutoff)))
        for k in ("desc", "dims", "takes", "counts"):
            c[k + "_ptr"] = _lib.ptr(c[k])
        if len(fb.cand) > 16:
            fb.cand.clear()
        fb.cand[key] = c
    return c


def _sample_batch(fb, slide: DeviceSource, plan: SamplePlan, c, k0: int, n: int) -> None:
    """count -> visit -> compact -> i0 -> read-back of candidates [k0, k0+n),
    one library call, stream-ordered (the first batch zeroes the arena)."""
    import ctypes

    from .fitcore import A_READ

    _lib.check(_lib.lib().spcn_fit_sample_step(
        _lib.ptr(slide.tensor), c["desc_ptr"] + k0 * PATCH_DT.itemsize, n, c["chunks"], k0,
        c["dims_ptr"] + 8 * k0, ctypes.byref(c["vp"]), int(plan.white_threshold),
        1 if k0 == 0 else 0, fb.arena_a_ptr, c["counts_ptr"],
        c["takes_ptr"] + k0 * TAKE_DT.itemsize, fb.sample_ptr, fb.pin_a_ptr, A_READ,
        _lib.stream_handle()), "fit_sample_step")


def _sample_start(fb, slide: DeviceSource, plan: SamplePlan):
    """Enqueue the first candidate batch of a resident slide's sampling (no
    wait); _fit_sample_resident(..., started=<this>) finishes it."""
    c = _resident_candidates(fb, slide, plan)
    k0, n = c["batches"][0]
    _sample_batch(fb, slide, plan, c, k0, n)
    return c


def _fit_sample_resident(fb, slide: DeviceSource, plan: SamplePlan, need_counts: bool = False,
                         started=None):
    """Sampling + i0 of a device-resident slide with ONE host read in the
    common case: count → visit loop (k_visit, on the device) → ordered
    compaction → i0, then a single read of (state, i0, empty flags).  A
    further candidate batch runs only when the first ran out before a stop
    rule fired.  Returns (m, i0, PixelSample meta, empty flags); the sample is
    fb.sample[:3m]."""
    L = _lib.lib()
    c = started if started is not None else _resident_candidates(fb, slide, plan)
    stream = _lib.stream_handle()
    from .fitcore import A_READ

    for i, (k0, n) in enumerate(c["batches"]):
        if i > 0 or started is None:
            _sample_batch(fb, slide, plan, c, k0, n)
        _lib.check(L.spcn_stream_sync(stream), "stream_sync")
        raw = fb.pin_a_np[:A_READ].copy()
        st = raw[:64].view(np.int64)
        if not st[7]:                              # a stop rule fired (or all candidates seen)
            break
    from .fitcore import A_EMPTY, A_I0

    m = int(st[0])
    used_counts = []
    if need_counts:                                # per-patch stats only (one more read)
        tk = np.frombuffer(c["takes"][:(k0 + n) * TAKE_DT.itemsize].cpu().numpy().tobytes(),
                           dtype=TAKE_DT)
        used_counts = [int(v) for v in tk["take_nonwhite"] if v > 0]
    meta = PixelSample(non_white=None, patch_counts=used_counts,     # sample: fb.sample[:3m]
                       bright=None, patches_visited=int(st[1]), patches_used=int(st[2]),
                       bright_hist=None)
    i0 = raw[A_I0:A_EMPTY].view(np.float64).copy()
    empty = raw[A_EMPTY:A_EMPTY + 12].view(np.int32).astype(bool)
    return m, i0, meta, empty


def _sample_device(slide, plan: SamplePlan):
    """Device sampling; returns (sample CUDA uint8 (M,3), PixelSample meta)."""
    t = _dev.torch()
    L = _lib_sample()
    order, ncand, rects = _candidates(slide.width, slide.height, plan)
    pimg = _PatchImage(slide, rects)
    thr = int(plan.white_threshold)
    # counts in growing batches (most slides stop after one or two patches; a
    # host slide uploads only the batches it counts, so it starts with one)
    tot = np.zeros((0, 4), dtype=np.int64)
    dev_counts = []
    batch = min(ncand, max(2, min(plan.max_patches, 8))) if pimg.device else 1

    def counts_of(k):
        nonlocal tot, batch
        while k >= tot.shape[0]:
            lo = tot.shape[0]
            hi = min(ncand, lo + batch)
            img, desc = pimg.batch(lo, hi)
            c, chunks = _count(L, img, desc, thr)
            dev_counts.append((lo, hi, c, chunks, img, desc))
            tot = np.concatenate([tot, c.sum(dim=1).cpu().numpy().astype(np.int64)])
            batch = min(2 * batch, _VISIT_BATCH_MAX)
        return tuple(int(v) for v in tot[k])

    takes, used_counts, collected, visited, used = _visit(plan, order[:ncand], rects, counts_of)
    if collected == 0:
        raise BlankSlideError("blank slide: no non-white pixels found in any sampled patch")
    sample = t.empty((collected, 3), dtype=t.uint8, device="cuda")
    hist = t.zeros((1, 3, 256), dtype=t.int32, device="cuda")
    for lo, hi, c, chunks, img, bdesc in dev_counts:
        sel = [tk for tk in takes if lo <= tk[0] < hi and (tk[1] > 0 or any(tk[3]))]
        if not sel:
            continue
        idx = np.array([tk[0] - lo for tk in sel], dtype=np.int64)
        desc = bdesc[idx]
        tk = np.zeros(len(sel), dtype=TAKE_DT)
        tk["take_nonwhite"] = [s[1] for s in sel]
        tk["out_base"] = [s[2] for s in sel]
        tk["take_bright"] = [s[3] for s in sel]
        tk["problem"] = 0
        cnt = c[t.from_numpy(idx).cuda()].contiguous()
        d = t.from_numpy(desc.view(np.uint8).copy()).cuda()
        dt = t.from_numpy(tk.view(np.uint8).copy()).cuda()
        _lib.check(L.spcn_sample_compact(_lib.ptr(img), _lib.ptr(d), len(sel), chunks, thr,
                                         _lib.ptr(cnt), _lib.ptr(dt), _lib.ptr(sample),
                                         _lib.ptr(hist), _lib.stream_handle()), "sample_compact")
    bh = hist.cpu().numpy()[0].astype(np.int64)
    meta = PixelSample(non_white=sample, patch_counts=used_counts, bright=None,
                       patches_visited=visited, patches_used=used, bright_hist=bh)
    return sample, meta


def sample_pixels(slide, plan: SamplePlan = SamplePlan()) -> PixelSample:
    """src/pipeline.py:128-200 (device sampling; numpy result like the reference).

    ``bright`` holds the pools as value-sorted arrays (the multiset the
    reference keeps; i0 only depends on it through an order statistic)."""
    sample, meta = _sample_device(slide, plan)
    meta.non_white = sample.cpu().numpy()
    meta.bright = tuple(np.repeat(np.arange(256, dtype=np.uint8), meta.bright_hist[c])
                        for c in range(3))
    return meta


# ----------------------------------------------------------------------------- fit
def _cfg_fields(plan, cfg, code_lam, per_patch_stats):
    from .fitcore import cfg_fields

    return cfg_fields(plan, cfg, code_lam, per_patch_stats)


def slide_chunks(slide, rows: int = 2048):
    """Callable yielding the slide as flat CUDA uint8 runs (for whole-slide
    passes): a device slide in one piece, a host slide strip by strip through
    one reusable device buffer (stream-ordered reuse)."""
    t = _dev.torch()

    def gen():
        if isinstance(slide, DeviceSource):
            x = slide.tensor.reshape(-1)
            if not x.is_contiguous() or x.data_ptr() % 16:
                x = x.contiguous().clone()
            yield x
            return
        buf = t.empty(rows * slide.width * 3, dtype=t.uint8, device="cuda")
        for y in range(0, slide.height, rows):
            h = min(rows, slide.height - y)
            px = np.ascontiguousarray(slide.read_region(0, y, slide.width, h).pixels).reshape(-1)
            buf[:px.size].copy_(t.from_numpy(px), non_blocking=_pinned(px))
            yield buf[:px.size]
    return gen


def _fit_sample_checked(fb, slide: DeviceSource, plan: SamplePlan, need_counts: bool,
                        started=None):
    """Resident slide: visit loop + i0 on the device (one host round trip),
    with the reference's blank-slide error and background warnings."""
    with _dev.nvtx("spcn.fit.sample"):
        m, i0, meta, empty = _stage("sampling", _fit_sample_resident, fb, slide, plan,
                                    need_counts, started=started)
    if m == 0:
        raise BlankSlideError("sampling: blank slide: no non-white pixels found in any "
                              "sampled patch")
    for c in np.flatnonzero(empty):
        warnings.warn(f"no pixels brighter than the white threshold in the "
                      f"{('red', 'green', 'blue')[c]} channel; falling back to 255",
                      optics.BackgroundEstimateWarning, stacklevel=4)
    return m, i0, meta


def fit(slide, plan: SamplePlan = SamplePlan(), cfg: SnmfConfig = SnmfConfig(), *,
        code_lam: float = 0.0, per_patch_stats: bool = False, source_label: str = "",
        stats: RunStats | None = None, p99_mode: str = "sample") -> FitParams:
    """src/pipeline.py:203-257 on the device.

    p99_mode="sample" (default) is the reference; "global" takes the p99 over
    the densities of every non-white pixel of the slide (global_stats.py)."""
    if p99_mode not in ("sample", "global"):
        raise ValueError("p99_mode must be 'sample' or 'global'")
    t = _dev.torch()
    stats = stats if stats is not None else RunStats()
    if isinstance(slide, np.ndarray):
        slide = ArraySource(slide)
    elif _dev.is_tensor(slide):
        slide = DeviceSource(slide)
    from . import fitcore

    fb = fitcore.buffers(slide.tensor.device if isinstance(slide, DeviceSource) else "cuda",
                         plan.target_pixels, cfg.max_outer_iters)
    t0 = time.perf_counter()
    if isinstance(slide, DeviceSource):
        m, i0, meta = _fit_sample_checked(fb, slide, plan, per_patch_stats)
        sample_flat = fb.sample[:3 * m]
        stats.sampling_s += time.perf_counter() - t0
        t0 = time.perf_counter()
    else:
        sample, meta = _stage("sampling", _sample_device, slide, plan)
        stats.sampling_s += time.perf_counter() - t0
        m = int(sample.shape[0])
        t0 = time.perf_counter()
        i0 = _stage("background estimation", optics.i0_from_counts, meta.bright_hist)
        sample_flat = sample.reshape(-1)
        fb.offsets().copy_(t.tensor([0, m], dtype=t.int64), non_blocking=False)
    stats.sampled_pixels = m
    stats.patches = meta.patches_used
    with _dev.nvtx("spcn.fit.basis_stats"):
        fp = fitcore.fit_tail(fb, sample_flat, m, i0, plan, cfg, code_lam=code_lam,
                              per_patch_stats=per_patch_stats, p99_mode=p99_mode,
                              used_counts=meta.patch_counts, source_label=source_label,
                              chunks=slide_chunks(slide) if p99_mode == "global" else None,
                              stage=_stage)
    stats.basis_fit_s += time.perf_counter() - t0
    return fp


# ----------------------------------------------------------------------------- transform
class _Staging(threading.local):
    """Per-thread reusable stream + device/pinned buffers of the streamed
    transform's slots (and the host fit's upload buffer): allocating pinned
    memory and streams on every call costs more than a 2048^2 tile's work."""

    def __init__(self):
        self.slots = []       # dicts: stream, dsrc, ddst, hin, hout (flat uint8, grow-only)
        self.upload = None    # pinned flat uint8
        self.upload_ev = None

    @staticmethod
    def _grow(buf, nbytes, pinned):
        t = _dev.torch()
        if buf is not None and buf.numel() >= nbytes:
            return buf
        if pinned:
            return t.empty(nbytes, dtype=t.uint8, pin_memory=True)
        return t.empty(nbytes, dtype=t.uint8, device="cuda")

    def slot(self, k, nbytes, want_hin, want_hout):
        t = _dev.torch()
        while len(self.slots) <= k:
            self.slots.append(dict(stream=t.cuda.Stream(), dsrc=None, ddst=None, hin=None,
                                   hout=None))
        sl = self.slots[k]
        if sl["stream"].device != t.device("cuda", t.cuda.current_device()):
            sl.update(stream=t.cuda.Stream(), dsrc=None, ddst=None)
        sl["dsrc"] = self._grow(sl["dsrc"], nbytes, False)
        sl["ddst"] = self._grow(sl["ddst"], nbytes, False)
        if want_hin:
            sl["hin"] = self._grow(sl["hin"], nbytes, True)
        if want_hout:
            sl["hout"] = self._grow(sl["hout"], nbytes, True)
        return sl

    def to_device_fill(self, nbytes: int, fill):
        """Upload nbytes written by fill(pinned flat numpy view)."""
        t = _dev.torch()
        if self.upload_ev is not None:
            self.upload_ev.synchronize()      # the previous upload has left the buffer
        self.upload = self._grow(self.upload, nbytes, True)
        stage = self.upload[:nbytes]
        fill(stage.numpy())
        out = stage.to("cuda", non_blocking=True)
        self.upload_ev = t.cuda.Event()
        self.upload_ev.record()
        return out

    def to_device(self, host: np.ndarray):
        """Upload a contiguous uint8 array through the reusable pinned buffer."""
        t = _dev.torch()
        flat = host.reshape(-1)
        if self.upload_ev is not None:
            self.upload_ev.synchronize()      # the previous upload has left the buffer
        self.upload = self._grow(self.upload, flat.size, True)
        stage = self.upload[:flat.size]
        stage.numpy()[...] = flat
        out = stage.to("cuda", non_blocking=True)
        self.upload_ev = t.cuda.Event()
        self.upload_ev.record()
        return out


_STAGING = _Staging()
_COPY_POOL = None


def _pcopy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[...] = src, split across 4 threads for multi-MB blocks (numpy
    releases the GIL while copying; one core's memcpy is the bottleneck of a
    host-resident tile's staging)."""
    global _COPY_POOL
    if dst.nbytes < (4 << 20) or dst.shape[0] < 8:
        dst[...] = src
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(max_workers=4)
    n = dst.shape[0]
    cuts = [n * i // 4 for i in range(5)]

    def part(i):
        dst[cuts[i]:cuts[i + 1]] = src[cuts[i]:cuts[i + 1]]

    list(_COPY_POOL.map(part, range(4)))


def _pinned(a: np.ndarray) -> bool:
    t = _dev.torch()
    try:
        return bool(t.from_numpy(a).is_pinned())
    except Exception:  # pragma: no cover
        return False


def transform(slide, source: FitParams, target: FitParams, sink, *,
              strip_height: int = DEFAULT_STRIP_HEIGHT, workers: int | None = None,
              code_lam: float = 0.0, stats: RunStats | None = None,
              gauge: BufferGauge | None = None, progress=None,
              precision: str = "exact", _calibrate=None) -> RunStats:
    """src/pipeline.py:275-345 on the device.

    Output is byte-identical for any strip height / worker count (and, with
    precision="exact", to the reference).  Device source + DeviceWriter: one
    launch over the resident slide, stream-ordered on the current stream
    (returns without waiting for it, like a torch op; RunStats.transform_s
    is then the launch time).  Host source: strips stream through
    ``workers`` (default 2) CUDA streams — H2D, recolor, D2H overlap — and
    are committed to the sink in order; pinned host arrays are copied
    directly without a staging copy.
    """
    t = _dev.torch()
    stats = stats if stats is not None else RunStats()
    gauge = gauge if gauge is not None else BufferGauge()
    factors = scale_factors(source.stats, target.stats)
    if np.any(factors <= 0):
        raise DegenerateStainError("degenerate stain density: target p99 is zero for a stain")
    device_only = isinstance(slide, DeviceSource) and isinstance(sink, DeviceWriter) and \
        progress is None
    if device_only:                      # one launch: only the first strip's height is needed
        if strip_height < 1 or slide.height < 1:
            plan_strips(slide.height, strip_height)      # raises the reference's ValueError
        strips = [(0, min(strip_height, slide.height))]
    else:
        strips = plan_strips(slide.height, strip_height)
    width = slide.width
    plan = XformPlan(source.i0, source.basis, code_lam, factors, target.basis, target.i0,
                     precision=precision)
    t0 = time.perf_counter()
    one_launch = isinstance(slide, DeviceSource)
    if _calibrate is not None and one_launch:
        _calibrate(plan, width * slide.height)      # collective (distributed.RowBandGroup)
    else:
        plan.maybe_calibrate(width * slide.height, inline=one_launch)

    if isinstance(slide, DeviceSource):
        src = slide.tensor
        if isinstance(sink, DeviceWriter):
            with _dev.nvtx("spcn.transform"):
                plan.run(src, sink.pixels, width * slide.height)
            if progress is None:            # one launch wrote every strip in place
                gauge.add(strips[0][1] * width)
                sink.mark_written(0, slide.height)
                gauge.release(strips[0][1] * width)
            else:
                for y, h in strips:
                    gauge.add(h * width)
                    sink.mark_written(y, h)
                    gauge.release(h * width)
                    progress(y + h, slide.height)
            # device in, device out: stream-ordered like any torch op (no host
            # wait; the next call's host work overlaps this launch)
        else:
            out = t.empty_like(src)
            plan.run(src, out, width * slide.height)
            host = out.cpu().numpy()
            for y, h in strips:
                gauge.add(h * width)
                sink.write_strip(PixelBlock(0, y, host[y:y + h]))
                gauge.release(h * width)
                if progress is not None:
                    progress(y + h, slide.height)
    else:
        _transform_streamed(slide, sink, plan, strips, width, workers or 2, gauge, progress)

    stats.transform_s += time.perf_counter() - t0
    stats.transformed_pixels = slide.width * slide.height
    stats.peak_strip_pixels = max(stats.peak_strip_pixels, gauge.peak)
    stats.total_s = stats.sampling_s + stats.basis_fit_s + stats.transform_s
    return stats


def _transform_streamed(slide, sink, plan, strips, width, nslots, gauge, progress):
    """Host-resident slide: bounded in-flight window of strips, in-order commit
    (src/pipeline.py:298-339), each slot its own stream + device/pinned buffers."""
    t = _dev.torch()
    max_h = max(h for _, h in strips)
    nslots = max(1, min(nslots, len(strips)))
    src_arr = slide.array if isinstance(slide, ArraySource) else None
    direct_in = src_arr is not None and _pinned(src_arr)
    direct_out = isinstance(sink, ArrayWriter) and _pinned(sink.pixels)
    slots = []
    nbytes = max_h * width * 3
    for k in range(nslots):
        st = _STAGING.slot(k, nbytes, not direct_in, not direct_out)
        view = lambda b: None if b is None else b[:nbytes].view(max_h, width, 3)  # noqa: E731
        slots.append(dict(stream=st["stream"], dsrc=view(st["dsrc"]), ddst=view(st["ddst"]),
                          hin=None if direct_in else view(st["hin"]),
                          hout=None if direct_out else view(st["hout"]), ev=None, job=None))
    pending = deque()

    def commit():
        slot = pending.popleft()
        y, h = slot["job"]
        slot["ev"].synchronize()
        if direct_out:
            sink.mark_written(y, h)
        else:
            if isinstance(sink, ArrayWriter):
                _pcopy(sink.rows(y, h), slot["hout"][:h].numpy())
                sink.mark_written(y, h)
            else:
                sink.write_strip(PixelBlock(0, y, slot["hout"][:h].numpy()))
        gauge.release(h * width)
        if progress is not None:
            progress(y + h, slide.height)

    for i, (y, h) in enumerate(strips):
        slot = slots[i % nslots]
        while len(pending) >= nslots:
            commit()
        gauge.add(h * width)
        s = slot["stream"]
        with t.cuda.stream(s):
            if direct_in:
                hsrc = t.from_numpy(src_arr[y:y + h])
            else:
                block = src_arr[y:y + h] if src_arr is not None else \
                    slide.read_region(0, y, width, h).pixels
                _pcopy(slot["hin"][:h].numpy(), block)
                hsrc = slot["hin"][:h]
            slot["dsrc"][:h].copy_(hsrc, non_blocking=True)
            plan.run(slot["dsrc"], slot["ddst"], h * width, stream=s)
            if direct_out:
                t.from_numpy(sink.pixels[y:y + h]).copy_(slot["ddst"][:h], non_blocking=True)
            else:
                slot["hout"][:h].copy_(slot["ddst"][:h], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(s)
        slot["ev"] = ev
        slot["job"] = (y, h)
        pending.append(slot)
    while pending:
        commit()


def _fused_ok(src: DeviceSource, tp: FitParams, out, precision: str, p99_mode: str,
              per_patch_stats: bool) -> bool:
    """Whether normalize() may run fit -> transform as one stream-ordered
    sequence with the recolouring built on the device (fit_transform_resident)."""
    if os.environ.get("SPCN_FUSED", "1") == "0":
        return False
    if tp is not None:          # (None: a target fitted on the device, checked there)
        tgt_p99 = np.asarray(tp.stats.p99, dtype=np.float64)
        if not (np.all(tgt_p99 > 0) and np.all(np.isfinite(tgt_p99))):
            return False
    return (precision == "exact" and p99_mode == "sample" and not per_patch_stats
            and (src.tensor.data_ptr() - out.data_ptr()) % 16 == 0)


def fit_transform_resident(src: DeviceSource, target: FitParams, out, *,
                           plan: SamplePlan = SamplePlan(), cfg: SnmfConfig = SnmfConfig(),
                           code_lam: float = 0.0, stats: RunStats | None = None,
                           source_label: str = "") -> FitParams:
    """fit(src) then transform(src, fit, target) into the CUDA tensor `out`
    (src/cli.py:220-244 for a resident slide, pooled p99, EXACT) with one host
    round trip after sampling and one after the parameter build: the SNMF,
    p99, the recolouring's parameters (spcn_xform_rgb8_fitted builds them on
    the device from the fit), the calibration and the recolour run back to
    back on the stream, and the call returns while the recolour is still
    running (stream-ordered, like transform() of a resident slide).  Same bytes, warnings and errors as fit + transform: the
    fit's are raised from its read-back before anything else, and a
    recolouring the device path declines (degenerate p99, ill-conditioned
    basis) is redone by transform() with host parameters, which raises the
    reference's error or takes the strict path.  Returns the source fit."""
    from . import fitcore

    stats = stats if stats is not None else RunStats()
    t0 = time.perf_counter()
    fb = fitcore.buffers(src.tensor.device, plan.target_pixels, cfg.max_outer_iters)
    L = _lib.lib()
    npix = src.width * src.height
    # everything that does not depend on the sample, before the sampling wait
    p = _fitted_params(target, float(code_lam), npix)
    p.src_od_table = fb.lut_ptr
    p.src_fit = fb.arena_b_ptr
    ws_bytes = int(L.spcn_xform_workspace_bytes(npix))
    st = _lib.stream_handle()
    ws = _dev.workspace(ws_bytes, stream=st)
    m, i0, meta = _fit_sample_checked(fb, src, plan, False)
    stats.sampled_pixels = m
    stats.patches = meta.patches_used
    t1 = time.perf_counter()
    stats.sampling_s += t1 - t0
    with _dev.nvtx("spcn.fit_transform"):
        fitcore.basis_enqueue(fb, fb.sample_ptr, m, i0, cfg, code_lam=code_lam, pooled=True)
        fb.pin_status_np[0] = -1
        # returns once the build status (and the fit's read-back before it)
        # is in host memory; the recolour is still running, stream-ordered
        _lib.check(L.spcn_xform_rgb8_fitted(src.tensor.data_ptr(), out.data_ptr(), npix,
                                            ctypes.byref(p), _lib.ptr(ws), ws_bytes,
                                            fb.pin_status_ptr, st), "xform_rgb8_fitted")
    prov = fitcore.provenance(plan, cfg, code_lam, False, "sample", source_label)
    sp = fitcore.parse_pooled(fb, m, i0, cfg, prov, stacklevel=3)
    t2 = time.perf_counter()
    stats.basis_fit_s += t2 - t1
    if int(fb.pin_status_np[0]) != 0:
        transform(src, sp, target, DeviceWriter(src.width, src.height, out=out),
                  code_lam=code_lam, stats=stats, precision="exact")
    else:
        stats.transform_s += time.perf_counter() - t2
        stats.transformed_pixels = npix
        stats.total_s = stats.sampling_s + stats.basis_fit_s + stats.transform_s
    return sp


def fit_pair_transform_resident(src: DeviceSource, tgt: DeviceSource, out, *,
                                plan: SamplePlan = SamplePlan(),
                                cfg: SnmfConfig = SnmfConfig(), code_lam: float = 0.0,
                                stats: RunStats | None = None):
    """normalize(source, target) for two resident images (src/cli.py:220-244:
    fit(target), fit(source), transform): the two fits run in lockstep — both
    samplings, one wait, both SNMF/p99 tails — and the recolouring is built
    on the device from both fits (spcn_xform_rgb8_fitted with tgt_fit), so a
    call has two host waits instead of four.  The target's errors and
    warnings come first, as in the reference; a recolouring the device
    declines is redone by transform() with host parameters.  Returns
    (source fit, target fit)."""
    from . import fitcore

    stats = stats if stats is not None else RunStats()
    t0 = time.perf_counter()
    fb_s = fitcore.buffers(src.tensor.device, plan.target_pixels, cfg.max_outer_iters, slot=0)
    fb_t = fitcore.buffers(tgt.tensor.device, plan.target_pixels, cfg.max_outer_iters, slot=1)
    L = _lib.lib()
    npix = src.width * src.height
    p = _lib.XformFitted()
    p.code_lam = float(code_lam)
    p.max_sweeps = 2000
    p.flags = FITTED_ANALYTIC if npix < XformPlan.CALIBRATE_MIN_PIXELS else 0
    p.src_od_table, p.src_fit = fb_s.lut_ptr, fb_s.arena_b_ptr
    p.tgt_fit, p.tgt_i0_dev = fb_t.arena_b_ptr, fb_t.arena_a_ptr + fitcore.A_I0
    ws_bytes = int(L.spcn_xform_workspace_bytes(npix))
    st = _lib.stream_handle()
    ws = _dev.workspace(ws_bytes, stream=st)
    # the target's fit on a side stream beside the source's (each fit's
    # kernels fill only a few SMs: its SNMF is one 16-CTA cluster)
    t = _dev.torch()
    main = t.cuda.current_stream()
    if os.environ.get("SPCN_PAIR_SIDE", "1") == "0":       # (A/B: one stream)
        side, fork, join = main, t.cuda.Event(), t.cuda.Event()
    else:
        side, fork, join = _side_stream(src.tensor.device)
    fork.record(main)
    side.wait_event(fork)
    with _dev.fast_stream(side):
        started_t = _sample_start(fb_t, tgt, plan)
    started_s = _sample_start(fb_s, src, plan)
    with _dev.fast_stream(side):
        m_t, i0_t, _ = _fit_sample_checked(fb_t, tgt, plan, False, started=started_t)
    m_s, i0_s, meta = _fit_sample_checked(fb_s, src, plan, False, started=started_s)
    stats.sampled_pixels = m_s
    stats.patches = meta.patches_used
    t1 = time.perf_counter()
    stats.sampling_s += t1 - t0
    with _dev.nvtx("spcn.fit_pair_transform"):
        with _dev.fast_stream(side):
            fitcore.basis_enqueue(fb_t, fb_t.sample_ptr, m_t, i0_t, cfg, code_lam=code_lam,
                                  pooled=True)
            join.record(side)
        fitcore.basis_enqueue(fb_s, fb_s.sample_ptr, m_s, i0_s, cfg, code_lam=code_lam,
                              pooled=True)
        main.wait_event(join)      # the build reads the target's arena
        fb_s.pin_status_np[0] = -1
        # returns once the build status (and both fits' read-backs before it)
        # is in host memory; the recolour is still running, stream-ordered
        _lib.check(L.spcn_xform_rgb8_fitted(src.tensor.data_ptr(), out.data_ptr(), npix,
                                            ctypes.byref(p), _lib.ptr(ws), ws_bytes,
                                            fb_s.pin_status_ptr, st), "xform_rgb8_fitted")
    from . import fitcore as fc

    prov = fc.provenance(plan, cfg, code_lam, False, "sample", "")
    tp = fc.parse_pooled(fb_t, m_t, i0_t, cfg, prov, stacklevel=3)
    sp = fc.parse_pooled(fb_s, m_s, i0_s, cfg, prov, stacklevel=3)
    t2 = time.perf_counter()
    stats.basis_fit_s += t2 - t1
    if int(fb_s.pin_status_np[0]) != 0:
        transform(src, sp, tp, DeviceWriter(src.width, src.height, out=out),
                  code_lam=code_lam, stats=stats, precision="exact")
    else:
        stats.transform_s += time.perf_counter() - t2
        stats.transformed_pixels = npix
        stats.total_s = stats.sampling_s + stats.basis_fit_s + stats.transform_s
    return sp, tp


_SIDE = threading.local()


def _side_stream(device):
    """Per-thread side stream + fork/join events of a device (reused: fresh
    streams per call would defeat the caching allocator's per-stream pools)."""
    t = _dev.torch()
    key = t.device(device).index
    cache = _SIDE.__dict__.setdefault("by_dev", {})
    hit = cache.get(key)
    if hit is None:
        with t.cuda.device(key):
            hit = cache[key] = (t.cuda.Stream(), t.cuda.Event(), t.cuda.Event())
    return hit


FITTED_ANALYTIC = 1   # include/spcn.h SPCN_FITTED_ANALYTIC


def _fitted_params(target: FitParams, code_lam: float, total_pixels: int):
    """spcn_xform_fitted's host half (target profile + options).  Images
    below XformPlan.CALIBRATE_MIN_PIXELS use the analytic bound, as
    XformPlan.maybe_calibrate decides for the host-built path."""
    p = _lib.XformFitted()
    np.frombuffer(p, dtype=np.float64, count=12, offset=16)[:] = np.concatenate([
        _dev.f64_array(target.basis, 6, "tgt_basis"),
        np.asarray(target.stats.p99, dtype=np.float64).reshape(2),
        _dev.f64_array(target.i0, 3, "tgt_i0"), [code_lam]])
    p.max_sweeps = 2000
    p.flags = FITTED_ANALYTIC if total_pixels < XformPlan.CALIBRATE_MIN_PIXELS else 0
    return p


WHOLE_UPLOAD_PIXELS = 1 << 26     # 64 Mpx (192 MB): host images up to this go up whole


def _whole_upload_ok(source, target) -> bool:
    """A host (numpy, uint8 (h, w, 3)) source — and a numpy target image, if
    one — small enough to go to the GPU whole."""
    if os.environ.get("SPCN_WHOLE_UPLOAD", "1") == "0":
        return False
    if not (isinstance(source, np.ndarray) and source.dtype == np.uint8 and
            source.ndim == 3 and source.shape[2] == 3 and 0 < source.size // 3 <= WHOLE_UPLOAD_PIXELS):
        return False
    if isinstance(target, np.ndarray):
        return (target.dtype == np.uint8 and target.ndim == 3 and target.shape[2] == 3
                and 0 < target.size // 3 <= WHOLE_UPLOAD_PIXELS)
    return isinstance(target, (FitParams, str, os.PathLike))


def normalize(source, target, *, plan: SamplePlan = SamplePlan(),
              cfg: SnmfConfig = SnmfConfig(), code_lam: float = 0.0,
              per_patch_stats: bool = False, strip_height: int = DEFAULT_STRIP_HEIGHT,
              precision: str = "exact", stats: RunStats | None = None,
              p99_mode: str = "sample", out=None):
    """The drop-in entry: fit(source), fit(target) (or use a FitParams / profile
    for the target), then transform — exactly the reference's _normalize_one
    (src/cli.py:220-244).  numpy in → numpy out; CUDA tensor in → CUDA tensor
    out (written into ``out`` when given, of the matching kind).  A resident slide with a pooled
    p99 and EXACT precision runs as fit_transform_resident (no host round
    trip between the fit and the recolour; same bytes).  A host image small
    enough (≤ WHOLE_UPLOAD_PIXELS) is uploaded whole and takes the device
    path (a tile's fits then need no per-patch uploads and run in lockstep
    with the target's); larger ones stream strips through the GPU."""
    from .normalize import load_profile

    t = _dev.torch()
    stats = stats if stats is not None else RunStats()
    host = not _dev.is_tensor(source)
    if host and out is not None:          # host image, caller's host buffer
        res = normalize(source, target, plan=plan, cfg=cfg, code_lam=code_lam,
                        per_patch_stats=per_patch_stats, strip_height=strip_height,
                        precision=precision, stats=stats, p99_mode=p99_mode)
        if tuple(np.shape(out)) != tuple(res.shape):
            raise ValueError("out must have the source's shape")
        np.copyto(out, res)
        return out
    if host and _whole_upload_ok(source, target):
        dev_t = target
        if isinstance(target, np.ndarray):
            dev_t = t.from_numpy(np.ascontiguousarray(target)).cuda()
        res = normalize(t.from_numpy(np.ascontiguousarray(source)).cuda(), dev_t, plan=plan,
                        cfg=cfg, code_lam=code_lam, per_patch_stats=per_patch_stats,
                        strip_height=strip_height, precision=precision, stats=stats,
                        p99_mode=p99_mode)
        return res.cpu().numpy()
    src = ArraySource(source) if host else DeviceSource(source)
    dst = None
    if not host:
        dst = out if out is not None else t.empty((src.height, src.width, 3), dtype=t.uint8,
                                                  device=src.tensor.device)
        if tuple(dst.shape) != (src.height, src.width, 3) or dst.dtype != t.uint8 or \
                dst.device != src.tensor.device or not dst.is_contiguous():
            raise ValueError("out must be a contiguous uint8 CUDA tensor shaped like the source")
    if isinstance(target, FitParams):
        tp = target
    elif isinstance(target, (str, os.PathLike)):
        tp = load_profile(target)
    else:
        tsrc = ArraySource(target) if not _dev.is_tensor(target) else DeviceSource(target)
        if dst is not None and isinstance(tsrc, DeviceSource) and \
                tsrc.tensor.device == src.tensor.device and \
                _fused_ok(src, None, dst, precision, p99_mode, per_patch_stats):
            # both resident: the two fits in lockstep, the recolouring built
            # from both on the device (fit_pair_transform_resident)
            fit_pair_transform_resident(src, tsrc, dst, plan=plan, cfg=cfg, code_lam=code_lam,
                                        stats=stats)
            return dst
        tp = fit(tsrc, plan, cfg, code_lam=code_lam, per_patch_stats=per_patch_stats,
                 p99_mode=p99_mode)
    if not host:
        if _fused_ok(src, tp, dst, precision, p99_mode, per_patch_stats):
            fit_transform_resident(src, tp, dst, plan=plan, cfg=cfg, code_lam=code_lam,
                                   stats=stats)
            return dst
    sp = fit(src, plan, cfg, code_lam=code_lam, per_patch_stats=per_patch_stats, stats=stats,
             p99_mode=p99_mode)
    if host:
        sink = ArrayWriter(src.width, src.height)
        transform(src, sp, tp, sink, strip_height=strip_height, code_lam=code_lam, stats=stats,
                  precision=precision)
        return sink.pixels
    sink = DeviceWriter(src.width, src.height, out=dst)
    transform(src, sp, tp, sink, strip_height=strip_height, code_lam=code_lam, stats=stats,
              precision=precision)
    return sink.pixels
