"""Whole-slide ("global") per-stain 99th percentile — ``p99_mode="global"``.

The reference's stain_stats (src/normalize.py:58-100) pools the densities of
the <= 100 k *sampled* non-white pixels (src/pipeline.py:226,238); that stays
the default (``p99_mode="sample"``).  Global mode (SURVEY.md §8(0).3, §8(a)
a7) pools the densities of every non-white pixel of the slide (non-white = not
all channels > white threshold, src/pipeline.py:176), coded with the fitted
basis exactly as code_densities (src/stain_sep.py:168-201) would, and returns
exactly ``percentile(those densities, 99)`` (src/order_stats.py:11-36).

Passes over the slide (csrc/stats.cu):
  1. histogram of fp32 densities (8192 bins of fp32 keys) over the bracket
     the sampled densities give (``sample_bracket``), else over all keys — K2
  2. (only if the bins are still too wide) a finer histogram around the bins
     holding ranks lo / hi                                          — K2
  3. exact refine: fp64 reference-order densities for the pixels that may
     fall in the final window, exact counts below it, the in-window values
     listed, then an exact select of the two ranks                  — K3
Across GPUs the histograms/counts are summed (``allreduce``, NCCL) and the
candidate lists gathered (``allgather``), SURVEY §8(e).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _dev, _lib
from .errors import StainAbsentError
from .order_stats import interpolate

NBINS = 8192
SHIFT0 = 19              # fp32 key >> 19: 8192 bins over all non-negative floats
CAND_CAP = 1 << 20       # in-window values listed per stain per rank (grown as needed)
REFINE_MAX = 1 << 22     # refine a window once it holds <= this many pixels: its
                         # pixels cost one colour-cache probe each, a zoom level a pass
MIN_SHIFT = 6            # finest bins: 64 fp32 ulps, > 2x the fp32 density error

_U32x2 = ctypes.c_uint32 * 2
_F64x2 = ctypes.c_double * 2


def _sig():
    L = _lib.lib()
    if not getattr(L, "_spcn_gstats_declared", False):
        P, I32, I64 = _lib.P, _lib.I32, _lib.I64
        _lib.declare("spcn_stats_hist", ctypes.c_int,
                     [P, I64, ctypes.POINTER(_lib.XformParams), I32, P, P, I32, P, P, P])
        _lib.declare("spcn_stats_refine", ctypes.c_int,
                     [P, I64, ctypes.POINTER(_lib.XformParams), I32, P, P, P, P, P,
                      ctypes.c_uint64, P])
        L._spcn_gstats_declared = True
    return L


def _key_value(key: int) -> float:
    """fp32 whose bit pattern is `key` (non-negative floats), as a double."""
    if key >= 0x7F800000:
        return math.inf
    return float(np.array([key], dtype=np.uint32).view(np.float32)[0])


def _key_of(x: float) -> int:
    """fp32 bit pattern (as int) of a non-negative value."""
    return int(np.array([x], dtype=np.float32).view(np.uint32)[0])


def _locate(hist: np.ndarray, rank: int):
    """Bin holding `rank` (0-based) of a histogram, or None past the end."""
    c = np.cumsum(hist, dtype=np.int64)
    b = int(np.searchsorted(c, rank, side="right"))
    return b if b < hist.size else None


class _Local:
    """Single-process reductions (identity)."""

    @staticmethod
    def allreduce(t):
        return t

    @staticmethod
    def allgather(t):
        return [t]


class DeviceEngine:
    """The two device passes (csrc/stats.cu) over a rank's part of the slide."""

    def __init__(self, chunks, src_i0, basis, code_lam, white_threshold, max_sweeps=2000):
        from .xform import XformPlan

        self.t = _dev.torch()
        self.L = _sig()
        self.chunks = chunks
        basis = np.asarray(basis, dtype=np.float64)
        self.plan = XformPlan(src_i0, basis, code_lam, [1.0, 1.0], basis, [255.0] * 3,
                              precision="exact", max_sweeps=max_sweeps)
        self.thr = int(white_threshold)

    def hist(self, base, shift):
        t, L = self.t, self.L
        hist = t.zeros((2, NBINS), dtype=t.int64, device="cuda")
        counts = t.zeros(3, dtype=t.int64, device="cuda")
        b, s = _U32x2(*base), _U32x2(*shift)
        for x in self.chunks():
            _lib.check(L.spcn_stats_hist(_lib.ptr(x), x.numel() // 3, ctypes.byref(self.plan.params),
                                         self.thr, ctypes.byref(b), ctypes.byref(s), NBINS,
                                         _lib.ptr(hist), _lib.ptr(counts), _lib.stream_handle()),
                       "stats_hist")
        return hist, counts

    def refine(self, lo, hi, cap):
        """-> counts (7: below[2], in-window pixels[2], fp64 evals, list sizes[2]),
        values (2, cap), pixel counts (2, cap)."""
        t, L = self.t, self.L
        counts = t.zeros(7, dtype=t.int64, device="cuda")
        cand = t.empty((2, max(cap, 1)), dtype=t.float64, device="cuda")
        wcnt = t.empty((2, max(cap, 1)), dtype=t.int64, device="cuda")
        a, b = _F64x2(*lo), _F64x2(*hi)
        for x in self.chunks():
            _lib.check(L.spcn_stats_refine(_lib.ptr(x), x.numel() // 3,
                                           ctypes.byref(self.plan.params), self.thr,
                                           ctypes.byref(a), ctypes.byref(b), _lib.ptr(counts),
                                           _lib.ptr(cand), _lib.ptr(wcnt), cap,
                                           _lib.stream_handle()), "stats_refine")
        return counts, cand, wcnt


def _table_sig():
    L = _sig()
    if not getattr(L, "_spcn_table_declared", False):
        P, I32, I64, U64 = _lib.P, _lib.I32, _lib.I64, ctypes.c_uint64
        XP = ctypes.POINTER(_lib.XformParams)
        _lib.declare("spcn_stats_table", ctypes.c_int, [P, I64, XP, I32, P, P, P, P])
        _lib.declare("spcn_stats_table_scan", ctypes.c_int, [XP, P, P, P, U64, P, P])
        _lib.declare("spcn_stats_cube_classes", ctypes.c_int, [XP, I32, P, P, P])
        _lib.declare("spcn_stats_table_cube", ctypes.c_int, [P, I64, XP, I32, P, P, P, P, P])
        _lib.declare("spcn_table_entries_hist", ctypes.c_int, [P, P, I64, P, P, I32, P, P])
        _lib.declare("spcn_table_entries_collect", ctypes.c_int,
                     [P, P, I64, P, P, I32, P, P, P, U64, P, P])
        L._spcn_table_declared = True
    return L


TABLE_CAP = 1 << 22      # present colours handled by the one-pass mode (else: histogram path)
SEL_BINS = 4096          # bins of the entry histogram (exact selection without a sort)


def _device_table(self, lo):
    """One pass: colour counts (2^24, int64 view of u64) of the pixels not
    surely below lo, and the non-white count.  The 8x8x8 colour-cell classes
    (32 KiB) are built once per call from the same parameters."""
    t, L = self.t, _table_sig()
    table = t.zeros(1 << 24, dtype=t.int64, device="cuda")
    counts = t.zeros(1, dtype=t.int64, device="cuda")
    cls = t.empty((32 << 10) + (2 << 20), dtype=t.uint8, device="cuda")   # SPCN_CUBE_CLASS_BYTES
    a = _F64x2(*lo)
    _lib.check(L.spcn_stats_cube_classes(ctypes.byref(self.plan.params), self.thr, ctypes.byref(a),
                                         _lib.ptr(cls), _lib.stream_handle()), "stats_cube_classes")
    for x in self.chunks():
        _lib.check(L.spcn_stats_table_cube(_lib.ptr(x), x.numel() // 3,
                                           ctypes.byref(self.plan.params), self.thr,
                                           ctypes.byref(a), _lib.ptr(cls), _lib.ptr(table),
                                           _lib.ptr(counts), _lib.stream_handle()),
                   "stats_table_cube")
    return table, counts


def _device_scan(self, table, cap=TABLE_CAP):
    """Present colours of this rank's table: exact densities (m, 2), pixel
    counts (m,), the per-stain maxima (2,) and whether more than `cap`
    colours were present (then the entries are incomplete)."""
    t, L = self.t, _table_sig()
    x = t.empty((cap, 2), dtype=t.float64, device="cuda")
    w = t.empty(cap, dtype=t.int64, device="cuda")
    n_out = t.zeros(4, dtype=t.int64, device="cuda")
    _lib.check(L.spcn_stats_table_scan(ctypes.byref(self.plan.params), _lib.ptr(table),
                                       _lib.ptr(x), _lib.ptr(w), cap, _lib.ptr(n_out),
                                       _lib.stream_handle()), "stats_table_scan")
    info = _dev.readback(n_out)
    m = int(info[0])
    xmax = info[2:4].view(np.float64).copy()
    return x[:min(m, cap)], w[:min(m, cap)], xmax, m > cap


def _device_entries_hist(self, x, w, lo, scale, nbins):
    t, L = self.t, _table_sig()
    hist = t.zeros((2, nbins), dtype=t.int64, device="cuda")
    _lib.check(L.spcn_table_entries_hist(_lib.ptr(x), _lib.ptr(w), int(w.numel()),
                                         ctypes.byref(_F64x2(*lo)), ctypes.byref(_F64x2(*scale)),
                                         nbins, _lib.ptr(hist), _lib.stream_handle()),
               "table_entries_hist")
    return hist


def _device_entries_collect(self, x, w, lo, scale, nbins, bins):
    """(values, weights) of stain j's entries in bins [bins[2j], bins[2j+1]]."""
    t, L = self.t, _table_sig()
    b = (ctypes.c_int32 * 4)(*[int(v) for v in bins])
    cap = 1 << 16
    while True:
        vals = t.empty((2, cap), dtype=t.float64, device="cuda")
        wts = t.empty((2, cap), dtype=t.int64, device="cuda")
        nsel = t.zeros(2, dtype=t.int64, device="cuda")
        _lib.check(L.spcn_table_entries_collect(_lib.ptr(x), _lib.ptr(w), int(w.numel()),
                                                ctypes.byref(_F64x2(*lo)),
                                                ctypes.byref(_F64x2(*scale)), nbins, b,
                                                _lib.ptr(vals), _lib.ptr(wts), cap, _lib.ptr(nsel),
                                                _lib.stream_handle()), "table_entries_collect")
        k = _dev.readback(nsel)
        if max(k) <= cap:
            return [(vals[j, :int(k[j])], wts[j, :int(k[j])]) for j in range(2)]
        cap = int(max(k))


DeviceEngine.table = _device_table
DeviceEngine.scan = _device_scan
DeviceEngine.entries_hist = _device_entries_hist
DeviceEngine.entries_collect = _device_entries_collect


def _table_select(eng, x, w, xmax, n: int, lo, ks, comm):
    """Order statistics `ks` (0-based ranks among the n non-white pixels of all
    ranks) of both stains from the per-rank colour-table entries, exactly and
    without sorting them: pixels off the tables are < lo[j], so rank k is the
    (k - below_j)-th smallest of the entries with x_j >= lo[j] (below_j = n -
    their weight).  A weighted histogram of those entries over SEL_BINS equal
    bins of [lo_j, max_j] (summed across ranks: 64 KiB) gives the bins that
    hold the ranks; only their entries are gathered and selected exactly.
    Returns (values (2, len(ks)), below) or None when a rank falls below lo."""
    local = isinstance(comm, _Local)
    if local:                      # one process: no device round trip for the maxima
        xm = np.asarray(xmax, dtype=np.float64)
    else:
        xm = np.max(np.stack([np.asarray(v.cpu() if hasattr(v, "cpu") else v, dtype=np.float64)
                              for v in comm.allgather(_as_tensor(xmax, x))]), axis=0)
    scale = [SEL_BINS / (xm[j] - lo[j]) if xm[j] > lo[j] else 0.0 for j in range(2)]
    hist = comm.allreduce(eng.entries_hist(x, w, lo, scale, SEL_BINS))
    hist = hist.cpu().numpy() if hasattr(hist, "cpu") else np.asarray(hist)
    kept = hist.sum(axis=1)
    below = [int(n - kept[j]) for j in range(2)]
    if int(kept.min()) == 0 or any(min(ks) < b for b in below):
        return None
    bins, before = [], []
    for j in range(2):
        c = np.cumsum(hist[j])
        r = [k - below[j] for k in ks]
        b0 = int(np.searchsorted(c, min(r), side="right"))
        b1 = int(np.searchsorted(c, max(r), side="right"))
        if b1 >= SEL_BINS:
            return None
        bins += [b0, b1]
        before.append(int(c[b0 - 1]) if b0 else 0)
    lists = eng.entries_collect(x, w, lo, scale, SEL_BINS, bins)
    vals = np.empty((2, len(ks)))
    if local and getattr(lists[0][0], "is_cuda", False):
        # one read of both stains' (value, weight) lists (weights as f64 bits)
        t = _dev.torch()
        parts = [lists[0][0], lists[1][0], lists[0][1].view(t.float64),
                 lists[1][1].view(t.float64)]
        flat = _dev.readback(t.cat(parts))
        n0, n1 = int(lists[0][0].numel()), int(lists[1][0].numel())
        got = [(flat[:n0], flat[n0 + n1:2 * n0 + n1].view(np.int64)),
               (flat[n0:n0 + n1], flat[2 * n0 + n1:].view(np.int64))]
        for j in range(2):
            vals[j] = weighted_select(got[j][0], got[j][1], [k - below[j] - before[j] for k in ks])
        return vals, below
    for j in range(2):
        v = np.concatenate([np.asarray(a.cpu() if hasattr(a, "cpu") else a, dtype=np.float64)
                            for a in comm.allgather(lists[j][0])])
        c = np.concatenate([np.asarray(a.cpu() if hasattr(a, "cpu") else a, dtype=np.int64)
                            for a in comm.allgather(lists[j][1])])
        vals[j] = weighted_select(v, c, [k - below[j] - before[j] for k in ks])
    return vals, below


def _as_tensor(v, like):
    import torch

    return torch.as_tensor(np.asarray(v, dtype=np.float64), device=like.device)


def bracket_ranks(m: int, p: float = 99.0):
    """0-based ranks of the sample quantiles p -+ d of an m-sample (see
    sample_bracket)."""
    q = p / 100.0
    d = max(0.005, 6.0 * math.sqrt(q * (1.0 - q) / m) * 10.0)
    return [int(math.floor(max(0.0, q - d) * (m - 1))), int(math.ceil(min(1.0, q + d) * (m - 1)))]


def sample_bracket(h, p: float = 99.0):
    """[lo, hi] per stain around the p-th percentile of the sampled densities
    `h` ((2, m) device tensor, one row per stain): the sample quantiles
    p -+ d, d = max(0.5, 600 * sqrt(p (1 - p) / m)) percent (6 standard errors
    of the quantile at a 100x smaller effective sample).  Exact k-th
    selections on the device (libspcn), one host read; None when the sample
    is empty."""
    m = int(h.shape[1])
    if m == 0:
        return None
    idx = bracket_ranks(m, p)
    import torch as t   # tensor plumbing on h's device
    from . import stats as dstats

    L = dstats._sig()
    v = h.contiguous()
    # four exact selections (2 stains x 2 ranks) in one libspcn call, no sort
    begin = t.tensor([0, 0, m, m], dtype=t.int64, device=h.device)
    end = t.tensor([m, m, 2 * m, 2 * m], dtype=t.int64, device=h.device)
    ks = t.tensor([idx[0], idx[1], idx[0], idx[1]], dtype=t.int64, device=h.device)
    q = t.empty(4 * dstats._QBYTES, dtype=t.uint8, device=h.device)
    out = t.empty(4, dtype=t.float64, device=h.device)
    _lib.check(L.spcn_select_kth(_lib.ptr(v), _lib.ptr(begin), _lib.ptr(end), _lib.ptr(ks), 4,
                                 _lib.ptr(q), _lib.ptr(out), _lib.stream_handle()), "select_kth")
    return _dev.readback(out).reshape(2, 2)


def weighted_select(values: np.ndarray, weights: np.ndarray, ks):
    """Order statistics of the multiset {values[i] repeated weights[i] times}
    (exact: a stable sort of the distinct values and integer cumulative
    counts)."""
    order = np.argsort(values, kind="stable")
    v, c = values[order], np.cumsum(weights[order].astype(np.int64))
    return [float(v[int(np.searchsorted(c, k, side="right"))]) for k in ks]


def global_p99(chunks, src_i0, basis, code_lam: float = 0.0, white_threshold: int = 220,
               p: float = 99.0, *, comm=None, max_sweeps: int = 2000, engine=None, guess=None):
    """Exact whole-slide percentile of both stains.

    chunks   : callable returning an iterable of flat CUDA uint8 tensors (RGB8
               pixel runs, 16-byte aligned) that together cover this rank's
               part of the slide; called once per pass.
    comm     : object with ``allreduce(tensor) -> tensor`` (sum) and
               ``allgather(tensor) -> list`` for multi-GPU; None = one process.
    engine   : the pass implementation (default: the CUDA kernels; the CPU
               tests substitute an emulation of their contracts).
    guess    : optional estimate of the two percentiles: a point (2,) (the
               first histogram level then spans +-2 octaves around it) or a
               bracket (2, 2) of [lo, hi] per stain (``sample_bracket``: the
               first level spans the bracket, usually fine enough to refine
               directly — two passes in all).  A miss costs one full-range
               level.
    Returns (p99 ndarray(2), non-white pixel count, info dict).
    """
    comm = comm or _Local()
    eng = engine or DeviceEngine(chunks, src_i0, basis, code_lam, white_threshold, max_sweeps)
    info = {"passes": 0}
    import torch as t   # tensor plumbing only (the engine does the compute)

    def hist_pass(base, shift):
        hist, counts = eng.hist(base, shift)
        info["passes"] += 1
        hist, counts = comm.allreduce(hist), comm.allreduce(counts)
        return hist.cpu().numpy(), counts.cpu().numpy()

    def refine_pass(lo, hi, cap):
        counts, cand, wcnt = eng.refine(lo, hi, cap)
        info["passes"] += 1
        local = counts.cpu().numpy()
        lists = []
        for j in range(2):
            m = int(min(local[5 + j], cap))
            vals = comm.allgather(cand[j, :m].contiguous())
            cnts = comm.allgather(wcnt[j, :m].contiguous())
            lists.append((t.cat(vals).cpu().numpy(), t.cat(cnts).cpu().numpy()))
        total = comm.allreduce(counts).cpu().numpy()
        overflow = bool(local[5] > cap or local[6] > cap)
        return total, lists, overflow

    # one-pass mode: colour table of the pixels not surely below the
    # bracket's lower ends (needs positive lower ends and a table engine)
    g = None if guess is None else np.asarray(guess, dtype=np.float64)
    if g is not None and g.shape == (2, 2) and np.isfinite(g).all() and (g[:, 0] > 0).all() \
            and hasattr(eng, "table"):
        lo_t = [float(g[0, 0]), float(g[1, 0])]
        with _dev.nvtx("spcn.global.table_pass"):
            tab, cnt = eng.table(lo_t)      # this rank's table: never exchanged
        info["passes"] += 1
        n = int(comm.allreduce(cnt).reshape(-1)[0].item())
        if n == 0:
            raise StainAbsentError("stain absent: no non-white pixels in the slide")
        rank = (p / 100.0) * (n - 1)
        klo, khi = int(math.floor(rank)), int(math.ceil(rank))
        with _dev.nvtx("spcn.global.scan"):
            x, w, xmax, over = eng.scan(tab)
        del tab
        if not isinstance(comm, _Local):   # any rank's table overflowing sends all to the fallback
            over = int(comm.allreduce(_as_tensor([1.0 if over else 0.0], x)).cpu().numpy()[0])
        with _dev.nvtx("spcn.global.select"):
            res = None if over else _table_select(eng, x, w, xmax, n, lo_t, [klo, khi], comm)
        if res is not None:
            vals, below = res
            p99 = np.array([interpolate(vals[j][0], vals[j][1], rank) for j in range(2)])
            info.update(mode="table", nonwhite=n, colours=int(w.numel()), below=below,
                        fp64_evaluations=int(w.numel()), levels=0)
            return p99, n, info
        info["table_miss"] = True

    # histogram levels: start over all fp32 keys, then zoom into the bins
    # holding ranks lo..hi (one bin of margin each side) until the window is
    # small enough to list, or its bins reach the fp32 error scale
    base, shift = [0, 0], [SHIFT0, SHIFT0]
    if g is not None and g.shape == (2,) and all(x > 0 and math.isfinite(x) for x in g):
        g = np.stack([g / 4.0, g * 4.0], axis=1)       # +-2 octaves around a point
    if g is not None and g.shape == (2, 2) and np.isfinite(g).all() and (g >= 0).all() \
            and (g[:, 1] >= g[:, 0]).all():
        # start from the estimated bracket; a miss falls back to the
        # full-range level below
        for j in range(2):
            k0, k1 = _key_of(g[j, 0]), _key_of(g[j, 1]) + 1
            base[j], shift[j] = k0, max(MIN_SHIFT, ((k1 - k0 - 1) // NBINS).bit_length())
    h, c = hist_pass(base, shift)
    n = int(c[0])
    if n == 0:
        raise StainAbsentError("stain absent: no non-white pixels in the slide")
    rank = (p / 100.0) * (n - 1)
    klo, khi = int(math.floor(rank)), int(math.ceil(rank))
    if g is not None and shift != [SHIFT0, SHIFT0]:
        inside = all(int(c[1 + j]) <= klo and khi < int(c[1 + j] + h[j].sum()) for j in range(2))
        if not inside:
            base, shift = [0, 0], [SHIFT0, SHIFT0]
            h, c = hist_pass(base, shift)
    windows = []                          # key windows of every level, outermost first
    while True:
        win, est = [], []
        for j in range(2):
            below = int(c[1 + j])
            flo = _locate(h[j], klo - below) if klo >= below else None
            fhi = _locate(h[j], khi - below) if khi >= below else None
            if flo is None or fhi is None:   # lost the ranks: keep the previous window
                win = None
                break
            f0, f1 = max(0, flo - 1), min(NBINS, fhi + 2)
            win.append((base[j] + (f0 << shift[j]), base[j] + (f1 << shift[j])))
            est.append(int(h[j][f0:f1].sum()))
        if win is None:
            break
        windows.append((win, max(est)))
        # refine now if the window is small, or if a zoom (<= 4x finer bins)
        # could not split it much (slides repeat colours: a bin can hold one value)
        if max(est) <= REFINE_MAX or min(shift) < MIN_SHIFT + 1 or \
                (max(shift) < MIN_SHIFT + 3 and max(est) <= 8 * REFINE_MAX):
            break
        for j in range(2):
            width = win[j][1] - win[j][0]
            s_ = 0
            while (width >> s_) > NBINS:
                s_ += 1
            base[j], shift[j] = win[j][0], max(s_, MIN_SHIFT)
        h, c = hist_pass(base, shift)
    info["levels"] = len(windows)

    def keys_to_values(win):
        return ([-math.inf if k[0] == 0 else _key_value(k[0]) for k in win],
                [_key_value(k[1]) for k in win])

    # pass: exact refine of the innermost window (widen outward if it misses)
    for win, est in reversed(windows):
        lo_w, hi_w = keys_to_values(win)
        cap = max(CAND_CAP, 2 * est + 4096)
        total, cands, overflow = refine_pass(lo_w, hi_w, cap)
        info.setdefault("refines", []).append(dict(window=(lo_w, hi_w), below=total[:2].tolist(),
                                                   inwin=total[2:4].tolist(), overflow=overflow))
        ok = not overflow and all(int(total[j]) <= klo and khi < int(total[j] + total[2 + j])
                                  for j in range(2))
        if ok:
            break
    else:
        raise RuntimeError(f"global p99: no refine window contains the ranks ({info})")
    p99 = np.empty(2)
    for j in range(2):
        below = int(total[j])
        vals = weighted_select(cands[j][0], cands[j][1], [klo - below, khi - below])
        p99[j] = interpolate(vals[0], vals[1], rank)
    info.update(nonwhite=n, fp64_evaluations=int(total[4]), window=(lo_w, hi_w),
                candidates=[int(total[2]), int(total[3])])
    # stain absent (src/normalize.py:91-94): max <= 0, i.e. no positive density
    for j in range(2):
        if p99[j] <= 0.0:
            tot, _, _ = refine_pass([5e-324, 5e-324], [math.inf, math.inf], 0)
            if int(tot[2 + j]) == 0:
                names = ("hematoxylin", "eosin")
                raise StainAbsentError(f"stain absent: no {names[j]} density observed")
            break
    return p99, n, info
