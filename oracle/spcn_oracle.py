"""NumPy restatement of the reference SPCN path — TEST INFRASTRUCTURE ONLY.

Every function cites the reference function it restates
(``src/`` = ``/root/reference/pkg/src/slidenorm/``).  Arithmetic is written
in the reference's operation order so that, on the same machine, results
are bit-identical to the reference (pinned by ``tests/test_oracle_golden.py``
against fixtures produced by ``oracle/make_golden.py``).

Not imported by the product package; see ``oracle/__init__.py``.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

WHITE = 220            # src/optics.py:22
CAP = 100_000          # src/optics.py:25
H_OD = (0.650, 0.704, 0.286)   # src/stain_sep.py:34
E_OD = (0.072, 0.990, 0.105)   # src/stain_sep.py:35
CHUNK = 64             # src/pipeline.py:36


class OracleError(Exception):
    """Domain error raised by the oracle; ``kind`` names the reference class."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# --------------------------------------------------------------------------
# order statistics — src/order_stats.py:11-47
# --------------------------------------------------------------------------
def pct(values, p):
    """src/order_stats.py:11-36 (linear interpolation, rank = p/100*(n-1))."""
    s = np.sort(np.asarray(values, dtype=np.float64).ravel())
    if s.size == 0:
        raise ValueError("empty")
    if not 0.0 <= p <= 100.0:
        raise ValueError("p out of range")
    r = (p / 100.0) * (s.size - 1)
    lo, hi = int(np.floor(r)), int(np.ceil(r))
    return float(s[lo] + (s[hi] - s[lo]) * (r - lo))


def mid(values):
    """src/order_stats.py:39-47."""
    s = np.sort(np.asarray(values, dtype=np.float64).ravel())
    if s.size == 0:
        raise ValueError("empty")
    k = s.size // 2
    return float(s[k]) if s.size % 2 else float((s[k - 1] + s[k]) / 2.0)


# --------------------------------------------------------------------------
# optics — src/optics.py:35-110
# --------------------------------------------------------------------------
def bg_intensity(pools):
    """src/optics.py:35-68: per-channel 80th percentile, 255 when empty."""
    out = np.empty(3)
    for c in range(3):
        a = np.asarray(pools[c], dtype=np.float64).ravel()
        out[c] = 255.0 if a.size == 0 else pct(a, 80.0)
    return out


def od_of(pixels, i0):
    """src/optics.py:71-94: v = ln(i0 / clip(i, 1, i0))."""
    i0 = np.asarray(i0, dtype=np.float64)
    if np.any(i0 < 1.0):
        raise ValueError("i0 < 1")
    x = np.array(pixels, dtype=np.float64)  # always a copy
    np.clip(x, 1.0, i0, out=x)
    return np.log(i0 / x)


def od_table(i0):
    """The (3, 256) OD lookup table: od_of on the 0..255 ramp, per channel."""
    ramp = np.repeat(np.arange(256, dtype=np.uint8)[:, None], 3, axis=1)
    return np.ascontiguousarray(od_of(ramp, i0).T)


def rgb_of(od, i0):
    """src/optics.py:97-110: floor(i0 * exp(-v) + 0.5) clipped to u8."""
    i0 = np.asarray(i0, dtype=np.float64)
    y = i0 * np.exp(-np.asarray(od, dtype=np.float64))
    y = np.floor(y + 0.5)
    np.clip(y, 0.0, 255.0, out=y)
    return y.astype(np.uint8)


# --------------------------------------------------------------------------
# stain separation — src/stain_sep.py:83-336
# --------------------------------------------------------------------------
def he_basis():
    """src/stain_sep.py:83-86."""
    m = np.array([H_OD, E_OD], dtype=np.float64).T
    return m / np.linalg.norm(m, axis=0)


def check_basis(w):
    """src/stain_sep.py:89-101."""
    w = np.asarray(w, dtype=np.float64)
    if w.shape != (3, 2) or not np.all(np.isfinite(w)) or np.any(w < 0):
        raise ValueError("bad basis")
    if np.any(np.abs(np.linalg.norm(w, axis=0) - 1.0) > 1e-9):
        raise ValueError("basis columns must have unit L2 norm")
    return w


def order_cols(w):
    """src/stain_sep.py:104-116: hematoxylin (larger red-blue) first."""
    w = check_basis(w)
    rb = w[0] - w[2]
    if rb[1] > rb[0]:
        return np.ascontiguousarray(w[:, ::-1]), (1, 0)
    return w.copy(), (0, 1)


def gram(w):
    """Gram entries in the reference's scalar order (src/stain_sep.py:197-199)."""
    g00 = w[0, 0] * w[0, 0] + w[1, 0] * w[1, 0] + w[2, 0] * w[2, 0]
    g11 = w[0, 1] * w[0, 1] + w[1, 1] * w[1, 1] + w[2, 1] * w[2, 1]
    g01 = w[0, 0] * w[0, 1] + w[1, 0] * w[1, 1] + w[2, 0] * w[2, 1]
    return g00, g01, g11


def nnl_cd(b0, b1, g00, g01, g11, lam, max_sweeps, tol=0.0):
    """src/stain_sep.py:119-165: seeded closed form + CD to bitwise fixed point."""
    t0, t1 = b0 - lam, b1 - lam
    det = g00 * g11 - g01 * g01
    if det > 1e-12:
        q0 = np.maximum(0.0, (g11 * t0 - g01 * t1) / det)
    else:
        q0 = np.maximum(0.0, t0 / g00)
    q1 = np.maximum(0.0, (t1 - g01 * q0) / g11)
    x0 = np.maximum(0.0, (t0 - g01 * q1) / g00)
    x1 = np.maximum(0.0, (t1 - g01 * x0) / g11)
    y0 = np.maximum(0.0, (t0 - g01 * x1) / g00)
    y1 = np.maximum(0.0, (t1 - g01 * y0) / g11)
    live = np.flatnonzero((np.abs(y0 - x0) > tol) | (np.abs(y1 - x1) > tol))
    x0, x1 = y0, y1
    for _ in range(max_sweeps):
        if live.size == 0:
            break
        y0 = np.maximum(0.0, (t0[live] - g01 * x1[live]) / g00)
        y1 = np.maximum(0.0, (t1[live] - g01 * y0) / g11)
        keep = (np.abs(y0 - x0[live]) > tol) | (np.abs(y1 - x1[live]) > tol)
        x0[live] = y0
        x1[live] = y1
        live = live[keep]
    return x0, x1


def densities(od, w, lam, max_sweeps=2000):
    """src/stain_sep.py:168-201: (3,N) OD -> (2,N) stain densities."""
    w = check_basis(w)
    if lam < 0:
        raise ValueError("lam < 0")
    v = np.asarray(od, dtype=np.float64)
    if v.ndim != 2 or v.shape[0] != 3:
        raise ValueError("od must be 3xN")
    b0 = w[0, 0] * v[0] + w[1, 0] * v[1] + w[2, 0] * v[2]
    b1 = w[0, 1] * v[0] + w[1, 1] * v[1] + w[2, 1] * v[2]
    g00, g01, g11 = gram(w)
    x0, x1 = nnl_cd(b0, b1, g00, g01, g11, float(lam), max_sweeps)
    return np.stack([x0, x1])


def objective(v, w, h, lam):
    """src/stain_sep.py:204-207."""
    r = v - w @ h
    return float(r.ravel() @ r.ravel() + lam * h.sum())


def snmf(v, lam=0.1, max_outer=200, rel_tol=1e-6, seed=0):
    """src/stain_sep.py:239-336 (with _w_step :210-236).

    Returns (basis, history, converged, iterations, flags) where flags lists
    the reference's warning conditions ("few", "noconv", "onestain").
    """
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.ndim != 2 or v.shape[0] != 3:
        raise ValueError("od_sample must be 3xM")
    m = v.shape[1]
    if m < 10:
        raise OracleError("InsufficientPixelsError", "need at least 10 OD samples")
    flags = ["few"] if m < 1000 else []
    w = he_basis() + np.random.default_rng(seed).uniform(0.0, 0.05, size=(3, 2))
    w = np.maximum(w, 0.0)
    w /= np.linalg.norm(w, axis=0)
    half = lam / 2.0

    def hstep(w):
        b0 = w[0, 0] * v[0] + w[1, 0] * v[1] + w[2, 0] * v[2]
        b1 = w[0, 1] * v[0] + w[1, 1] * v[1] + w[2, 1] * v[2]
        x0, x1 = nnl_cd(b0, b1, w[:, 0] @ w[:, 0], w[:, 0] @ w[:, 1],
                        w[:, 1] @ w[:, 1], half, max_sweeps=500, tol=1e-9)
        return np.stack([x0, x1])

    h = hstep(w)
    f = objective(v, w, h, lam)
    hist = [f]
    done = False
    it = 0
    for it in range(1, max_outer + 1):
        vht = v @ h.T
        hht = h @ h.T
        for j in (0, 1):                       # _w_step, src/stain_sep.py:221-235
            k = 1 - j
            if hht[j, j] <= 0.0:
                continue
            u = np.maximum(vht[:, j] - w[:, k] * hht[k, j], 0.0)
            nrm = float(np.linalg.norm(u))
            if nrm <= 1e-15:
                continue
            trial = w.copy()
            trial[:, j] = u / nrm
            ft = objective(v, trial, h, lam)
            if ft <= f:
                w, f = trial, ft
        h = hstep(w)
        f = objective(v, w, h, lam)
        hist.append(f)
        if abs(hist[-2] - f) <= rel_tol * max(abs(hist[-2]), 1e-12) or f <= 1e-12 * m:
            done = True
            break
    if not done:
        flags.append("noconv")
    rows = h.sum(axis=1)
    tot = float(rows.sum())
    if tot > 0 and float(rows.min()) <= 1e-9 * tot:
        flags.append("onestain")
    basis, _ = order_cols(w)
    return basis, hist, done, it, flags


# --------------------------------------------------------------------------
# statistics / recombination — src/normalize.py:58-151
# --------------------------------------------------------------------------
def p99_pooled(h):
    """src/normalize.py:83-100 (pooled mode)."""
    out = np.empty(2)
    for j in range(2):
        s = np.asarray(h[j], dtype=np.float64).ravel()
        if s.size == 0 or float(s.max(initial=0.0)) <= 0.0:
            raise OracleError("StainAbsentError", f"stain {j} absent")
        out[j] = pct(s, 99.0)
    return out


def p99_patchwise(pairs):
    """src/normalize.py:75-80 (median of per-patch p99 pairs)."""
    a = np.asarray(pairs, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 2 or a.shape[0] == 0:
        raise ValueError("bad pairs")
    return np.array([mid(a[:, 0]), mid(a[:, 1])])


def factors(src_p99, tgt_p99):
    """src/normalize.py:103-112 and the f<=0 check of src/pipeline.py:291-297."""
    s = np.asarray(src_p99, dtype=np.float64)
    t = np.asarray(tgt_p99, dtype=np.float64)
    if np.any(s <= 0.0):
        raise OracleError("DegenerateStainError", "source p99 is zero")
    f = t / s
    if np.any(f <= 0):
        raise OracleError("DegenerateStainError", "target p99 is zero")
    return f


def recolor(h, f, w_t, i0_t, shape):
    """src/normalize.py:115-151: W_t diag(f) h -> inverse Beer-Lambert."""
    w = check_basis(w_t)
    f = np.asarray(f, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    n = h.shape[1]
    if shape[0] * shape[1] != n:
        raise ValueError("shape mismatch")
    s0 = f[0] * h[0]
    s1 = f[1] * h[1]
    od = np.empty((n, 3))
    for c in range(3):
        od[:, c] = w[c, 0] * s0 + w[c, 1] * s1
    return rgb_of(od.reshape(shape[0], shape[1], 3), i0_t)


# --------------------------------------------------------------------------
# orchestration — src/pipeline.py:128-345
# --------------------------------------------------------------------------
class Plan:
    """SamplePlan fields, src/pipeline.py:39-59."""

    def __init__(self, max_patches=20, patch_size=1000, target_pixels=100_000,
                 background_fraction_cutoff=0.95, seed=0, white_threshold=WHITE,
                 sample_cap=CAP):
        self.max_patches = max_patches
        self.patch_size = patch_size
        self.target_pixels = target_pixels
        self.background_fraction_cutoff = background_fraction_cutoff
        self.seed = seed
        self.white_threshold = white_threshold
        self.sample_cap = sample_cap


def gather_sample(img, plan=None):
    """src/pipeline.py:128-200 on an in-memory (H, W, 3) u8 image.

    Returns dict(non_white=(M,3) u8, counts=[...], bright=(r,g,b) u8 arrays,
    visited=int, used=int).
    """
    plan = plan or Plan()
    hgt, wid = img.shape[:2]
    grid = [(x, y) for y in range(0, hgt, plan.patch_size)
            for x in range(0, wid, plan.patch_size)]
    order = np.random.default_rng(plan.seed).permutation(len(grid))
    limit = 10 * plan.max_patches
    thr = plan.white_threshold
    need_frac = 1.0 - plan.background_fraction_cutoff
    parts, counts = [], []
    pools, npool = [[], [], []], [0, 0, 0]
    got = visited = used = 0
    for k in order:
        if visited >= limit or used >= plan.max_patches or got >= plan.target_pixels:
            break
        x, y = grid[k]
        px = img[y:y + min(plan.patch_size, hgt - y),
                 x:x + min(plan.patch_size, wid - x)].reshape(-1, 3)
        visited += 1
        for c in range(3):
            if npool[c] < plan.sample_cap:
                vals = px[:, c]
                vals = vals[vals > thr][: plan.sample_cap - npool[c]]
                if vals.size:
                    pools[c].append(vals)
                    npool[c] += vals.size
        nw = ~np.all(px > thr, axis=1)
        if int(nw.sum()) < need_frac * px.shape[0]:
            continue
        used += 1
        take = px[nw][: plan.target_pixels - got]
        parts.append(take)
        counts.append(take.shape[0])
        got += take.shape[0]
    if got == 0:
        raise OracleError("BlankSlideError", "no non-white pixels")
    return dict(
        non_white=np.concatenate(parts),
        counts=counts,
        bright=tuple(np.concatenate(b) if b else np.empty(0, np.uint8) for b in pools),
        visited=visited,
        used=used,
    )


def fit_params(img, plan=None, lam=0.1, max_outer=200, rel_tol=1e-6, seed=0,
               code_lam=0.0, per_patch=False):
    """src/pipeline.py:203-257 → dict(i0, basis, p99, count, snmf_iters)."""
    s = gather_sample(img, plan)
    i0 = bg_intensity(s["bright"])
    v = np.ascontiguousarray(od_of(s["non_white"], i0).T)
    basis, hist, done, it, flags = snmf(v, lam, max_outer, rel_tol, seed)
    h = densities(v, basis, code_lam)
    if per_patch:
        pairs, at = [], 0
        for c in s["counts"]:
            part = h[:, at:at + c]
            if part.shape[1]:
                pairs.append((pct(part[0], 99.0), pct(part[1], 99.0)))
            at += c
        p99 = p99_patchwise(pairs)
    else:
        p99 = p99_pooled(h)
    return dict(i0=i0, basis=basis, p99=p99, count=h.shape[1], iters=it,
                history=hist, flags=flags, sample=s)


def recolor_strip(px, src, tgt, f, code_lam=0.0):
    """src/pipeline.py:260-272: the per-strip hot unit (64-row chunks)."""
    rows_all, wid = px.shape[:2]
    out = np.empty_like(px)
    for y in range(0, rows_all, CHUNK):
        rows = min(CHUNK, rows_all - y)
        od = od_of(px[y:y + rows], src["i0"])
        v = np.ascontiguousarray(od.reshape(-1, 3).T)
        h = densities(v, src["basis"], code_lam)
        out[y:y + rows] = recolor(h, f, tgt["basis"], tgt["i0"], (rows, wid))
    return out


def run_transform(img, src, tgt, strip_height=1024, workers=None, code_lam=0.0):
    """src/pipeline.py:275-345 on an in-memory image: strips through a pool.

    ``src``/``tgt`` are dicts with i0, basis, p99.  Returns the (H, W, 3) u8
    output.  The reference's bounded in-flight window and in-order commit are
    kept (at most ``workers`` strips outstanding).
    """
    f = factors(src["p99"], tgt["p99"])
    workers = workers or (os.cpu_count() or 1)
    hgt = img.shape[0]
    out = np.empty_like(img)
    strips = [(y, min(strip_height, hgt - y)) for y in range(0, hgt, strip_height)]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        window = []
        for y, h in strips:
            if len(window) >= workers:
                fut, y0, h0 = window.pop(0)
                out[y0:y0 + h0] = fut.result()
            window.append((pool.submit(recolor_strip, img[y:y + h].copy(), src, tgt,
                                       f, code_lam), y, h))
        for fut, y0, h0 in window:
            out[y0:y0 + h0] = fut.result()
    return out


# --------------------------------------------------------------------------
# synthetic fixtures — src/synthetic.py:26-121 (fixture generator only)
# --------------------------------------------------------------------------
def sparse_pairs(n, rng, pure_h=0.4, pure_e=0.4, lo=0.2, hi=2.0):
    """src/synthetic.py:26-41."""
    kind = rng.random(n)
    mag = rng.uniform(lo, hi, size=(2, n))
    h = np.zeros((2, n))
    only_h = kind < pure_h
    only_e = (kind >= pure_h) & (kind < pure_h + pure_e)
    both = ~(only_h | only_e)
    h[0, only_h] = mag[0, only_h]
    h[1, only_e] = mag[1, only_e]
    h[:, both] = mag[:, both] * 0.7
    return h


def dense_pairs(n, rng, min_h=0.65, max_h=2.0, zero_e=0.3, max_e=1.2):
    """src/synthetic.py:44-55."""
    h = np.empty((2, n))
    h[0] = rng.uniform(min_h, max_h, size=n)
    h[1] = rng.uniform(0.0, max_e, size=n)
    h[1, rng.random(n) < zero_e] = 0.0
    return h


def _render_block(width, height, y0, rows, seed, i0, tissue_fraction, layout, sampler):
    """src/synthetic.py:69-99 (_render_rows): rows [y0, y0+rows) of one
    256-row block; content depends only on (seed, y0 // 256)."""
    w = he_basis()
    rng = np.random.default_rng([seed, y0 // 256])
    n = width * rows
    if layout == "scatter":
        tissue = rng.random(n) < tissue_fraction
    elif layout == "block":
        side = max(1, int(round((tissue_fraction * width * height) ** 0.5)))
        bx, by = (width - side) // 2, (height - side) // 2
        ys = y0 + np.arange(rows)
        rin = (ys >= by) & (ys < by + side)
        cin = np.zeros(width, dtype=bool)
        cin[bx:bx + side] = True
        tissue = (rin[:, None] & cin[None, :]).ravel()
    else:
        raise ValueError(layout)
    h = np.zeros((2, n))
    k = int(tissue.sum())
    if k:
        h[:, tissue] = sampler(k, rng)
    od = (w @ h).T.reshape(rows, width, 3)
    return rgb_of(od, i0), h, tissue.reshape(rows, width)


def render(width, height, seed, i0=(255, 255, 255), tissue_fraction=0.6,
           layout="scatter", sampler=sparse_pairs):
    """src/synthetic.py:69-121 → (pixels u8 (H,W,3), densities (2,HW), mask)."""
    i0 = np.asarray(i0, dtype=np.float64)
    parts = [_render_block(width, height, y0, min(256, height - y0), seed, i0,
                           tissue_fraction, layout, sampler) for y0 in range(0, height, 256)]
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts], axis=1),
            np.concatenate([p[2] for p in parts]))


def render_band(width, height, seed, rows, i0=(255, 255, 255), tissue_fraction=0.6,
                layout="scatter", workers=None):
    """Pixels of the first ``rows`` rows of render(width, height, seed, ...)
    (identical bytes), 256-row blocks rendered on a thread pool — the
    CPU-baseline input of bench.py (fixture cost only)."""
    i0 = np.asarray(i0, dtype=np.float64)
    out = np.empty((rows, width, 3), np.uint8)

    def one(y0):
        keep = min(256, rows - y0)          # the block is drawn whole (same RNG stream)
        out[y0:y0 + keep] = _render_block(width, height, y0, min(256, height - y0), seed, i0,
                                          tissue_fraction, layout, sparse_pairs)[0][:keep]

    with ThreadPoolExecutor(max_workers=workers or (os.cpu_count() or 1)) as pool:
        list(pool.map(one, range(0, rows, 256)))
    return out
