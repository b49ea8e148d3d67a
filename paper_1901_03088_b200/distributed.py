"""Row-band sharding of one whole-slide image across GPUs.

Every rank holds a contiguous band of full-width rows [r0, r0 + rows) of a
W x H slide.  The transform needs no exchange (it is pointwise-pure: output
is bit-identical for any strip partition, src/pipeline.py:275-345).  The
sample-mode fit (src/pipeline.py:128-257) is made distributed without moving
pixels except the ≤100 k sampled ones:

  1. every rank derives the same seeded patch visit order (numpy PCG64);
  2. each rank counts (non-white, bright R/G/B) on its slice of every
     candidate patch; an all-gather of those per-rank totals (ranks x
     candidates x 4 int64) gives every rank the global per-patch counts and
     the per-rank prefix inside each patch's raster order;
  3. every rank replays the reference's visit loop on the global counts
     (identical decisions everywhere), converts the global takes into its own
     local takes (clip by the prefix of lower ranks), and compacts its
     pixels into their global positions of the sample buffer;
  4. one all-reduce(sum) of the sample bytes (disjoint writers) and of the
     3 x 256 bright histogram completes the sample on every rank;
  5. every rank runs the (deterministic) i0 → SNMF → coding → p99 chain on
     the identical sample, so all ranks hold identical FitParams with no
     broadcast.

Collectives: one all-gather (KBs) and two all-reduces (~300 KB) per fit over
NCCL/NVLink.  The host-side pieces (``local_parts``, ``split_takes``) are
pure functions tested on CPU with gloo, world size 2.
"""
from __future__ import annotations

import numpy as np

from . import _dev, _lib

CHUNK = 4096


def local_parts(rects, r0: int, rows: int, width: int):
    """Intersect global candidate rects (x, y, w, h) with the band.

    Returns a list aligned with ``rects`` of (base_px, w, h_local, row_offset)
    or None when the patch has no rows in this band.  ``base_px`` is the pixel
    offset of the slice's first pixel inside the band buffer, ``row_offset``
    the first patch row the slice covers (its raster rank start is
    row_offset * w).
    """
    out = []
    for (x, y, w, h) in rects:
        a, b = max(y, r0), min(y + h, r0 + rows)
        if a >= b:
            out.append(None)
        else:
            out.append(((a - r0) * width + x, w, b - a, a - y))
    return out


def split_takes(takes, per_rank_totals, rank: int):
    """Global takes → this rank's takes.

    takes: list of (cand, take_nonwhite, out_base, [tb_r, tb_g, tb_b]) from the
    visit loop; per_rank_totals: (world, ncand, 4) local counts of every rank
    (ranks are ordered by band, i.e. by raster order inside a patch).
    Returns list of (cand, take_nonwhite, out_base, [tb...]) for this rank,
    omitting entries with nothing to take.
    """
    prefix = per_rank_totals[:rank].sum(axis=0)        # (ncand, 4) counts of lower ranks
    mine = per_rank_totals[rank]
    res = []
    for cand, tnw, base, tb in takes:
        pre, loc = prefix[cand], mine[cand]
        lnw = int(np.clip(tnw - pre[0], 0, loc[0]))
        ltb = [int(np.clip(tb[c] - pre[1 + c], 0, loc[1 + c])) for c in range(3)]
        if lnw or any(ltb):
            res.append((cand, lnw, int(base + min(pre[0], tnw)), ltb))
    return res


def _host_staged(group) -> bool:
    """gloo moves CUDA tensors only for some collectives: stage through host."""
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def all_reduce_sum(t, group=None):
    """In-place sum all-reduce of a tensor on any device (NCCL: device-direct)."""
    import torch.distributed as dist

    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)
    return t


def all_reduce_max(t, group=None):
    """In-place max all-reduce (NCCL: device-direct; gloo: host-staged)."""
    import torch.distributed as dist

    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def all_gather_list(t, group=None):
    """All-gather of equal-shape tensors → list (host-staged under gloo)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    src = t.cpu() if (t.is_cuda and _host_staged(group)) else t
    out = [torch_empty_like(src) for _ in range(world)]
    dist.all_gather(out, src, group=group)
    return [o.to(t.device) for o in out]


def torch_empty_like(t):
    import torch

    return torch.empty_like(t)


class TorchComm:
    """Sum all-reduce and variable-size all-gather over a torch.distributed
    group (NCCL on GPUs, gloo in the CPU tests) — the collectives of the
    global-p99 passes."""

    def __init__(self, group=None):
        self.group = group

    def allreduce(self, t):
        return all_reduce_sum(t, self.group)

    def allgather(self, t):
        import torch

        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [int(x.item()) for x in all_gather_list(n, self.group)]
        m = max(sizes + [1])
        pad = torch.zeros(m, dtype=t.dtype, device=t.device)
        pad[:t.numel()] = t.reshape(-1)
        return [o[:k] for o, k in zip(all_gather_list(pad, self.group), sizes)]


class RowBandGroup:
    """Fit and transform of a row-band-sharded slide (one instance per rank;
    both methods are collectives)."""

    def __init__(self, width: int, height: int, r0: int, rows: int, group=None):
        self.width, self.height, self.r0, self.rows = width, height, r0, rows
        self.group = group

    def transform(self, band_source, source, target, sink, **kw):
        """pipeline.transform of this rank's band.  EXACT on a resident band:
        the exhaustive certification calibration is split across the ranks
        (each evaluates 1/N of the 2^24 colours, then a max all-reduce of one
        word) instead of every rank evaluating all of it."""
        import torch.distributed as dist

        from .pipeline import transform

        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)

        def calibrate(plan, npix):
            plan.calibrate_shared(self.width * self.height, npix, rank, world,
                                  lambda w: all_reduce_max(w, self.group))

        return transform(band_source, source, target, sink, _calibrate=calibrate, **kw)

    def fit(self, band_source, plan=None, cfg=None, *, code_lam: float = 0.0,
            per_patch_stats: bool = False, source_label: str = "", p99_mode: str = "sample"):
        """pipeline.fit of the whole slide from the row bands (a collective:
        every rank returns the same FitParams)."""
        from . import fitcore
        from .pipeline import SamplePlan, _stage, slide_chunks
        from .stain_sep import SnmfConfig

        plan = plan or SamplePlan()
        cfg = cfg or SnmfConfig()
        fb, sample, m, i0, used_counts = self._gather_sample(band_source, plan, cfg)
        return fitcore.fit_tail(fb, sample.reshape(-1), m, i0, plan, cfg, code_lam=code_lam,
                                per_patch_stats=per_patch_stats, p99_mode=p99_mode,
                                used_counts=used_counts, source_label=source_label,
                                chunks=slide_chunks(band_source) if p99_mode == "global" else None,
                                comm=TorchComm(self.group), stage=_stage)

    def fit_transform(self, band_source, target, out, plan=None, cfg=None, *,
                      code_lam: float = 0.0, source_label: str = ""):
        """fit() of the whole slide, then this rank's band recoloured into the
        CUDA tensor `out` (EXACT, pooled p99) with the recolouring built on
        the device from the fit (spcn_xform_fitted_prepare / _run): one host
        wait for the build, the certification calibration split across the
        ranks (1/N of the colours each, one int32 max all-reduce on the
        stream), no host round trip between the fit and the recolour.  Same
        bytes as fit() + transform(); a recolouring the device declines is
        redone by transform() with host parameters (identically on every
        rank: the fit is the same everywhere).  A collective; returns the fit."""
        import ctypes

        import torch.distributed as dist

        from . import fitcore
        from .image_io import DeviceWriter
        from .pipeline import SamplePlan, _fitted_params
        from .stain_sep import SnmfConfig

        plan = plan or SamplePlan()
        cfg = cfg or SnmfConfig()
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        src = band_source.tensor
        if (src.data_ptr() - out.data_ptr()) % 16 != 0:
            raise ValueError("fit_transform: band and out must share their 16-byte alignment phase")
        if tuple(out.shape) != tuple(src.shape) or not out.is_contiguous():
            raise ValueError("fit_transform: out must be a contiguous tensor shaped like the band")
        L = _lib.lib()
        npix = src.numel() // 3
        p = _fitted_params(target, float(code_lam), self.width * self.height)
        ws_bytes = int(L.spcn_xform_workspace_bytes(max(npix, 1)))
        st = _lib.stream_handle()
        ws = _dev.workspace(ws_bytes, stream=st)
        fb, sample, m, i0, _ = self._gather_sample(band_source, plan, cfg)
        p.src_od_table = fb.lut_ptr
        p.src_fit = fb.arena_b_ptr
        fitcore.basis_enqueue(fb, _lib.ptr(sample), m, i0, cfg, code_lam=code_lam, pooled=True)
        slot = ctypes.c_int32(-1)
        fb.pin_status_np[0] = -1
        _lib.check(L.spcn_xform_fitted_prepare(ctypes.byref(p), rank, world, _lib.ptr(ws),
                                               ws_bytes, fb.pin_status_ptr, ctypes.byref(slot),
                                               st), "xform_fitted_prepare")
        try:
            prov = fitcore.provenance(plan, cfg, code_lam, False, "sample", source_label)
            fp = fitcore.parse_pooled(fb, m, i0, cfg, prov, stacklevel=3)
        except Exception:
            L.spcn_xform_fitted_run(None, None, 0, slot.value, _lib.ptr(ws), ws_bytes, st)
            raise
        ok = int(fb.pin_status_np[0]) == 0
        all_reduce_max(ws[8:12].view(_dev.torch().int32), self.group)
        _lib.check(L.spcn_xform_fitted_run(_lib.ptr(src), _lib.ptr(out), npix if ok else 0,
                                           slot.value, _lib.ptr(ws), ws_bytes, st),
                   "xform_fitted_run")
        if not ok:
            self.transform(band_source, fp, target, DeviceWriter(src.shape[1], src.shape[0],
                                                                 out=out),
                           code_lam=code_lam, precision="exact")
        return fp

    def _gather_sample(self, band_source, plan, cfg):
        """The collective sampling of fit(): per-rank patch counts all-gathered,
        the reference's visit loop replayed on the host, each rank compacting
        the takes inside its band, sample + bright histograms summed in one
        all-reduce, i0 on the host.  Returns (FitBuffers, sample (m, 3) CUDA
        uint8, m, i0, used patch counts)."""
        import torch
        import torch.distributed as dist

        from . import fitcore, optics
        from .errors import BlankSlideError
        from .pipeline import PATCH_DT, TAKE_DT, _lib_sample, _stage, _visit

        L = _lib_sample()
        W = self.width
        rank = dist.get_rank(self.group)
        img = band_source.tensor
        thr = int(plan.white_threshold)
        dev = img.device
        # the seeded candidate patches and this band's parts of them: a pure
        # function of (slide geometry, band, plan), built once per plan (the
        # 10 000-origin grid of a 100 k^2 slide costs ~3 ms of Python)
        cache = self.__dict__.setdefault("_cand", {})
        c = cache.get((plan, dev))
        if c is None:
            from .pipeline import _candidates

            order, ncand, rects = _candidates(W, self.height, plan)
            parts = local_parts(rects, self.r0, self.rows, W)
            present = [i for i, p in enumerate(parts) if p is not None]
            chunks = max([1] + [-(-(p[1] * p[2]) // CHUNK) for p in parts if p is not None])
            c = dict(order=order[:ncand].copy(), ncand=ncand, rects=rects, parts=parts,
                     present=present, chunks=chunks)
            if present:
                desc = np.array([(parts[i][0], parts[i][1], parts[i][2], W) for i in present],
                                dtype=PATCH_DT)
                c["d"] = torch.from_numpy(desc.view(np.uint8).copy()).to(dev)
                c["present_dev"] = torch.tensor(present, dtype=torch.int64, device=dev)
            if len(cache) > 8:
                cache.clear()
            cache[(plan, dev)] = c
        order, ncand, rects, parts = c["order"], c["ncand"], c["rects"], c["parts"]
        present, chunks = c["present"], c["chunks"]
        lt = torch.zeros((ncand, 4), dtype=torch.int64, device=dev)
        cnt_dev = None
        if present:
            cnt_dev = torch.empty((len(present), chunks, 4), dtype=torch.int32, device=dev)
            _lib.check(L.spcn_sample_count(_lib.ptr(img), _lib.ptr(c["d"]), len(present), chunks,
                                           thr, _lib.ptr(cnt_dev), _lib.stream_handle()),
                       "sample_count")
            lt[c["present_dev"]] = cnt_dev.sum(dim=1).to(torch.int64)
        # all-gather of per-rank totals (ranks in band order), one host read
        gathered = all_gather_list(lt, self.group)
        per_rank = torch.stack([g.to(dev) for g in gathered]).cpu().numpy()
        glob = per_rank.sum(axis=0)
        takes, used_counts, collected, visited, used = _visit(
            plan, order, rects, lambda k: tuple(int(v) for v in glob[k]))
        if collected == 0:
            raise BlankSlideError("sampling: blank slide: no non-white pixels found in any "
                                  "sampled patch")
        # sample bytes and bright histograms in ONE int32 buffer, one all-reduce:
        # each sample byte has a single writer, so word sums are byte sums
        nw = -(-3 * collected // 4)
        buf = torch.zeros(nw + 3 * 256, dtype=torch.int32, device=dev)
        sample = buf[:nw].view(torch.uint8)[:3 * collected].view(collected, 3)
        hist = buf[nw:].view(1, 3, 256)
        mine = [tk for tk in split_takes(takes, per_rank, rank) if parts[tk[0]] is not None]
        if mine:
            pos = {c: j for j, c in enumerate(present)}
            idx = np.array([pos[tk[0]] for tk in mine], dtype=np.int64)
            desc = np.array([(parts[tk[0]][0], parts[tk[0]][1], parts[tk[0]][2], W)
                             for tk in mine], dtype=PATCH_DT)
            tk = np.zeros(len(mine), dtype=TAKE_DT)
            tk["take_nonwhite"] = [m[1] for m in mine]
            tk["out_base"] = [m[2] for m in mine]
            tk["take_bright"] = [m[3] for m in mine]
            cnt = cnt_dev[torch.from_numpy(idx).to(dev)].contiguous()
            d = torch.from_numpy(desc.view(np.uint8).copy()).to(dev)
            dt = torch.from_numpy(tk.view(np.uint8).copy()).to(dev)
            _lib.check(L.spcn_sample_compact(_lib.ptr(img), _lib.ptr(d), len(mine), chunks, thr,
                                             _lib.ptr(cnt), _lib.ptr(dt), _lib.ptr(sample),
                                             _lib.ptr(hist), _lib.stream_handle()),
                       "sample_compact")
        all_reduce_sum(buf, self.group)        # disjoint sample writers: sum == gather
        # --- identical, deterministic fit on every rank (the single-process tail)
        m = collected
        i0 = _stage("background estimation", optics.i0_from_counts,
                    hist.cpu().numpy()[0].astype(np.int64))
        fb = fitcore.buffers(dev, plan.target_pixels, cfg.max_outer_iters)
        # [0, m] through the pinned staging buffer: stream-ordered, no host wait
        # (the previous fit's copy from it completed before that fit's read-back)
        fb.pin_a_np[128:144].view(np.int64)[:] = (0, m)
        fb.offsets().copy_(fb.pin_a[128:144].view(torch.int64), non_blocking=True)
        return fb, sample, m, i0, used_counts
