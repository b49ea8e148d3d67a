"""Multi-process (gloo, world size 2, CPU) test of the row-band sharded fit logic.

The device kernels are replaced by NumPy emulations of their contracts
(per-chunk counts; ordered compaction), everything else is the product code:
``distributed.local_parts``, ``distributed.split_takes``, the reference visit
loop ``pipeline._visit``, and the all-gather / all-reduce(sum) exchange.  The
assembled sample must equal the single-process reference sampling.
"""
import os
import socket

import numpy as np
import pytest

from oracle import spcn_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _emulate_counts(band, part, thr):
    base, w, h, _ = part
    W = band.shape[1]
    rows = np.stack([band.reshape(-1, 3)[base + r * W: base + r * W + w] for r in range(h)])
    px = rows.reshape(-1, 3)
    nw = ~np.all(px > thr, axis=1)
    return np.array([nw.sum(), (px[:, 0] > thr).sum(), (px[:, 1] > thr).sum(),
                     (px[:, 2] > thr).sum()], dtype=np.int64), px


def _worker(rank, world, port, img, plan_kw, q):
    import torch.distributed as dist
    import torch

    from paper_1901_03088_b200 import distributed as dd
    from paper_1901_03088_b200.pipeline import SamplePlan, _visit

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, W = img.shape[:2]
        per = H // world
        r0 = rank * per
        rows = per if rank < world - 1 else H - r0
        band = np.ascontiguousarray(img[r0:r0 + rows])
        plan = SamplePlan(**plan_kw)
        rng = np.random.default_rng(plan.seed)
        origins = [(x, y) for y in range(0, H, plan.patch_size) for x in range(0, W, plan.patch_size)]
        order = rng.permutation(len(origins))
        ncand = min(len(order), 10 * plan.max_patches)
        rects = [(origins[i][0], origins[i][1], min(plan.patch_size, W - origins[i][0]),
                  min(plan.patch_size, H - origins[i][1])) for i in order[:ncand]]
        parts = dd.local_parts(rects, r0, rows, W)
        thr = plan.white_threshold
        local = np.zeros((ncand, 4), dtype=np.int64)
        pix = {}
        for i, p in enumerate(parts):
            if p is not None:
                local[i], pix[i] = _emulate_counts(band, p, thr)
        lt = torch.from_numpy(local)
        gathered = [torch.empty_like(lt) for _ in range(world)]
        dist.all_gather(gathered, lt)
        per_rank = np.stack([g.numpy() for g in gathered])
        glob = per_rank.sum(axis=0)
        takes, counts, collected, visited, used = _visit(
            plan, order[:ncand], rects, lambda k: tuple(int(v) for v in glob[k]))
        sample = np.zeros((collected, 3), dtype=np.int64)
        hist = np.zeros((3, 256), dtype=np.int64)
        for cand, tnw, base, tb in dd.split_takes(takes, per_rank, rank):
            px = pix[cand]
            nw = px[~np.all(px > thr, axis=1)][:tnw]
            sample[base:base + len(nw)] = nw
            for c in range(3):
                vals = px[:, c][px[:, c] > thr][:tb[c]]
                hist[c] += np.bincount(vals, minlength=256)
        st = torch.from_numpy(sample)
        ht = torch.from_numpy(hist)
        dist.all_reduce(st)
        dist.all_reduce(ht)
        if rank == 0:
            q.put((st.numpy().astype(np.uint8), ht.numpy(), counts, visited, used))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("plan_kw", [dict(patch_size=128, target_pixels=30_000, seed=3),
                                     dict(patch_size=100, target_pixels=5_000, seed=1,
                                          sample_cap=700, max_patches=4)])
def test_row_band_fit_sample_equals_single_process(plan_kw):
    import torch.multiprocessing as mp

    img, _, _ = orc.render(300, 333, 5, tissue_fraction=0.5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, img, plan_kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    sample, hist, counts, visited, used = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = orc.gather_sample(img, orc.Plan(**plan_kw))
    assert np.array_equal(sample, ref["non_white"])
    assert np.array_equal(hist, np.stack([np.bincount(b, minlength=256) for b in ref["bright"]]))
    assert list(counts) == list(ref["counts"])
    assert (visited, used) == (ref["visited"], ref["used"])


def test_split_takes_partitions_global_takes():
    from paper_1901_03088_b200.distributed import split_takes

    per_rank = np.array([[[5, 3, 0, 9]], [[7, 4, 2, 1]], [[2, 2, 2, 2]]], dtype=np.int64)
    takes = [(0, 10, 100, [6, 1, 10])]
    got = [split_takes(takes, per_rank, r) for r in range(3)]
    assert got[0] == [(0, 5, 100, [3, 0, 9])]
    assert got[1] == [(0, 5, 105, [3, 1, 1])]
    assert got[2] == []


# ---------------------------------------------------------------------------
# global p99 across ranks: window logic + TorchComm (gloo), passes emulated
class _NumpyEngine:
    """Contract of the stats passes on exact densities (fp32 keys for the
    histograms, exact values for the refine), as the kernels provide them."""

    def __init__(self, h):
        self.h = h

    def hist(self, base, shift):
        import torch

        from paper_1901_03088_b200.global_stats import NBINS

        hist = np.zeros((2, NBINS), np.int64)
        counts = np.zeros(3, np.int64)
        counts[0] = self.h.shape[1]
        for j in range(2):
            keys = self.h[j].astype(np.float32).view(np.uint32).astype(np.int64)
            counts[1 + j] = int((keys < base[j]).sum())
            d = (keys[keys >= base[j]] - base[j]) >> shift[j]
            d = d[d < NBINS]
            hist[j] += np.bincount(d, minlength=NBINS)[:NBINS]
        return torch.from_numpy(hist), torch.from_numpy(counts)

    def refine(self, lo, hi, cap):
        import torch

        counts = np.zeros(7, np.int64)
        cand = np.zeros((2, max(cap, 1)))
        wcnt = np.zeros((2, max(cap, 1)), np.int64)
        for j in range(2):
            x = self.h[j]
            counts[j] = int((x < lo[j]).sum())
            w = x[(x >= lo[j]) & (x < hi[j])]
            counts[2 + j] = w.size
            u, c = np.unique(w, return_counts=True)        # (value, count) pairs
            counts[5 + j] = u.size
            cand[j, :min(cap, u.size)] = u[:cap]
            wcnt[j, :min(cap, u.size)] = c[:cap]
        return torch.from_numpy(counts), torch.from_numpy(cand), torch.from_numpy(wcnt)


class _TableEngine(_NumpyEngine):
    """Adds the one-pass colour-table contract: `ids` maps each pixel to a
    colour of the shared palette `pal` (2, C) of exact densities."""

    def __init__(self, h, ids, pal):
        super().__init__(h)
        self.ids, self.pal = ids, pal

    def table(self, lo):
        import torch

        cand = (self.h[0] >= lo[0]) | (self.h[1] >= lo[1])   # superset of "not surely below"
        tab = np.bincount(self.ids[cand], minlength=self.pal.shape[1]).astype(np.int64)
        return torch.from_numpy(tab), torch.tensor([self.h.shape[1]], dtype=torch.int64)

    def scan(self, tab):
        import torch

        present = torch.nonzero(tab).reshape(-1)
        x = torch.from_numpy(np.ascontiguousarray(self.pal.T))[present]
        xmax = x.max(dim=0).values.numpy() if x.numel() else np.zeros(2)
        return x, tab[present], xmax, False

    # the selection kernels' contract (csrc/stats.cu k_entries_hist / _collect)
    @staticmethod
    def _bins(v, lo, scale, nbins):
        b = np.minimum(np.floor((v - lo) * scale), nbins - 1).astype(np.int64)
        return np.where(v >= lo, b, -1)

    def entries_hist(self, x, w, lo, scale, nbins):
        import torch

        x, w = x.numpy(), w.numpy()
        hist = np.zeros((2, nbins), np.int64)
        for j in range(2):
            b = self._bins(x[:, j], lo[j], scale[j], nbins)
            np.add.at(hist[j], b[b >= 0], w[b >= 0])
        return torch.from_numpy(hist)

    def entries_collect(self, x, w, lo, scale, nbins, bins):
        import torch

        x, w = x.numpy(), w.numpy()
        out = []
        for j in range(2):
            b = self._bins(x[:, j], lo[j], scale[j], nbins)
            sel = (b >= bins[2 * j]) & (b <= bins[2 * j + 1])
            out.append((torch.from_numpy(x[sel, j].copy()), torch.from_numpy(w[sel].copy())))
        return out


def _palette_slide(n, seed):
    """Densities drawn from a palette of 3000 colours (as a slide's are)."""
    rng = np.random.default_rng(seed)
    pal = np.zeros((2, 3000))
    pal[0] = rng.gamma(2.0, 0.4, 3000)
    pal[1] = rng.gamma(1.5, 0.3, 3000)
    pal[:, :300] = 0.0
    ids = rng.integers(0, 3000, n)
    return pal[:, ids], ids, pal


def test_global_p99_table_mode():
    from paper_1901_03088_b200.global_stats import global_p99

    h, ids, pal = _palette_slide(100_000, 3)
    ref = np.array([orc.pct(h[0], 99.0), orc.pct(h[1], 99.0)])
    good = np.stack([ref * 0.9, ref * 1.1], axis=1)
    p99, n, info = global_p99(None, None, None, engine=_TableEngine(h, ids, pal), guess=good)
    assert n == h.shape[1] and np.array_equal(p99, ref), info
    assert info["passes"] == 1 and info["mode"] == "table", info
    high = np.stack([ref * 1.2, ref * 1.3], axis=1)              # lower end above p99: miss
    p99, _, info = global_p99(None, None, None, engine=_TableEngine(h, ids, pal), guess=high)
    assert np.array_equal(p99, ref) and info.get("table_miss") and info["passes"] >= 2, info


def _table_worker(rank, world, port, parts, pal, q):
    import torch.distributed as dist

    from paper_1901_03088_b200 import distributed as dd
    from paper_1901_03088_b200.global_stats import global_p99

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h, ids = parts[rank]
        ref = [0.5, 0.5]
        p99, n, info = global_p99(None, None, None, comm=dd.TorchComm(),
                                  engine=_TableEngine(h, ids, pal),
                                  guess=np.array([[r * 0.5, r * 4] for r in ref]))
        q.put((rank, p99.tolist(), n, info.get("mode")))
    finally:
        dist.destroy_process_group()


def test_global_p99_table_mode_two_ranks_gloo():
    import multiprocessing as mp

    h, ids, pal = _palette_slide(60_000, 8)
    parts = [(h[:, :25_000], ids[:25_000]), (h[:, 25_000:], ids[25_000:])]
    ref = [orc.pct(h[0], 99.0), orc.pct(h[1], 99.0)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_table_worker, args=(r, 2, port, parts, pal, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    got = [q.get(timeout=120) for _ in ps]
    for pr in ps:
        pr.join(timeout=60)
    for rank, p99, n, mode in got:
        assert n == h.shape[1] and mode == "table"
        assert p99 == ref, (rank, p99, ref)


def _global_worker(rank, world, port, hs, q):
    import torch.distributed as dist

    from paper_1901_03088_b200 import distributed as dd
    from paper_1901_03088_b200.global_stats import global_p99

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p99, n, info = global_p99(None, None, None, comm=dd.TorchComm(),
                                  engine=_NumpyEngine(hs[rank]))
        q.put((rank, p99.tolist(), n))
    finally:
        dist.destroy_process_group()


def test_global_p99_bracket_window_logic():
    """Window logic seeded with a bracket (hit: one histogram level + one
    refine; miss: full-range fallback), single process."""
    from paper_1901_03088_b200.global_stats import global_p99

    rng = np.random.default_rng(9)
    n = 200_000
    h = np.zeros((2, n))
    h[0] = rng.gamma(2.0, 0.4, n)
    h[1] = rng.gamma(1.5, 0.3, n)
    h[:, rng.random(n) < 0.2] = 0.0
    ref = np.array([orc.pct(h[0], 99.0), orc.pct(h[1], 99.0)])
    good = np.stack([ref * 0.97, ref * 1.02], axis=1)
    for guess, passes in ((good, 2), (np.array([[9.0, 9.5], [9.0, 9.5]]), None), (ref, None)):
        p99, cnt, info = global_p99(None, None, None, engine=_NumpyEngine(h), guess=guess)
        assert cnt == n and np.array_equal(p99, ref), (guess, info)
        if passes:
            assert info["passes"] == passes, info


def test_global_p99_two_ranks_gloo():
    import multiprocessing as mp

    rng = np.random.default_rng(4)
    n = 50_000
    h = np.zeros((2, n))
    h[0] = rng.gamma(2.0, 0.4, n)
    h[1] = rng.gamma(1.5, 0.3, n)
    h[:, rng.random(n) < 0.3] = 0.0                   # many exact zeros (clamped densities)
    hs = [h[:, :20_000], h[:, 20_000:]]              # unequal bands
    ref = [orc.pct(h[0], 99.0), orc.pct(h[1], 99.0)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_global_worker, args=(r, 2, port, hs, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, p99, cnt in out:
        assert cnt == n
        assert p99 == ref, (rank, p99, ref)


def test_sample_bracket_ranks_contain_the_percentile():
    """The bracket's ranks around p99 of a 100 k sample contain the sample's
    own p99 (sample_bracket selects exactly these order statistics on the
    device; its GPU test is tests/test_global_stats_gpu.py)."""
    from paper_1901_03088_b200.global_stats import bracket_ranks

    rng = np.random.default_rng(5)
    h = np.stack([rng.gamma(2.0, 0.4, 100_000), rng.gamma(1.5, 0.3, 100_000)])
    lo, hi = bracket_ranks(h.shape[1])
    assert 0 <= lo < hi < h.shape[1]
    for j in range(2):
        srt = np.sort(h[j])
        p = orc.pct(h[j], 99.0)
        assert srt[lo] <= p <= srt[hi]
        assert srt[lo] > 0


def test_fit_slide_cluster_choice_and_fallback(monkeypatch):
    """One slide's SNMF: one CTA below 20 k samples, a 16-CTA cluster above,
    and a sticky fall-back to 8 when 16-CTA clusters cannot be launched."""
    from paper_1901_03088_b200 import snmf

    calls = []

    def fake(samples, offsets, luts, cfg, cluster=1, od=None):
        calls.append(cluster)
        if cluster == 16:
            raise RuntimeError("cluster too large")
        return cluster

    monkeypatch.setattr(snmf, "snmf_batched", fake)
    monkeypatch.setattr(snmf, "_BIG_CLUSTER", [16])
    assert snmf.fit_slide(None, None, None, None, 1_000) == 1
    assert snmf.fit_slide(None, None, None, None, 50_000) == 8
    assert snmf.fit_slide(None, None, None, None, 50_000) == 8
    assert calls == [1, 16, 8, 8]


def test_host_copy_helpers():
    """pipeline._pcopy (threaded multi-MB copies) and batch._sliced_copy
    (copies in <= 64 MB pieces) are plain copies."""
    import torch

    from paper_1901_03088_b200 import batch, pipeline

    rng = np.random.default_rng(3)
    src = rng.integers(0, 256, (1500, 1200, 3), dtype=np.uint8)     # 5.4 MB: threaded path
    dst = np.empty_like(src)
    pipeline._pcopy(dst, src)
    assert np.array_equal(dst, src)
    small = src[:10]
    d2 = np.empty_like(small)
    pipeline._pcopy(d2, small)
    assert np.array_equal(d2, small)
    t_src = torch.from_numpy(rng.integers(0, 256, (37, 64, 64, 3), dtype=np.uint8))
    t_dst = torch.empty_like(t_src)
    old = batch._SLICE_BYTES
    try:
        batch._SLICE_BYTES = 5 * 64 * 64 * 3          # pieces of 5 items
        batch._sliced_copy(t_dst, t_src, False)
    finally:
        batch._SLICE_BYTES = old
    assert torch.equal(t_dst, t_src)


def _max_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1901_03088_b200 import distributed as dd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the calibration word: bits of a non-negative float, max-reduced as int32
        w = torch.tensor(np.array([0.5e-6 * (rank + 1)], dtype=np.float32).view(np.int32))
        dd.all_reduce_max(w)
        q.put((rank, float(w.numpy().view(np.float32)[0])))
    finally:
        dist.destroy_process_group()


def test_all_reduce_max_of_float_bits_two_ranks():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_max_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    got = [q.get(timeout=120) for _ in ps]
    for pr in ps:
        pr.join(timeout=60)
    want = float(np.float32(1.0e-6))
    assert all(v == want for _, v in got), got
