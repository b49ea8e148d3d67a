"""GPU parity of the batched path (configs[1]: many patches, one target).

Each item must give exactly what the single-image path and the reference
give for it: fit parameters (i0 exact, basis/p99 as in test_fit_gpu), output
bytes bit-identical in exact/strict precision, per-item errors of the same
class as the reference's (src/cli.py:220-244, 270-301) without disturbing the
other items.
"""
import warnings

import numpy as np
import pytest

from oracle import spcn_oracle as orc

pytestmark = pytest.mark.gpu


def _pb():
    import paper_1901_03088_b200 as pb

    return pb


def _items(h, w, n, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        i0 = tuple(int(v) for v in rng.integers(228, 256, size=3))
        frac = float(rng.uniform(0.3, 0.9))
        sampler = orc.sparse_pairs if k % 2 == 0 else orc.dense_pairs
        px, _, _ = orc.render(w, h, seed * 1000 + k, i0=i0, tissue_fraction=frac,
                              sampler=sampler)
        out.append(px)
    return out


def _target(pb, seed=77):
    px, _, _ = orc.render(256, 192, seed, i0=(246, 242, 250))
    ft = orc.fit_params(px)
    return pb.FitParams(i0=ft["i0"], basis=ft["basis"],
                        stats=pb.StainStats(p99=np.asarray(ft["p99"]), sample_count=ft["count"]))


def _oracle_item(px, plan, tgt, code_lam=0.0):
    """(fit dict, output) or (error kind, None) for one item."""
    try:
        src = orc.fit_params(px, plan)
    except orc.OracleError as e:
        return e.kind, None
    t = {"i0": tgt.i0, "basis": tgt.basis, "p99": tgt.stats.p99}
    try:
        out = orc.run_transform(px, src, t, workers=1, code_lam=code_lam)
    except orc.OracleError as e:
        return e.kind, None
    return src, out


def _run(pb, imgs, plan, tgt, precision="exact"):
    import torch

    x = torch.from_numpy(np.stack(imgs)).cuda()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out, errors, fits = pb.normalize_batch(x, tgt, plan=plan, precision=precision)
    return out.cpu().numpy(), errors, fits


@pytest.mark.parametrize("shape,plan_kw", [
    ((96, 160), {}),                                                   # one patch per item
    ((128, 192), dict(patch_size=64, max_patches=2, target_pixels=3000)),  # visit loop
    ((33, 37), {}),                                                    # unaligned item size
])
def test_batch_matches_reference_per_item(shape, plan_kw):
    pb = _pb()
    h, w = shape
    imgs = _items(h, w, 9, seed=h)
    imgs[3] = np.full((h, w, 3), 255, np.uint8)                 # blank item
    tgt = _target(pb)
    plan = pb.SamplePlan(**plan_kw)
    oplan = orc.Plan(**plan_kw)
    out, errors, fits = _run(pb, imgs, plan, tgt)
    for i, px in enumerate(imgs):
        src, ref = _oracle_item(px, oplan, tgt)
        if ref is None:
            assert errors[i] is not None and type(errors[i]).__name__ == src, (i, errors[i], src)
            continue
        assert errors[i] is None, (i, errors[i])
        fp = fits.params(i)
        assert np.array_equal(fp.i0, src["i0"]), i
        np.testing.assert_allclose(fp.basis, src["basis"], atol=1e-9, err_msg=str(i))
        np.testing.assert_allclose(fp.stats.p99, src["p99"], rtol=1e-9, err_msg=str(i))
        assert fp.stats.sample_count == src["count"], i
        assert np.array_equal(out[i], ref), (i, int((out[i] != ref).sum()))


def test_batch_equals_single_item_path():
    import torch

    pb = _pb()
    imgs = _items(112, 144, 6, seed=5)
    tgt = _target(pb, 3)
    plan = pb.SamplePlan()
    out, errors, fits = _run(pb, imgs, plan, tgt)
    for i, px in enumerate(imgs):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fp = pb.fit(torch.from_numpy(px).cuda(), plan)
        bp = fits.params(i)
        assert np.array_equal(bp.i0, fp.i0)
        assert np.array_equal(bp.basis, fp.basis)
        assert np.array_equal(bp.stats.p99, fp.stats.p99)
        sink = pb.DeviceWriter(px.shape[1], px.shape[0])
        pb.transform(pb.DeviceSource(torch.from_numpy(px).cuda()), fp, tgt, sink)
        assert np.array_equal(sink.pixels.cpu().numpy(), out[i])


@pytest.mark.parametrize("precision", ["strict", "fast"])
def test_batch_precisions(precision):
    pb = _pb()
    imgs = _items(64, 96, 5, seed=11)
    tgt = _target(pb, 4)
    exact, _, _ = _run(pb, imgs, pb.SamplePlan(), tgt, "exact")
    out, errors, _ = _run(pb, imgs, pb.SamplePlan(), tgt, precision)
    assert all(e is None for e in errors)
    if precision == "strict":
        assert np.array_equal(out, exact)
    else:
        d = np.abs(out.astype(np.int16) - exact.astype(np.int16))
        assert d.max() <= 1 and (d > 0).mean() <= 1e-3


def test_batch_degenerate_target_reports_every_item():
    pb = _pb()
    imgs = _items(64, 64, 4, seed=2)
    tgt = _target(pb)
    tgt = pb.FitParams(i0=tgt.i0, basis=tgt.basis,
                       stats=pb.StainStats(p99=np.array([tgt.stats.p99[0], 0.0])))
    _, errors, _ = _run(pb, imgs, pb.SamplePlan(), tgt)
    assert all(isinstance(e, pb.DegenerateStainError) for e in errors)


def test_batch_many_items_one_launch_per_148():
    """A batch larger than one launch (148 items) keeps item order and results."""
    pb = _pb()
    base = _items(48, 64, 4, seed=9)
    imgs = [base[k % 4] for k in range(300)]
    tgt = _target(pb, 8)
    out, errors, _ = _run(pb, imgs, pb.SamplePlan(), tgt)
    assert all(e is None for e in errors)
    for k in range(300):
        assert np.array_equal(out[k], out[k % 4]), k
    _, ref = _oracle_item(base[1], orc.Plan(), tgt)
    assert np.array_equal(out[1], ref)


def test_normalize_batch_host_matches_device_batch():
    import torch

    pb = _pb()
    imgs = _items(64, 80, 11, seed=13)
    tgt = _target(pb, 5)
    dev_out, dev_err, _ = _run(pb, imgs, pb.SamplePlan(), tgt)
    host = torch.from_numpy(np.stack(imgs)).pin_memory()
    with __import__("warnings").catch_warnings():
        __import__("warnings").simplefilter("ignore")
        out, errs = pb.normalize_batch_host(host, tgt, chunk=4, streams=3)
    assert np.array_equal(out.numpy(), dev_out)
    assert [type(e) for e in errs] == [type(e) for e in dev_err]


def test_table_percentiles_equal_per_sample_percentiles():
    """Coding each distinct colour once and selecting with weights gives the
    same densities and p99 as coding every sample (exact)."""
    import torch

    pb = _pb()
    from paper_1901_03088_b200 import batch, snmf, stats as dstats

    imgs = _items(96, 128, 7, seed=21)
    imgs[2] = np.full((96, 128, 3), 255, np.uint8)             # blank item (no samples)
    x = torch.from_numpy(np.stack(imgs)).cuda()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fits = pb.fit_batch(x, pb.SamplePlan())
    # rebuild the sample arrays the way fit_batch does and compare both paths
    n = len(imgs)
    flat = []
    offs = [0]
    for i in range(n):
        px = imgs[i].reshape(-1, 3)
        nw = px[~np.all(px > 220, axis=1)][:100_000]
        flat.append(nw)
        offs.append(offs[-1] + len(nw))
    samples = torch.from_numpy(np.concatenate(flat).reshape(-1)).cuda()
    d_off = torch.tensor(offs, dtype=torch.int64, device="cuda")
    total = offs[-1]
    r = snmf.snmf_batched(samples, d_off, fits.luts, pb.SnmfConfig(), cluster=1)
    assert r.table is not None
    h_s = snmf.code_samples(samples, d_off, fits.luts, r.basis, 0.0, max(np.diff(offs)))
    p_s, a_s = dstats.segment_percentiles(h_s, d_off, 99.0)
    h_t = snmf.code_table(r.table, d_off, fits.luts, r.basis, 0.0, max(np.diff(offs)), total)
    p_t, a_t = snmf.percentile_table(h_t, r.table, d_off, total, 99.0)
    assert np.array_equal(p_s.cpu().numpy(), p_t.cpu().numpy())
    assert np.array_equal(a_s.cpu().numpy(), a_t.cpu().numpy())
    assert np.array_equal(fits.p99.cpu().numpy(), p_t.cpu().numpy())


def test_speculative_tail_hit_and_miss_equal_the_cold_path():
    """One-patch batches enqueue the SNMF/p99 tail behind the compaction with
    memoised OD rows looked up on the device once the previous batch's i0
    values were all memoised; a batch with a new i0 value re-runs the tail
    with the exact rows.  Both give what a cold thread (empty memo) gives."""
    import threading

    import torch

    pb = _pb()
    from paper_1901_03088_b200 import batch as bt

    a = torch.from_numpy(np.stack(_items(96, 128, 6, seed=3))).cuda()
    b = torch.from_numpy(np.stack(_items(96, 128, 6, seed=4))).cuda()

    def fit(x):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            f = pb.fit_batch(x)
        return [f.params(i) for i in range(x.shape[0])], f.status.copy()

    def cold(x, box):
        box.append(fit(x))

    ref = {}
    for name, x in (("a", a), ("b", b)):
        box = []
        th = threading.Thread(target=cold, args=(x, box))
        th.start()
        th.join()
        ref[name] = box[0]

    def same(got, want):
        (pg, sg), (pw, sw) = got, want
        assert np.array_equal(sg, sw)
        for fg, fw in zip(pg, pw):
            assert np.array_equal(fg.i0, fw.i0)
            assert np.array_equal(fg.basis, fw.basis)
            assert np.array_equal(fg.stats.p99, fw.stats.p99)
            assert fg.stats.sample_count == fw.stats.sample_count

    fit(a)
    fit(a)                                     # memo now holds every value of a
    assert bt._od_rows_device(a.device) is not None
    same(fit(a), ref["a"])                     # speculative, all rows memoised
    assert bt._od_rows_device(a.device) is not None
    same(fit(b), ref["b"])                     # speculative, new values: re-run
    if bt._od_rows_device(a.device) is None:   # (b had a value a did not)
        same(fit(b), ref["b"])                 # cold, then speculative again
        same(fit(b), ref["b"])
