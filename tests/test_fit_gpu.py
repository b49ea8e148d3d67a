"""GPU parity of the fit path (sampling, i0, SNMF, coding, p99) vs the reference.

Integer/byte results (sample selection, bright pools, i0) must be bit-exact;
the SNMF basis is compared with the north_star tolerance (cosine 1e-3, and in
practice ~1e-12); p99 given identical densities is exact.
"""
import math
import warnings

import numpy as np
import pytest

from conftest import golden
from oracle import spcn_oracle as orc

pytestmark = pytest.mark.gpu


def _pb():
    import paper_1901_03088_b200 as pb

    return pb


def _plan(pb, cfg):
    return pb.SamplePlan(max_patches=int(cfg[0]), patch_size=int(cfg[1]),
                         target_pixels=int(cfg[2]), background_fraction_cutoff=float(cfg[3]),
                         seed=int(cfg[4]), white_threshold=int(cfg[5]), sample_cap=int(cfg[6]))


def _cos(a, b):
    return float(np.dot(a, b) / (np.linalg.norm(a) * np.linalg.norm(b)))


@pytest.mark.parametrize("device_slide", [False, True])
def test_sampling_bit_exact_vs_reference(device_slide):
    import torch

    pb = _pb()
    g = golden("slides")
    for name in g["names"]:
        name = str(name)
        px = g[f"{name}/pixels"]
        src = pb.DeviceSource(torch.from_numpy(px).cuda()) if device_slide else pb.ArraySource(px)
        s = pb.sample_pixels(src, _plan(pb, g[f"{name}/cfg"]))
        assert np.array_equal(s.non_white, g[f"{name}/non_white"]), name
        assert list(s.patch_counts) == list(g[f"{name}/sample_counts"]), name
        assert [s.patches_visited, s.patches_used] == list(g[f"{name}/visited_used"]), name
        assert np.array_equal(s.bright_hist, g[f"{name}/bright_hist"]), name


def test_fit_matches_reference_fits():
    pb = _pb()
    g = golden("slides")
    for name in g["names"]:
        name = str(name)
        cfg = g[f"{name}/cfg"]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fp = pb.fit(pb.ArraySource(g[f"{name}/pixels"]), _plan(pb, cfg),
                        pb.SnmfConfig(lam=float(cfg[7]), seed=int(cfg[8])),
                        code_lam=float(cfg[9]), per_patch_stats=bool(cfg[10]))
        assert np.array_equal(fp.i0, g[f"{name}/i0"]), name
        for j in range(2):
            assert 1.0 - _cos(fp.basis[:, j], g[f"{name}/basis"][:, j]) <= 1e-3, name
        np.testing.assert_allclose(fp.basis, g[f"{name}/basis"], atol=1e-9, err_msg=name)
        np.testing.assert_allclose(fp.stats.p99, g[f"{name}/p99"], rtol=1e-9, err_msg=name)
        assert fp.stats.sample_count == int(g[f"{name}/count"]), name


def test_fit_basis_matches_reference_snmf():
    pb = _pb()
    g = golden("snmf")
    for m, lam, seed, iters, conv in g["cases"]:
        i = int(seed)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = pb.fit_basis(g[f"v{i}"], pb.SnmfConfig(lam=float(lam), seed=i))
        np.testing.assert_allclose(r.basis, g[f"basis{i}"], atol=1e-9)
        assert r.iterations == int(iters) and r.converged == bool(conv)
        np.testing.assert_allclose(r.objective, g[f"hist{i}"], rtol=1e-9)
        assert np.all(np.diff(r.objective) <= 1e-10)   # criterion 3


def test_fit_basis_recovers_reference_basis_and_warns():
    pb = _pb()
    wstar = orc.he_basis()
    rng = np.random.default_rng(20)
    v = wstar @ orc.sparse_pairs(10_000, rng)
    r = pb.fit_basis(v, pb.SnmfConfig(seed=0))
    for j in range(2):
        c = _cos(r.basis[:, j], wstar[:, j])
        assert math.degrees(math.acos(min(1.0, c))) < 5.0
    with pytest.raises(pb.InsufficientPixelsError):
        pb.fit_basis(np.ones((3, 9)))
    rng = np.random.default_rng(23)
    rank1 = wstar[:, :1] @ rng.uniform(0.2, 2.0, size=(1, 5_000))
    from paper_1901_03088_b200.stain_sep import StainDegeneracyWarning

    with pytest.warns(StainDegeneracyWarning):
        pb.fit_basis(rank1, pb.SnmfConfig(seed=3))
    with pytest.warns(StainDegeneracyWarning, match="unreliable"):
        pb.fit_basis(wstar @ orc.sparse_pairs(200, np.random.default_rng(26)), pb.SnmfConfig(seed=6))


def test_device_percentiles_exact():
    import torch

    pb = _pb()
    g = golden("pct")
    for a, (n, p), val in zip(g["arrays"], g["np_"], g["vals"]):
        t = torch.from_numpy(a[: int(n)].copy()).cuda()
        assert pb.percentile(t, float(p)) == val
    rng = np.random.default_rng(9)
    for _ in range(20):
        h = rng.gamma(2.0, 1.0, size=(2, int(rng.integers(5, 5000))))
        h[:, ::7] = 0.0
        st = pb.stain_stats(torch.from_numpy(h).cuda())
        assert st.p99[0] == orc.pct(h[0], 99.0) and st.p99[1] == orc.pct(h[1], 99.0)
    with pytest.raises(pb.StainAbsentError, match="eosin"):
        pb.stain_stats(torch.from_numpy(np.stack([np.ones(10), np.zeros(10)])).cuda())


def test_blank_slide_and_stage_labels():
    pb = _pb()
    white = pb.ArraySource(np.full((256, 256, 3), 255, np.uint8))
    with pytest.raises(pb.BlankSlideError):
        pb.sample_pixels(white, pb.SamplePlan(patch_size=64))
    with pytest.raises(pb.BlankSlideError, match="sampling"):
        pb.fit(pb.ArraySource(np.full((128, 128, 3), 255, np.uint8)), pb.SamplePlan(patch_size=64))


def test_sample_capped_at_target():
    pb = _pb()
    rng = np.random.default_rng(0)
    pixels = np.full((1100, 1100, 3), 255, np.uint8)
    region = rng.integers(40, 200, size=(1000, 1000, 3)).astype(np.uint8)
    keep_white = rng.random((1000, 1000)) > 0.6
    region[keep_white] = 255
    pixels[50:1050, 50:1050] = region
    s = pb.sample_pixels(pb.ArraySource(pixels), pb.SamplePlan(seed=1))
    ref = orc.gather_sample(pixels, orc.Plan(seed=1))
    assert s.non_white.shape[0] == 100_000
    assert np.array_equal(s.non_white, ref["non_white"])


def test_normalize_end_to_end_config1_small():
    """fit(src) + fit(tgt) + transform through the drop-in entry vs the reference."""
    pb = _pb()
    g = golden("slides")
    src, tgt = g["sparse320/pixels"], g["sparse320b/pixels"]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = pb.normalize(src, tgt)
    ref = g["xform/sparse320->sparse320b"]
    d = np.abs(out.astype(int) - ref.astype(int))
    assert d.max() <= 1
    assert np.mean(np.any(d > 0, axis=-1)) <= 1e-3


def test_transform_streamed_strip_and_worker_invariance():
    import torch

    pb = _pb()
    g = golden("slides")
    px = g["dense256/pixels"]
    fp = pb.FitParams(g["dense256/i0"], g["dense256/basis"], pb.StainStats(g["dense256/p99"]))
    ref = g["xform/dense256->dense256"]
    for sh, workers in ((64, 1), (100, 3), (256, 2), (1000, 2)):
        sink = pb.ArrayWriter(256, 256)
        pb.transform(pb.ArraySource(px), fp, fp, sink, strip_height=sh, workers=workers)
        sink.close()
        assert np.array_equal(sink.pixels, ref)
    pin = torch.from_numpy(px.copy()).pin_memory()
    outp = torch.empty_like(pin).pin_memory()
    sink = pb.ArrayWriter(256, 256, out=outp.numpy())
    gauge = pb.BufferGauge()
    pb.transform(pb.ArraySource(pin.numpy()), fp, fp, sink, strip_height=64, workers=2,
                 gauge=gauge)
    assert np.array_equal(outp.numpy(), ref)
    assert 0 < gauge.peak <= 2 * 64 * 256 and gauge.current == 0
    dsink = pb.DeviceWriter(256, 256)
    pb.transform(pb.DeviceSource(torch.from_numpy(px).cuda()), fp, fp, dsink)
    assert np.array_equal(dsink.pixels.cpu().numpy(), ref)


def test_transform_degenerate_and_progress():
    pb = _pb()
    g = golden("slides")
    px = g["dense256/pixels"]
    fp = pb.FitParams(g["dense256/i0"], g["dense256/basis"], pb.StainStats(g["dense256/p99"]))
    broken = pb.FitParams(fp.i0, fp.basis, pb.StainStats(np.array([0.0, 1.0])))
    with pytest.raises(pb.DegenerateStainError):
        pb.transform(pb.ArraySource(px), broken, fp, pb.ArrayWriter(256, 256))
    seen = []
    pb.transform(pb.ArraySource(px), fp, fp, pb.ArrayWriter(256, 256), strip_height=100,
                 progress=lambda d, t: seen.append((d, t)))
    assert seen == [(100, 256), (200, 256), (256, 256)]


@pytest.mark.parametrize("thr", [0, 60, 127, 128, 200, 254, 255])
def test_sampling_white_thresholds_and_take_limits(thr):
    """The byte-parallel flags of the count/compaction kernels on both sides
    of thr = 128 (two SWAR forms) and at the ends of the range, on an odd
    slide whose 100-px patches give unaligned rows and short tails, with a
    small target and bright cap so pools fill inside chunks: the sample, the
    visit counts and the bright pools equal the oracle's."""
    import torch

    pb = _pb()
    px, _, _ = orc.render(517, 333, 21, tissue_fraction=0.5, i0=(250, 238, 226))
    oplan = orc.Plan(max_patches=20, patch_size=100, target_pixels=7000,
                     background_fraction_cutoff=0.95, seed=5, white_threshold=thr,
                     sample_cap=3000)
    plan = pb.SamplePlan(max_patches=20, patch_size=100, target_pixels=7000,
                         background_fraction_cutoff=0.95, seed=5, white_threshold=thr,
                         sample_cap=3000)
    try:
        ref = orc.gather_sample(px, oplan)
    except orc.OracleError:
        ref = None
    for src in (pb.ArraySource(px), pb.DeviceSource(torch.from_numpy(px).cuda())):
        if ref is None:
            with pytest.raises(Exception):
                pb.sample_pixels(src, plan)
            continue
        s = pb.sample_pixels(src, plan)
        assert np.array_equal(s.non_white, ref["non_white"]), thr
        assert list(s.patch_counts) == list(ref["counts"]), thr
        assert [s.patches_visited, s.patches_used] == [ref["visited"], ref["used"]], thr
        want = np.stack([np.bincount(ref["bright"][c], minlength=256) for c in range(3)])
        assert np.array_equal(np.asarray(s.bright_hist).reshape(3, 256), want), thr


@pytest.mark.parametrize("thr", [100, 220])
def test_batch_sampling_many_items_take_limits(thr):
    """1024 items of 96 x 96 (three chunks each: the many-patch compaction
    with several chunks per CTA) with a target and bright cap that end inside
    the chunks: per-item sample sizes and i0 equal the oracle's."""
    import torch

    pb = _pb()
    n = 1024
    imgs = np.stack([orc.render(96, 96, 300 + (k % 16), tissue_fraction=0.3 + 0.04 * (k % 16),
                                i0=(252, 240, 231))[0] for k in range(n)])
    plan = pb.SamplePlan(target_pixels=5000, white_threshold=thr, sample_cap=2500)
    oplan = orc.Plan(target_pixels=5000, white_threshold=thr, sample_cap=2500)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fits = pb.fit_batch(torch.from_numpy(imgs).cuda(), plan)
    i0 = fits.i0.cpu().numpy()
    for k in (0, 1, 7, 15, 500, 1023):
        ref = orc.gather_sample(imgs[k], oplan)
        assert int(fits.count[k]) == ref["non_white"].shape[0], k
        assert np.array_equal(i0[k], orc.bg_intensity(ref["bright"])), k
