"""Whole-slide ("global") p99 mode on the GPU.

Oracle: the reference's percentile (src/order_stats.py:11-36) over the
reference-order fp64 densities (code_densities, src/stain_sep.py:168-201) of
every non-white pixel (src/pipeline.py:176).  The result must be identical.
"""
import numpy as np
import pytest

from oracle import spcn_oracle as orc

pytestmark = pytest.mark.gpu


def _oracle_global(px, i0, basis, code_lam=0.0, thr=220):
    flat = px.reshape(-1, 3)
    nw = ~np.all(flat > thr, axis=1)
    v = np.ascontiguousarray(orc.od_of(flat[nw], i0).T)
    h = orc.densities(v, basis, code_lam)
    return np.array([orc.pct(h[0], 99.0), orc.pct(h[1], 99.0)]), int(nw.sum())


@pytest.mark.parametrize("seed,i0,code_lam,layout", [
    (3, (255, 255, 255), 0.0, "scatter"),
    (4, (250, 243, 230), 0.0, "block"),
    (5, (252, 249, 246), 0.05, "scatter"),
])
def test_global_p99_matches_reference(seed, i0, code_lam, layout):
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200.global_stats import global_p99
    from paper_1901_03088_b200.pipeline import slide_chunks

    px, _, _ = orc.render(700, 520, seed, i0=i0, tissue_fraction=0.55, layout=layout)
    fitp = orc.fit_params(px)
    ref, n = _oracle_global(px, fitp["i0"], fitp["basis"], code_lam)
    src = pb.DeviceSource(torch.from_numpy(px).cuda())
    p99, nw, info = global_p99(slide_chunks(src), fitp["i0"], fitp["basis"], code_lam)
    assert nw == n
    assert np.array_equal(p99, ref), (p99, ref, info)
    assert info["fp64_evaluations"] < 0.25 * n          # only the window is recomputed


@pytest.mark.parametrize("thr,i0", [
    (220, (255, 255, 255)),   # white test on the OD values
    (0, (255, 255, 255)),     # threshold 0: byte test (OD(0) == OD(1))
    (248, (250, 243, 230)),   # threshold >= an i0 component: byte test
    (255, (252, 249, 246)),   # nothing is white
])
def test_global_p99_white_thresholds_and_tail(thr, i0):
    """Odd pixel count (a < 16-px tail after the TMA-streamed body) and
    every branch of the white test."""
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200.global_stats import global_p99
    from paper_1901_03088_b200.pipeline import slide_chunks

    px, _, _ = orc.render(701, 523, 7, i0=i0, tissue_fraction=0.5)
    fitp = orc.fit_params(px)
    src = pb.DeviceSource(torch.from_numpy(px).cuda())
    if thr == 0 and px.min(axis=2).min() > 0:        # every pixel is white
        with pytest.raises(pb.StainAbsentError):
            global_p99(slide_chunks(src), fitp["i0"], fitp["basis"], 0.0, thr)
        return
    ref, n = _oracle_global(px, fitp["i0"], fitp["basis"], 0.0, thr)
    p99, nw, info = global_p99(slide_chunks(src), fitp["i0"], fitp["basis"], 0.0, thr)
    assert nw == n
    assert np.array_equal(p99, ref), (p99, ref, info)
    # one-pass colour-table mode (bracket around the answer)
    br = np.stack([ref * 0.8, ref * 1.2], axis=1)
    p99, nw, info = global_p99(slide_chunks(src), fitp["i0"], fitp["basis"], 0.0, thr, guess=br)
    assert nw == n and info.get("mode") == "table", info
    assert np.array_equal(p99, ref), (p99, ref, info)


def test_global_p99_sample_bracket_two_passes():
    """Seeded with the bracket of the sampled densities, the search is one
    pass (colour table), and a wrong bracket still gives the exact answer."""
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import synthetic
    from paper_1901_03088_b200.global_stats import global_p99, sample_bracket
    from paper_1901_03088_b200.pipeline import slide_chunks

    dev = synthetic.render_slide(2048, 1536, 5, tissue_fraction=0.6)
    px = dev.cpu().numpy()
    basis, i0 = orc.he_basis(), np.array([255.0, 255.0, 255.0])
    ref, n = _oracle_global(px, i0, basis)
    flat = px.reshape(-1, 3)
    nw = ~np.all(flat > 220, axis=1)
    sub = flat[nw][::97]
    h = orc.densities(np.ascontiguousarray(orc.od_of(sub, i0).T), basis, 0.0)
    br = sample_bracket(torch.from_numpy(np.ascontiguousarray(h)).cuda())
    assert br.shape == (2, 2) and (br[:, 0] <= ref).all() and (ref <= br[:, 1]).all()
    p99, nw_, info = global_p99(slide_chunks(pb.DeviceSource(dev)), i0, basis, guess=br)
    assert nw_ == n and np.array_equal(p99, ref), (p99, ref, info)
    assert info["passes"] == 1 and info["mode"] == "table", info
    wrong = np.array([[5.0, 6.0], [5.0, 6.0]])
    p99, _, info = global_p99(slide_chunks(pb.DeviceSource(dev)), i0, basis, guess=wrong)
    assert np.array_equal(p99, ref) and info["passes"] >= 3, info


def test_fit_global_mode_host_and_device_slides():
    import torch

    import paper_1901_03088_b200 as pb

    px, _, _ = orc.render(1100, 900, 11, i0=(248, 246, 250), tissue_fraction=0.6)
    for src in (pb.ArraySource(px), pb.DeviceSource(torch.from_numpy(px).cuda())):
        fp = pb.fit(src, p99_mode="global")
        ref, n = _oracle_global(px, fp.i0, fp.basis)
        assert np.array_equal(fp.stats.p99, ref)
        assert fp.stats.sample_count == n
    with pytest.raises(ValueError):
        pb.fit(pb.ArraySource(px), p99_mode="everything")


def test_global_p99_large_slide_window_logic():
    """4 Mpx GPU-rendered slide: the fine window must hold both ranks."""
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import synthetic
    from paper_1901_03088_b200.global_stats import global_p99
    from paper_1901_03088_b200.pipeline import slide_chunks

    dev = synthetic.render_slide(2048, 2048, 21, tissue_fraction=0.6)
    px = dev.cpu().numpy()
    basis = orc.he_basis()
    i0 = np.array([255.0, 255.0, 255.0])
    ref, n = _oracle_global(px, i0, basis)
    p99, nw, info = global_p99(slide_chunks(pb.DeviceSource(dev)), i0, basis)
    assert nw == n and np.array_equal(p99, ref), (p99, ref, info)
    assert max(info["candidates"]) < 1 << 23


def test_sample_bracket_selects_exact_order_statistics():
    """sample_bracket = the exact order statistics at bracket_ranks (libspcn
    k-th selection, no sort), and None for an empty sample."""
    import torch

    from paper_1901_03088_b200.global_stats import bracket_ranks, sample_bracket

    rng = np.random.default_rng(5)
    for m in (1, 7, 1000, 100_000):
        h = np.stack([rng.gamma(2.0, 0.4, m), rng.gamma(1.5, 0.3, m)])
        br = sample_bracket(torch.from_numpy(h).cuda())
        lo, hi = bracket_ranks(m)
        for j in range(2):
            srt = np.sort(h[j])
            assert br[j, 0] == srt[lo] and br[j, 1] == srt[hi]
    assert sample_bracket(torch.zeros((2, 0), dtype=torch.float64, device="cuda")) is None
