"""Pin the NumPy oracle to the reference (CPU only).

Two anchors: (1) golden fixtures produced by running the reference itself
(``oracle/make_golden.py``), (2) the reference test-suite's own known-answer
values (cited per test).  When /root/reference is importable (this
container) a few cases are also checked against it live.
"""
import math

import numpy as np
import pytest

from conftest import golden
from oracle import refimport
from oracle import spcn_oracle as orc


# ---------------------------------------------------------------- known answers
def test_percentile_known_answers():
    # tests/test_order_stats.py:10-12, tests/test_optics.py:25-29
    assert orc.pct([230, 235, 240, 245, 250], 80.0) == 246.0
    assert orc.pct([255] * 9, 80.0) == 255.0
    assert orc.pct([7.0], 99.0) == 7.0
    # tests/test_normalize.py:23-28
    d = np.arange(0.0, 101.0)
    assert list(orc.p99_pooled(np.stack([d, d]))) == [99.0, 99.0]


def test_median_known_answers():
    # tests/test_normalize.py:35-41
    assert list(orc.p99_patchwise([(1.0, 1.0), (2.0, 2.0), (3.0, 3.0)])) == [2.0, 2.0]
    assert list(orc.p99_patchwise([(1.0, 0.5), (2.0, 1.5), (3.0, 2.5), (10.0, 9.5)])) == [2.5, 2.0]


def test_beer_lambert_known_answers():
    # tests/test_optics.py:63-80
    assert np.all(orc.od_of(np.full((4, 4, 3), 200, np.uint8), [200.0] * 3) == 0.0)
    od = orc.od_of(np.array([[[25, 25, 25]]], np.uint8), [255.0] * 3)
    assert od[0, 0, 0] == pytest.approx(math.log(255 / 25), abs=1e-12)
    assert od[0, 0, 0] == pytest.approx(2.32239, abs=1e-5)
    od = orc.od_of(np.zeros((1, 1, 3), np.uint8), [255.0] * 3)
    assert od[0, 0, 0] == pytest.approx(5.54126, abs=1e-5)
    assert np.all(orc.od_of(np.full((1, 1, 3), 255, np.uint8), [240.0] * 3) == 0.0)
    with pytest.raises(ValueError):
        orc.od_of(np.zeros((1, 1, 3), np.uint8), [0.5, 255, 255])


def test_inverse_known_answers():
    # tests/test_optics.py:98-125
    out = orc.rgb_of(np.zeros((2, 2, 3)), [250.0, 245.0, 230.0])
    assert np.all(out == np.array([250, 245, 230], np.uint8))
    assert orc.rgb_of(np.full((1, 1, 3), 5.54126), [255.0] * 3)[0, 0, 0] == 1
    assert np.all(orc.rgb_of(np.full((1, 1, 3), 50.0), [255.0] * 3) == 0)
    for i0 in (np.array([255.0] * 3), np.array([240.0] * 3), np.array([250.0, 245.0, 230.0])):
        i = np.arange(1, 256, dtype=np.uint8)
        px = np.stack([i, i, i], axis=-1)[None]
        back = orc.rgb_of(orc.od_of(px, i0), i0)
        for c in range(3):
            top = int(i0[c])
            assert np.array_equal(back[0, :top, c], i[:top])
            assert np.all(back[0, top:, c] == top)


def test_coder_known_answers():
    # tests/test_stain_sep.py:78-97
    w = orc.he_basis()
    v = (2.0 * w[:, 0])[:, None]
    np.testing.assert_allclose(orc.densities(v, w, 0.0)[:, 0], [2.0, 0.0], atol=1e-8)
    assert np.array_equal(orc.densities(np.zeros((3, 5)), w, 0.0), np.zeros((2, 5)))
    h = orc.densities(v, w, 0.1)
    g00 = w[:, 0] @ w[:, 0]
    assert h[0, 0] == pytest.approx((2.0 * g00 - 0.1) / g00, abs=1e-12)
    assert h[1, 0] == 0.0


def test_normalize_block_known_answers():
    # tests/test_normalize.py:93-104
    out = orc.recolor(np.zeros((2, 6)), [1.0, 1.0], orc.he_basis(), [250.0, 245.0, 230.0], (2, 3))
    assert np.all(out == np.array([250, 245, 230], np.uint8))
    w = orc.he_basis()
    out = orc.recolor(np.array([[1.0], [0.0]]), [2.0, 1.0], w, [255.0] * 3, (1, 1))
    for c in range(3):
        assert out[0, 0, c] == round(255.0 * math.exp(-2.0 * w[c, 0]))


def test_order_and_objective_known_answers():
    # tests/test_stain_sep.py:29-37, 211-215
    w = orc.he_basis()
    for cand in (w, w[:, ::-1].copy()):
        np.testing.assert_allclose(orc.order_cols(cand)[0], w, atol=1e-12)
    h = np.array([[1.0, 0.0], [0.5, 2.0]])
    assert orc.objective(w @ h, w, h, 0.1) == pytest.approx(0.35, abs=1e-12)


# ---------------------------------------------------------------- golden fixtures
def test_od_tables_match_golden():
    g = golden("optics")
    for i0, table in zip(g["i0_cases"], g["od_tables"]):
        assert np.array_equal(orc.od_table(i0), table)
    for i0, out in zip(g["i0_cases"], g["inv_out"]):
        assert np.array_equal(orc.rgb_of(g["inv_od"], i0), out)
    pools = [g["pool0"], g["pool1"], g["pool2"]]
    assert np.array_equal(orc.bg_intensity(pools), g["pool_i0"])


def test_coder_matches_golden_bitwise():
    g = golden("coder")
    for w, lam, v, h in zip(g["bases"], g["lams"], g["ods"], g["hs"]):
        assert np.array_equal(orc.densities(v, w, float(lam)), h)


def test_percentiles_match_golden():
    g = golden("pct")
    for a, (n, p), val in zip(g["arrays"], g["np_"], g["vals"]):
        assert orc.pct(a[: int(n)], p) == val


def test_snmf_matches_golden():
    g = golden("snmf")
    for m, lam, seed, iters, conv in g["cases"]:
        i = int(seed)
        basis, hist, done, it, _ = orc.snmf(g[f"v{i}"], lam=lam, seed=i)
        # same machine + same NumPy/BLAS calls -> identical; across machines
        # BLAS summation order may differ in the last bits
        np.testing.assert_allclose(basis, g[f"basis{i}"], rtol=0, atol=1e-9)
        assert it == int(iters) and done == bool(conv)
        np.testing.assert_allclose(hist, g[f"hist{i}"], rtol=1e-9)


def test_slide_fits_and_transforms_match_golden():
    g = golden("slides")
    from oracle.make_golden import PAIRS, SLIDES  # noqa: F401  (cfg table only)

    fits = {}
    for name in g["names"]:
        name = str(name)
        cfg = g[f"{name}/cfg"]
        plan = orc.Plan(max_patches=int(cfg[0]), patch_size=int(cfg[1]),
                        target_pixels=int(cfg[2]), background_fraction_cutoff=cfg[3],
                        seed=int(cfg[4]), white_threshold=int(cfg[5]), sample_cap=int(cfg[6]))
        r = orc.fit_params(g[f"{name}/pixels"], plan, lam=cfg[7], seed=int(cfg[8]),
                           code_lam=cfg[9], per_patch=bool(cfg[10]))
        s = r["sample"]
        assert np.array_equal(s["non_white"], g[f"{name}/non_white"])
        assert list(s["counts"]) == list(g[f"{name}/sample_counts"])
        assert [s["visited"], s["used"]] == list(g[f"{name}/visited_used"])
        hist = np.stack([np.bincount(b, minlength=256) for b in s["bright"]])
        assert np.array_equal(hist, g[f"{name}/bright_hist"])
        assert np.array_equal(r["i0"], g[f"{name}/i0"])
        np.testing.assert_allclose(r["basis"], g[f"{name}/basis"], atol=1e-12)
        np.testing.assert_allclose(r["p99"], g[f"{name}/p99"], rtol=1e-12)
        fits[name] = dict(i0=g[f"{name}/i0"], basis=g[f"{name}/basis"], p99=g[f"{name}/p99"],
                          code_lam=float(cfg[9]))
    for a, b, sh in PAIRS:
        out = orc.run_transform(g[f"{a}/pixels"], fits[a], fits[b], strip_height=sh,
                                workers=2, code_lam=fits[a]["code_lam"])
        assert np.array_equal(out, g[f"xform/{a}->{b}"])


def test_synthetic_generator_matches_reference_c1_inputs():
    import hashlib

    g = golden("c1")
    px, _, _ = orc.render(2048, 2048, 1, tissue_fraction=0.6)
    assert hashlib.sha256(px.tobytes()).hexdigest() == str(g["c1/sha_src"])


@pytest.mark.skipif(not refimport.available(), reason="reference not mounted")
def test_oracle_matches_live_reference_on_random_strips():
    sn = refimport.load()
    from slidenorm import pipeline

    rng = np.random.default_rng(77)
    px = rng.integers(0, 256, size=(70, 50, 3)).astype(np.uint8)
    w = orc.he_basis()
    f = np.array([1.3, 0.8])
    ref = pipeline._process_strip(px, np.array([250.0, 243.0, 230.0]), w, 0.0, f, w,
                                  np.array([255.0, 255.0, 255.0]))
    mine = orc.recolor_strip(px, dict(i0=np.array([250.0, 243.0, 230.0]), basis=w),
                             dict(i0=np.array([255.0] * 3), basis=w), f)
    assert np.array_equal(ref, mine)
    assert sn.__version__ == "0.1.0"
