"""Generate golden fixtures by running the REFERENCE itself (this container).

    python oracle/make_golden.py          # writes tests/golden/*.npz

Every array in ``tests/golden/`` comes from calling the reference package
(``/root/reference/pkg/src/slidenorm``, imported via ``oracle/refimport.py``)
on seeded inputs.  The fixtures pin the NumPy oracle (CPU tests) and the CUDA
path (GPU tests) without needing /root/reference at run time.
"""
from __future__ import annotations

import hashlib
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

from oracle import refimport  # noqa: E402

sn = refimport.load()
from slidenorm import optics, order_stats, pipeline, stain_sep, synthetic  # noqa: E402
from slidenorm.image_io import ArraySource, StripWriter  # noqa: E402


class _Mem(StripWriter):
    def __init__(self, w, h):
        super().__init__(w, h)
        self.pixels = np.zeros((h, w, 3), np.uint8)

    def _write(self, rows):
        y = self._rows_written
        self.pixels[y:y + rows.shape[0]] = rows

    def close(self):
        self._closed = True


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


I0_CASES = np.array([
    [255.0, 255.0, 255.0], [240.0, 240.0, 240.0], [250.0, 245.0, 230.0],
    [250.0, 243.0, 230.0], [251.0, 244.5, 230.0 + 1.0 / 3.0], [246.0, 240.0, 229.0],
    [1.0, 2.0, 3.5],
])


def optics_fixture():
    ramp = np.repeat(np.arange(256, dtype=np.uint8)[:, None], 3, axis=1)
    tables = np.stack([optics.beer_lambert(ramp, i0).T for i0 in I0_CASES])
    rng = np.random.default_rng(100)
    od = rng.uniform(0.0, 6.0, size=(64, 64, 3))
    od[0, :8] = 0.0
    inv = np.stack([optics.inverse_beer_lambert(od, i0) for i0 in I0_CASES])
    pools = [rng.integers(221, 256, size=n) for n in (17, 400, 3)]
    i0_pools = optics.estimate_max_intensity(pools)
    return dict(i0_cases=I0_CASES, od_tables=tables, inv_od=od, inv_out=inv,
                pool0=pools[0], pool1=pools[1], pool2=pools[2], pool_i0=i0_pools)


def random_basis(rng):
    while True:
        w = np.abs(rng.standard_normal((3, 2)))
        w /= np.linalg.norm(w, axis=0)
        if w[:, 0] @ w[:, 1] <= 0.995:
            return w


def coder_fixture():
    rng = np.random.default_rng(200)
    bases, lams, ods, hs = [], [], [], []
    cases = [(stain_sep.reference_basis(), 0.0), (stain_sep.reference_basis(), 0.1),
             (stain_sep.reference_basis(), 0.05)]
    for _ in range(5):
        cases.append((random_basis(rng), float(rng.choice([0.0, 0.05, 0.1, 0.5]))))
    for w, lam in cases:
        # OD values drawn the way pixels produce them: LUT values of random u8
        i0 = np.array([255.0, 250.0, 240.0])
        px = rng.integers(0, 256, size=(3000, 3)).astype(np.uint8)
        px[:50] = 255
        v = np.ascontiguousarray(optics.beer_lambert(px, i0).T)
        v = np.concatenate([v, rng.uniform(0, 3, size=(3, 1000))], axis=1)
        bases.append(w)
        lams.append(lam)
        ods.append(v)
        hs.append(stain_sep.code_densities(v, w, lam))
    return dict(bases=np.stack(bases), lams=np.array(lams), ods=np.stack(ods),
                hs=np.stack(hs))


def pct_fixture():
    rng = np.random.default_rng(300)
    arrays, ps, vals, meds = [], [], [], []
    for n in (1, 2, 5, 7, 100, 101, 999, 4096):
        a = rng.gamma(2.0, 1.0, size=n)
        for p in (0.0, 50.0, 80.0, 99.0, 100.0):
            arrays.append(np.pad(a, (0, 4096 - n), constant_values=np.nan))
            ps.append((n, p))
            vals.append(order_stats.percentile(a, p))
        meds.append(order_stats.median(a))
    return dict(arrays=np.stack(arrays), np_=np.array(ps), vals=np.array(vals),
                medians=np.array(meds))


def snmf_fixture():
    wstar = stain_sep.reference_basis()
    out = {}
    cases = []
    for i, (m, noisy, lam) in enumerate([(10_000, False, 0.1), (10_000, True, 0.1),
                                          (3_000, False, 0.0), (2_000, True, 0.1)]):
        rng = np.random.default_rng(1000 + i)
        v = wstar @ synthetic.sparse_densities(m, rng)
        if noisy:
            v = np.maximum(v * (1.0 + 0.01 * rng.standard_normal(v.shape)), 0.0)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = stain_sep.fit_basis(v, stain_sep.SnmfConfig(lam=lam, seed=i))
        out[f"v{i}"] = v
        out[f"basis{i}"] = res.basis
        out[f"hist{i}"] = np.array(res.objective)
        cases.append((m, lam, i, res.iterations, int(res.converged)))
    out["cases"] = np.array(cases, dtype=np.float64)
    return out


SLIDES = {
    # name: (render kwargs, plan kwargs, snmf kwargs, fit kwargs)
    "dense256": (dict(width=256, height=256, seed=42, tissue_fraction=0.6,
                      density_sampler=synthetic.dense_densities),
                 dict(patch_size=128, target_pixels=30_000, seed=3),
                 dict(lam=0.0, seed=1), dict(code_lam=0.0)),
    "tinted256": (dict(width=256, height=256, seed=3, i0=(250, 243, 230),
                       tissue_fraction=0.5, density_sampler=synthetic.dense_densities),
                  dict(patch_size=128, target_pixels=30_000, seed=3),
                  dict(lam=0.0, seed=2), dict(code_lam=0.0)),
    "target256": (dict(width=256, height=256, seed=9, tissue_fraction=0.6,
                       density_sampler=synthetic.dense_densities),
                  dict(patch_size=128, target_pixels=30_000, seed=3),
                  dict(lam=0.0, seed=3), dict(code_lam=0.0)),
    "sparse320": (dict(width=320, height=320, seed=11, tissue_fraction=0.6),
                  dict(), dict(), dict()),
    "sparse320b": (dict(width=320, height=320, seed=12, tissue_fraction=0.6),
                   dict(), dict(), dict()),
    "perpatch512": (dict(width=512, height=300, seed=42, tissue_fraction=0.6,
                         density_sampler=synthetic.dense_densities),
                    dict(patch_size=128, target_pixels=30_000, seed=3),
                    dict(lam=0.0, seed=1), dict(code_lam=0.0, per_patch_stats=True)),
    "codelam200": (dict(width=200, height=180, seed=5, tissue_fraction=0.7),
                   dict(patch_size=64, target_pixels=20_000, seed=4, max_patches=8),
                   dict(lam=0.1, seed=4), dict(code_lam=0.05)),
}

PAIRS = [("dense256", "dense256", 96), ("tinted256", "target256", 1024),
         ("sparse320", "sparse320b", 1024), ("codelam200", "sparse320b", 64)]


def slide_fixture():
    out = {}
    names = []
    for name, (rk, pk, sk, fk) in SLIDES.items():
        sl = synthetic.render_slide(**rk)
        plan = pipeline.SamplePlan(**pk)
        sample = pipeline.sample_pixels(ArraySource(sl.pixels), plan)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            fp = pipeline.fit(ArraySource(sl.pixels), plan, stain_sep.SnmfConfig(**sk), **fk)
        out[f"{name}/pixels"] = sl.pixels
        out[f"{name}/i0"] = fp.i0
        out[f"{name}/basis"] = fp.basis
        out[f"{name}/p99"] = fp.stats.p99
        out[f"{name}/count"] = np.array(fp.stats.sample_count)
        out[f"{name}/sample_counts"] = np.array(sample.patch_counts)
        out[f"{name}/visited_used"] = np.array([sample.patches_visited, sample.patches_used])
        out[f"{name}/bright_hist"] = np.stack(
            [np.bincount(b, minlength=256) for b in sample.bright])
        out[f"{name}/non_white"] = sample.non_white
        out[f"{name}/cfg"] = np.array([
            plan.max_patches, plan.patch_size, plan.target_pixels,
            plan.background_fraction_cutoff, plan.seed, plan.white_threshold,
            plan.sample_cap, sk.get("lam", 0.1), sk.get("seed", 0),
            fk.get("code_lam", 0.0), float(fk.get("per_patch_stats", False))])
        names.append(name)
    for a, b, sh in PAIRS:
        sl = out[f"{a}/pixels"]
        src = sn.FitParams(out[f"{a}/i0"], out[f"{a}/basis"], sn.StainStats(out[f"{a}/p99"]))
        tgt = sn.FitParams(out[f"{b}/i0"], out[f"{b}/basis"], sn.StainStats(out[f"{b}/p99"]))
        code_lam = float(out[f"{a}/cfg"][9])
        sink = _Mem(sl.shape[1], sl.shape[0])
        pipeline.transform(ArraySource(sl), src, tgt, sink, strip_height=sh, workers=2,
                           code_lam=code_lam)
        out[f"xform/{a}->{b}"] = sink.pixels
    out["names"] = np.array(names)
    return out


def c1_fixture():
    """Config 1: 2048^2 sparse tile vs 2048^2 target, defaults;
    plus the tinted-source variant.  Outputs are too large to commit, so the
    fixture keeps FitParams and SHA-256 digests of inputs and outputs."""
    out = {}
    runs = [("c1", dict(seed=1), dict(seed=2)),
            ("c1tint", dict(seed=1, i0=(250, 243, 230)), dict(seed=2))]
    for tag, sk, tk in runs:
        s = synthetic.render_slide(2048, 2048, tissue_fraction=0.6, **sk)
        t = synthetic.render_slide(2048, 2048, tissue_fraction=0.6, **tk)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            ps = pipeline.fit(ArraySource(s.pixels))
            pt = pipeline.fit(ArraySource(t.pixels))
        sink = _Mem(2048, 2048)
        pipeline.transform(ArraySource(s.pixels), ps, pt, sink, strip_height=1024, workers=8)
        for role, p in (("src", ps), ("tgt", pt)):
            out[f"{tag}/{role}_i0"] = p.i0
            out[f"{tag}/{role}_basis"] = p.basis
            out[f"{tag}/{role}_p99"] = p.stats.p99
        out[f"{tag}/sha_src"] = np.array(sha(s.pixels))
        out[f"{tag}/sha_tgt"] = np.array(sha(t.pixels))
        out[f"{tag}/sha_out"] = np.array(sha(sink.pixels))
        # a 64-row band of the output, for a direct byte comparison
        out[f"{tag}/band_out"] = sink.pixels[1000:1064]
    return out


def make_profile_fixture(out_dir):
    """A profile file written by the reference's own save_profile
    (src/normalize.py:160-190), for the byte-compatibility test."""
    import importlib

    import numpy as np

    rn = importlib.import_module("slidenorm.normalize")
    rs = importlib.import_module("slidenorm.stain_sep")
    w = rn.FitParams(i0=np.array([250., 244., 251.5]), basis=rs.reference_basis(),
                     stats=rn.StainStats(p99=np.array([1.2534567890123456, 0.5]),
                                         sample_count=1234),
                     provenance={"source": "slide_7.tif", "config_hash": "0f1e2d"})
    rn.save_profile(os.path.join(out_dir, "profile_ref.txt"), w)


PNG_SHAPE, PNG_STRIP, PNG_SEED = (37, 53), 10, 2024


def png_pixels():
    """The pixels of the PNG fixture (regenerated by the test)."""
    h, w = PNG_SHAPE
    return np.random.default_rng(PNG_SEED).integers(0, 256, size=(h, w, 3), dtype=np.uint8)


def make_png_fixture(out_dir):
    """A PNG written strip by strip by the reference's own streaming encoder
    (PngStripWriter, src/image_io.py:316-358), for the byte-level parity of
    ours and of our reader."""
    import importlib

    from slidenorm.image_io import PixelBlock

    rio = importlib.import_module("slidenorm.image_io")
    px = png_pixels()
    h, w = PNG_SHAPE
    wr = rio.PngStripWriter(os.path.join(out_dir, "png_ref_strips.png"), w, h)
    for y in range(0, h, PNG_STRIP):
        wr.write_strip(PixelBlock(0, y, px[y:y + PNG_STRIP]))
    wr.close()


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--png" in sys.argv:
        make_png_fixture(OUT)
        return
    for name, fn in [("optics", optics_fixture), ("coder", coder_fixture),
                     ("pct", pct_fixture), ("snmf", snmf_fixture),
                     ("slides", slide_fixture), ("c1", c1_fixture)]:
        data = fn()
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{path}: {os.path.getsize(path) / 1e6:.2f} MB")
    make_profile_fixture(OUT)
    make_png_fixture(OUT)


if __name__ == "__main__":
    main()

