"""CPU checks of the drop-in boundary: libspcn.so builds, loads without a GPU,
and exports exactly the entry points include/spcn.h declares; host-side
logic of the package (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "spcn.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(spcn_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_1901_03088_b200 import _build, _lib

    _build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _header_functions()
    assert declared, "no functions parsed from include/spcn.h"
    missing = [f for f in declared if not hasattr(lib, f)]
    assert not missing, f"libspcn.so lacks {missing}"
    assert sorted(_lib.EXPORTS) == declared


def test_version_and_error_string_without_gpu():
    from paper_1901_03088_b200 import _lib

    L = _lib.lib()
    assert L.spcn_version().startswith(b"spcn-b200")
    assert L.spcn_last_error() == b""


def test_argument_validation_runs_on_host():
    """Invalid parameters are rejected before any CUDA call (no GPU needed)."""
    from paper_1901_03088_b200 import _lib

    L = _lib.lib()
    p = _lib.XformParams()
    p.src_i0[:] = [255.0] * 3
    p.tgt_i0[:] = [255.0] * 3
    p.src_basis[:] = [1.0, 0.0, 0.0, 1.0, 0.0, 0.0]
    p.tgt_basis[:] = [1.0, 0.0, 0.0, 1.0, 0.0, 0.0]
    p.factors[:] = [1.0, 1.0]
    p.precision = 0
    p.max_sweeps = 2000
    buf = ctypes.create_string_buffer(64)
    addr = ctypes.addressof(buf)
    assert L.spcn_xform_rgb8(addr, addr, 0, ctypes.byref(p), None, 0, None) == _lib.SPCN_OK
    p.src_basis[0] = -1.0
    assert L.spcn_xform_rgb8(addr, addr, 4, ctypes.byref(p), None, 0, None) == _lib.SPCN_EINVAL
    assert b"non-negative" in L.spcn_last_error()
    p.src_basis[0] = 1.0
    p.factors[0] = 0.0
    assert L.spcn_xform_rgb8(addr, addr, 4, ctypes.byref(p), None, 0, None) == _lib.SPCN_EINVAL
    p.factors[0] = 1.0
    p.src_i0[1] = 0.5
    assert L.spcn_xform_rgb8(addr, addr, 4, ctypes.byref(p), None, 0, None) == _lib.SPCN_EINVAL
    assert b"i0" in L.spcn_last_error()


def test_error_codes_map_to_reference_exceptions():
    from paper_1901_03088_b200 import _lib, errors

    with pytest.raises(errors.BlankSlideError):
        _lib.check(_lib.SPCN_EBLANK)
    with pytest.raises(errors.DegenerateStainError):
        _lib.check(_lib.SPCN_EDEGENERATE)
    with pytest.raises(ValueError):
        _lib.check(_lib.SPCN_EINVAL)


def test_host_helpers_match_oracle():
    from oracle import spcn_oracle as orc
    from paper_1901_03088_b200 import optics, order_stats, stain_sep

    rng = np.random.default_rng(3)
    for i0 in ([255.0] * 3, [250.0, 243.0, 230.0], [251.0, 244.5, 230.0 + 1 / 3]):
        assert np.array_equal(optics.od_table(i0), orc.od_table(i0))
    for _ in range(50):
        pool = rng.integers(221, 256, size=int(rng.integers(1, 400)))
        c = np.bincount(pool, minlength=256)
        assert order_stats.percentile_from_counts(c, 80.0) == orc.pct(pool, 80.0)
    assert np.array_equal(stain_sep.reference_basis(), orc.he_basis())
    w = orc.he_basis()
    assert np.array_equal(stain_sep.order_stains(w[:, ::-1].copy())[0], orc.order_cols(w)[0])


def test_profile_round_trip(tmp_path):
    import importlib

    nz = importlib.import_module("paper_1901_03088_b200.normalize")
    from paper_1901_03088_b200.stain_sep import reference_basis

    p = nz.FitParams(i0=np.array([251.0, 244.5, 230.0 + 1 / 3]), basis=reference_basis(),
                     stats=nz.StainStats(np.array([1.9705, 1.0308]), sample_count=100_000),
                     provenance={"source": "s.tiff", "config_hash": nz.config_hash({"a": 1})})
    path = tmp_path / "t.profile"
    nz.save_profile(path, p)
    back = nz.load_profile(path)
    assert np.array_equal(back.i0, p.i0) and np.array_equal(back.basis, p.basis)
    assert np.array_equal(back.stats.p99, p.stats.p99)
    assert back.provenance == p.provenance


def test_profile_files_byte_compatible_with_reference(tmp_path):
    """A profile written by the reference's save_profile (fixture made by
    oracle/make_golden.py) loads, and is written back byte for byte."""
    import importlib

    from conftest import GOLDEN as GOLDEN_DIR

    nz = importlib.import_module("paper_1901_03088_b200.normalize")

    ref_path = os.path.join(GOLDEN_DIR, "profile_ref.txt")
    p = nz.load_profile(ref_path)
    assert p.stats.sample_count == 1234 and p.provenance["source"] == "slide_7.tif"
    assert p.i0.tolist() == [250.0, 244.0, 251.5]
    out = tmp_path / "ours.txt"
    nz.save_profile(out, p)
    assert out.read_bytes() == open(ref_path, "rb").read()


@pytest.mark.gpu
def test_integration_binding_in_the_reference_transform_loop(monkeypatch):
    """the reference's transform loop (restated by the
    oracle: strips through a bounded worker pool, in-order commit) with its
    per-strip unit swapped for the ctypes binding gives the same bytes."""
    import integration_binding as ib
    from oracle import spcn_oracle as orc

    px, _, _ = orc.render(700, 530, 21, tissue_fraction=0.6)
    tg, _, _ = orc.render(400, 400, 22, tissue_fraction=0.6, i0=(250, 243, 230))
    src, tgt = orc.fit_params(px), orc.fit_params(tg)
    ref = orc.run_transform(px, src, tgt, strip_height=128, workers=3)
    table = orc.od_table(src["i0"])

    def gpu_strip(strip, s, t, f, code_lam=0.0):
        return ib.process_strip_gpu(strip, s["i0"], s["basis"], code_lam, f, t["basis"],
                                    t["i0"], table)

    monkeypatch.setattr(orc, "recolor_strip", gpu_strip)
    got = orc.run_transform(px, src, tgt, strip_height=128, workers=3)
    assert np.array_equal(got, ref)
