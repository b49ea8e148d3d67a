"""GPU: the device-built recolouring (spcn_xform_rgb8_fitted) and the fused
normalize() of a resident slide (pipeline.fit_transform_resident).

The fused path must give the same bytes, FitParams, warnings and errors as
fit() + transform() with host-built parameters (src/cli.py:220-244), for any
alignment of the buffers, and must leave the output untouched whenever its
device-side checks decline a recolouring (the host path then raises or runs
the strict path).
"""
import ctypes
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pb():
    import paper_1901_03088_b200 as pb

    return pb


def _quiet(fn, *a, **k):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return fn(*a, **k)


@pytest.fixture(scope="module")
def slides():
    import torch

    from paper_1901_03088_b200 import synthetic

    torch.cuda.set_device(0)
    src = synthetic.render_slide(4096, 4096, 5, tissue_fraction=0.5)          # 2^24 px
    tgt = synthetic.render_slide(1024, 1024, 6, tissue_fraction=0.6, i0=(250, 243, 230))
    target = _quiet(_pb().fit, _pb().DeviceSource(tgt))
    return src, target


def _unfused(src, target, monkeypatch, **kw):
    monkeypatch.setenv("SPCN_FUSED", "0")
    out = _quiet(_pb().normalize, src, target, **kw)
    monkeypatch.delenv("SPCN_FUSED")
    return out


def test_fused_normalize_matches_fit_then_transform(slides, monkeypatch):
    import torch

    pb = _pb()
    src, target = slides
    ref = _unfused(src, target, monkeypatch)
    from paper_1901_03088_b200 import _lib

    L = _lib.lib()
    n0 = L.spcn_launch_count()
    out = torch.empty_like(src)
    got = _quiet(pb.normalize, src, target, out=out)
    assert got.data_ptr() == out.data_ptr()
    assert L.spcn_launch_count() > n0
    assert torch.equal(out, ref)
    # the returned fit equals pb.fit's
    stats = pb.RunStats()
    fp = _quiet(pb.pipeline.fit_transform_resident, pb.DeviceSource(src), target,
                torch.empty_like(src), stats=stats)
    fp_ref = _quiet(pb.fit, pb.DeviceSource(src))
    assert np.array_equal(fp.i0, fp_ref.i0)
    assert np.array_equal(fp.basis, fp_ref.basis)
    assert np.array_equal(fp.stats.p99, fp_ref.stats.p99)
    assert fp.provenance == fp_ref.provenance
    assert stats.transformed_pixels == src.shape[0] * src.shape[1]


def test_fused_repeated_and_two_streams(slides, monkeypatch):
    """Consecutive calls rotate the __constant__ parameter slots; two streams
    with different targets in flight at once must not see each other's."""
    import torch

    pb = _pb()
    src, target = slides
    from paper_1901_03088_b200 import synthetic

    tgt2_img = synthetic.render_slide(1024, 1024, 9, tissue_fraction=0.4)
    target2 = _quiet(pb.fit, pb.DeviceSource(tgt2_img))
    ref1 = _unfused(src, target, monkeypatch)
    ref2 = _unfused(src, target2, monkeypatch)
    outs = [torch.empty_like(src) for _ in range(5)]
    for k, o in enumerate(outs):
        _quiet(pb.normalize, src, target if k % 2 == 0 else target2, out=o)
    for k, o in enumerate(outs):
        assert torch.equal(o, ref1 if k % 2 == 0 else ref2), k
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2 = torch.empty_like(src), torch.empty_like(src)
    torch.cuda.synchronize()
    for _ in range(2):
        with torch.cuda.stream(s1):
            _quiet(pb.normalize, src, target, out=o1)
        with torch.cuda.stream(s2):
            _quiet(pb.normalize, src, target2, out=o2)
    torch.cuda.synchronize()
    assert torch.equal(o1, ref1) and torch.equal(o2, ref2)


def test_fused_unaligned_head_and_tail(monkeypatch):
    """Buffers starting off a 16-byte boundary (same phase) and a pixel count
    that is not a multiple of 16: the < 16-px head and tail go through the
    fp64 path inside the repair launch."""
    import torch

    from paper_1901_03088_b200 import synthetic

    pb = _pb()
    H, W = 4099, 4097                         # > 2^24 px, npix % 16 != 0
    img = synthetic.render_slide(W, H, 17, tissue_fraction=0.5)
    tgt = synthetic.render_slide(1024, 1024, 18, tissue_fraction=0.6)
    target = _quiet(pb.fit, pb.DeviceSource(tgt))
    n = 3 * H * W
    for off in (5, 13):                       # bytes past a 16-byte boundary
        sb = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
        db = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
        src = sb[16 + off:16 + off + n].view(H, W, 3)
        src.copy_(img)
        out = db[16 + off:16 + off + n].view(H, W, 3)
        _quiet(pb.normalize, src, target, out=out)
        ref = _unfused(img, target, monkeypatch)
        assert torch.equal(out, ref), off
    # different phases: normalize takes the host-parameter path (same bytes)
    out = db[16 + 1:16 + 1 + n].view(H, W, 3)
    _quiet(pb.normalize, src, target, out=out)
    assert torch.equal(out, ref)


def _arena(basis, p99, absent=(0, 0)):
    import torch

    raw = np.zeros(88, dtype=np.uint8)
    raw[0:48] = np.asarray(basis, np.float64).reshape(-1).view(np.uint8)
    raw[48:64] = np.asarray(p99, np.float64).view(np.uint8)
    raw[80:88] = np.asarray(absent, np.int32).view(np.uint8)
    return torch.from_numpy(raw).cuda()


def _fitted_call(src, out, lut_dev, arena, target, code_lam=0.0):
    import torch

    from paper_1901_03088_b200 import _lib, pipeline

    L = _lib.lib()
    npix = src.numel() // 3
    p = pipeline._fitted_params(target, code_lam, npix)
    p.src_od_table = _lib.ptr(lut_dev)
    p.src_fit = _lib.ptr(arena)
    ws_bytes = int(L.spcn_xform_workspace_bytes(npix))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    status = torch.full((4,), 7, dtype=torch.int32).pin_memory()
    _lib.check(L.spcn_xform_rgb8_fitted(_lib.ptr(src), _lib.ptr(out), npix, ctypes.byref(p),
                                        _lib.ptr(ws), ws_bytes, _lib.ptr(status),
                                        _lib.stream_handle()), "fitted")
    torch.cuda.synchronize()
    return int(status[0])


def test_fitted_entry_matches_host_parameters(slides):
    """Hand-made fit arena: the device-built block gives the bytes of
    spcn_xform_rgb8 with the host-built block (inline calibration)."""
    import torch

    pb = _pb()
    from paper_1901_03088_b200.fitcore import od_table_cached

    src, target = slides
    i0 = np.array([252.0, 247.0, 241.0])
    basis = np.array([[0.65, 0.07], [0.70, 0.99], [0.29, 0.11]])
    basis /= np.linalg.norm(basis, axis=0)
    p99 = np.array([1.7, 0.9])
    lut = torch.from_numpy(od_table_cached(i0.tobytes()).reshape(-1).copy()).cuda()
    for code_lam in (0.0, 0.05):
        out = torch.empty_like(src)
        assert _fitted_call(src, out, lut, _arena(basis, p99), target, code_lam) == 0
        plan = pb.XformPlan(i0, basis, code_lam, np.asarray(target.stats.p99) / p99,
                            target.basis, target.i0, precision="exact")
        plan.maybe_calibrate(src.numel() // 3, inline=True)
        ref = torch.empty_like(src)
        plan.run(src, ref, src.numel() // 3)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), code_lam


@pytest.mark.parametrize("case", ["absent", "zero_p99", "nonfinite_p99", "bad_norm",
                                  "ill_conditioned"])
def test_fitted_entry_declines_and_leaves_output(slides, case):
    import torch

    from paper_1901_03088_b200.fitcore import od_table_cached

    src, target = slides
    i0 = np.array([255.0, 255.0, 255.0])
    basis = np.array([[0.65, 0.07], [0.70, 0.99], [0.29, 0.11]])
    basis /= np.linalg.norm(basis, axis=0)
    p99, absent = np.array([1.7, 0.9]), (0, 0)
    if case == "absent":
        absent = (0, 1)
    elif case == "zero_p99":
        p99 = np.array([0.0, 0.9])
    elif case == "nonfinite_p99":
        p99 = np.array([np.inf, 0.9])
    elif case == "bad_norm":
        basis = basis * 1.001
    else:                                  # two almost parallel stain vectors
        basis = np.array([[0.6, 0.6000001], [0.64, 0.64], [0.48, 0.4799999]])
        basis /= np.linalg.norm(basis, axis=0)
    lut = torch.from_numpy(od_table_cached(i0.tobytes()).reshape(-1).copy()).cuda()
    out = torch.full_like(src, 77)
    st = _fitted_call(src, out, lut, _arena(basis, p99, absent), target)
    if case == "ill_conditioned":
        assert st == 1, st                   # strict path only: the host path runs it
    else:
        assert st < 0, (case, st)            # invalid: the host path raises
    assert bool((out == 77).all()), case


def test_fitted_entry_argument_errors(slides):
    import torch

    pb = _pb()
    from paper_1901_03088_b200 import _lib, pipeline

    src, target = slides
    L = _lib.lib()
    p = pipeline._fitted_params(target, 0.0, src.numel() // 3)
    ws = torch.empty(1024, dtype=torch.uint8, device="cuda")
    rc = L.spcn_xform_rgb8_fitted(_lib.ptr(src), _lib.ptr(src), src.numel() // 3, ctypes.byref(p),
                                  _lib.ptr(ws), 1024, None, _lib.stream_handle())
    assert rc != 0   # NULL table / arena
    assert L.spcn_last_error()
    del pb


@pytest.mark.parametrize("shape", [(320, 384), (333, 517), (2048, 2048)])
def test_fused_small_images_analytic_bound(shape, monkeypatch):
    """Below 2^24 px the device-built recolouring takes the analytic bound
    (no calibration), as the host path does: same bytes."""
    import torch

    from paper_1901_03088_b200 import synthetic

    pb = _pb()
    h, w = shape
    img = synthetic.render_slide(w, h, 40 + h, tissue_fraction=0.6)
    tgt = synthetic.render_slide(512, 512, 41, tissue_fraction=0.6, i0=(250, 243, 230))
    target = _quiet(pb.fit, pb.DeviceSource(tgt))
    ref = _unfused(img, target, monkeypatch)
    out = torch.empty_like(img)
    _quiet(pb.normalize, img, target, out=out)
    assert torch.equal(out, ref)
    # and normalize(image, image): the target fitted in the same call
    both = _quiet(pb.normalize, img, tgt)
    monkeypatch.setenv("SPCN_FUSED", "0")
    both_ref = _quiet(pb.normalize, img, tgt)
    assert torch.equal(both, both_ref)


def test_fused_pair_errors_match_the_host_order(monkeypatch):
    """normalize(image, image) with both resident runs the two fits in
    lockstep: the target's errors still come first, with the reference's
    types and messages."""
    import torch

    from paper_1901_03088_b200 import synthetic

    pb = _pb()
    img = synthetic.render_slide(640, 480, 77, tissue_fraction=0.6)
    blank = torch.full_like(img, 255)
    sparse = blank.clone()
    sparse[0, :5] = 40                                   # 5 non-white pixels: < 10
    for tgt, src in ((blank, img), (img, blank), (sparse, img), (img, sparse)):
        got = exp = None
        try:
            _quiet(pb.normalize, src, tgt)
        except Exception as exc:      # noqa: BLE001
            got = exc
        monkeypatch.setenv("SPCN_FUSED", "0")
        try:
            _quiet(pb.normalize, src, tgt)
        except Exception as exc:      # noqa: BLE001
            exp = exc
        monkeypatch.delenv("SPCN_FUSED")
        assert exp is not None
        assert type(got) is type(exp) and str(got) == str(exp), (got, exp)


def test_fused_pair_large_calibrated(monkeypatch):
    """Pair path above 2^24 px (calibrated bound), target fitted on the device."""
    import torch

    pb = _pb()
    from paper_1901_03088_b200 import synthetic

    img = synthetic.render_slide(4096, 4100, 91, tissue_fraction=0.5)
    tgt = synthetic.render_slide(1500, 1400, 92, tissue_fraction=0.6, i0=(250, 243, 230))
    out = torch.empty_like(img)
    _quiet(pb.normalize, img, tgt, out=out)
    monkeypatch.setenv("SPCN_FUSED", "0")
    ref = _quiet(pb.normalize, img, tgt)
    assert torch.equal(out, ref)


def test_fused_random_shapes_match_host_path(monkeypatch):
    """Fuzz: odd shapes (down to a few pixels, blank and near-blank images,
    odd strides of the output) — the fused normalize and fit + transform with
    host parameters agree byte for byte, or raise the same error."""
    import torch

    from paper_1901_03088_b200 import synthetic

    pb = _pb()
    rng = np.random.default_rng(7)
    tgt = synthetic.render_slide(300, 260, 5, tissue_fraction=0.6, i0=(250, 243, 230))
    target = _quiet(pb.fit, pb.DeviceSource(tgt))
    for trial in range(24):
        h, w = (int(v) for v in rng.integers(1, 600, size=2))
        tissue = float(rng.choice([0.0, 0.02, 0.3, 0.7]))
        img = synthetic.render_slide(w, h, 100 + trial, tissue_fraction=tissue)
        for tg in (target, tgt):
            res = {}
            for mode in ("1", "0"):
                monkeypatch.setenv("SPCN_FUSED", mode)
                try:
                    res[mode] = _quiet(pb.normalize, img, tg)
                except Exception as exc:      # noqa: BLE001
                    res[mode] = exc
            monkeypatch.delenv("SPCN_FUSED")
            a, b = res["1"], res["0"]
            if isinstance(b, Exception):
                assert type(a) is type(b) and str(a) == str(b), (trial, h, w, a, b)
            else:
                assert torch.is_tensor(a) and torch.equal(a, b), (trial, h, w)
