"""Row-band sharded fit (distributed.RowBandGroup) equals the
single-process fit — 2 ranks in 2 processes.  With gloo both ranks share
cuda:0 (a functional check of the exchange logic; no kernel waits on another
rank's kernel); with NCCL (needs >= 2 GPUs, skipped otherwise) each rank owns
its GPU and the collectives run device-direct.  Sample mode and global-p99
mode."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


BACKENDS = ["gloo", pytest.param("nccl", marks=pytest.mark.skipif(
    "__import__('torch').cuda.device_count() < 2", reason="NCCL ranks need >= 2 GPUs"))]


def _init(rank, world, port, backend):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker(rank, world, port, px, mode, q, backend="gloo"):
    import torch.distributed as dist

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import distributed as dd

    _init(rank, world, port, backend)
    try:
        import torch
        H, W = px.shape[:2]
        r0 = rank * (H // world)
        rows = H // world if rank < world - 1 else H - r0
        band = torch.from_numpy(np.ascontiguousarray(px[r0:r0 + rows])).cuda()
        g = dd.RowBandGroup(W, H, r0, rows)
        fp = g.fit(pb.DeviceSource(band), pb.SamplePlan(patch_size=256, max_patches=6,
                                                        target_pixels=40_000), p99_mode=mode)
        q.put((rank, fp.i0.tolist(), fp.basis.tolist(), fp.stats.p99.tolist(),
               fp.stats.sample_count))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", BACKENDS)
@pytest.mark.parametrize("mode", ["sample", "global"])
def test_rowband_fit_equals_single_process(mode, backend):
    import multiprocessing as mp

    import torch

    import paper_1901_03088_b200 as pb
    from oracle import spcn_oracle as orc

    px, _, _ = orc.render(900, 1000, 17, i0=(249, 246, 252), tissue_fraction=0.5)
    ref = pb.fit(pb.DeviceSource(torch.from_numpy(px).cuda()),
                 pb.SamplePlan(patch_size=256, max_patches=6, target_pixels=40_000), p99_mode=mode)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, px, mode, q, backend)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, i0, basis, p99, count in out:
        assert i0 == ref.i0.tolist(), rank
        assert np.array_equal(np.array(basis), ref.basis), rank
        assert p99 == ref.stats.p99.tolist(), rank
        assert count == ref.stats.sample_count, rank


def _xform_worker(rank, world, port, q, backend="gloo"):
    import torch
    import torch.distributed as dist

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import distributed as dd, synthetic

    _init(rank, world, port, backend)
    try:
        W, H = 4096, 4096                      # >= 2^24 px: the EXACT bound is calibrated
        full = synthetic.render_slide(W, H, 5, tissue_fraction=0.6)
        tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(1024, 1024, 6, tissue_fraction=0.6)))
        src_fp = pb.fit(pb.DeviceSource(full))
        r0, rows = rank * (H // world), H // world
        band = full[r0:r0 + rows].contiguous()
        g = dd.RowBandGroup(W, H, r0, rows)
        sink = pb.DeviceWriter(W, rows)
        g.transform(pb.DeviceSource(band), src_fp, tgt, sink)
        ref = pb.DeviceWriter(W, H)
        pb.transform(pb.DeviceSource(full), src_fp, tgt, ref)   # one full calibration
        q.put((rank, bool(torch.equal(sink.pixels, ref.pixels[r0:r0 + rows]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", BACKENDS)
def test_rowband_transform_with_split_calibration(backend):
    """Each rank calibrates 1/N of the colours, one max all-reduce: the bands
    are byte-identical to the single-process transform."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_xform_worker, args=(r, 2, port, q, backend)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok for _, ok in out), out


def test_calibration_parts_max_equals_full():
    import ctypes

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import _dev, _lib
    from paper_1901_03088_b200.xform import XformPlan
    from oracle import spcn_oracle as orc

    w = orc.he_basis()
    plan = XformPlan([250.0, 243.0, 247.0], w, 0.0, [1.1, 0.9], w, [255.0, 255.0, 255.0])
    full = plan.calibrate()
    words = []
    for part in range(3):
        box = {}

        def grab(word, box=box):
            box["w"] = int(word.cpu()[0])
        p2 = XformPlan([250.0, 243.0, 247.0], w, 0.0, [1.1, 0.9], w, [255.0, 255.0, 255.0])
        p2.calibrate_shared(1 << 24, 1 << 20, part, 3, grab)
        words.append(box["w"])
    worst = np.array([max(words)], dtype=np.uint32).view(np.float32)[0]
    assert float(worst) * (1.0 + 2.0 ** -20) == full, (worst, full)   # spcn_xform_calibrate's alpha


def _fused_worker(rank, world, port, q, backend="gloo", side=4096):
    import torch
    import torch.distributed as dist

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import distributed as dd, synthetic

    _init(rank, world, port, backend)
    try:
        W, H = side, side
        full = synthetic.render_slide(W, H, 7, tissue_fraction=0.5)
        tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(1024, 1024, 8, tissue_fraction=0.6)))
        r0, rows = rank * (H // world), H // world
        band = full[r0:r0 + rows].contiguous()
        g = dd.RowBandGroup(W, H, r0, rows)
        out = torch.empty_like(band)
        fp = None
        for _ in range(3):                    # rotates the parameter slots
            fp = g.fit_transform(pb.DeviceSource(band), tgt, out)
        fp_ref = g.fit(pb.DeviceSource(band))
        ref = pb.normalize(full, tgt)          # single process: fit + transform
        q.put((rank, bool(torch.equal(out, ref[r0:r0 + rows])),
               bool(np.array_equal(fp.basis, fp_ref.basis)) and fp.stats.p99.tolist() ==
               fp_ref.stats.p99.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("side", [4096, 1024])      # calibrated bound / analytic bound
@pytest.mark.parametrize("backend", BACKENDS)
def test_rowband_fit_transform_device_built(backend, side):
    """RowBandGroup.fit_transform (device-built parameters, calibration split
    across the ranks) gives each rank the bytes of the single-process
    normalize and the same fit as RowBandGroup.fit."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_fused_worker, args=(r, 2, port, q, backend, side))
          for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok and same for _, ok, same in out), out
