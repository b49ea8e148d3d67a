"""Row-band sharded fit (distributed.RowBandGroup) equals the
single-process fit — 2 ranks in 2 processes with gloo collectives, both on
cuda:0 (a functional check of the exchange logic; no kernel waits on another
rank's kernel).  Sample mode and global-p99 mode."""
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


def _worker(rank, world, port, px, mode, q):
    import torch
    import torch.distributed as dist

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import distributed as dd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
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


@pytest.mark.parametrize("mode", ["sample", "global"])
def test_rowband_fit_equals_single_process(mode):
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
    ps = [ctx.Process(target=_worker, args=(r, 2, port, px, mode, q)) for r in range(2)]
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
