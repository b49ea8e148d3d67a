"""Host-array entry (numpy in -> numpy out) through the reusable per-thread
staging buffers: repeated and concurrent calls give the device path's bytes."""
import threading
import warnings

import numpy as np
import pytest

from oracle import spcn_oracle as orc

pytestmark = pytest.mark.gpu


def _pair(seed):
    s, _, _ = orc.render(1500, 1100, seed, tissue_fraction=0.6)
    t, _, _ = orc.render(900, 700, seed + 1, tissue_fraction=0.6, i0=(250, 243, 230))
    return s, t


def test_numpy_path_equals_device_path_repeated():
    import torch

    import paper_1901_03088_b200 as pb

    warnings.simplefilter("ignore")
    for seed in (3, 4, 3):                       # sizes repeat: buffers are reused
        s, t = _pair(seed)
        host = pb.normalize(s, t)
        dev = pb.normalize(torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda())
        assert np.array_equal(host, dev.cpu().numpy()), seed


def test_numpy_path_concurrent_threads():
    import paper_1901_03088_b200 as pb

    warnings.simplefilter("ignore")
    pairs = [_pair(10 + k) for k in range(3)]
    ref = [pb.normalize(s, t) for s, t in pairs]
    # (more threads than recolouring parameter slots: a prepared slot must
    # not be taken by another thread before its recolour is enqueued)
    nthr = 12
    got = [None] * nthr
    errs = []

    def work(i):
        try:
            s, t = pairs[i % 3]
            got[i] = pb.normalize(s, t)
        except Exception as exc:   # pragma: no cover
            errs.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(nthr)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for i in range(nthr):
        assert np.array_equal(got[i], ref[i % 3]), i


def test_streamed_strips_in_flight_keep_their_repair_lists():
    """Many short strips on several streams at once (each with its own fp64
    repair list): byte-identical to one device launch and to the oracle."""
    import torch

    import paper_1901_03088_b200 as pb

    warnings.simplefilter("ignore")
    s, t = _pair(21)
    sp = pb.fit(pb.ArraySource(s))
    tp = pb.fit(pb.ArraySource(t))
    ref = pb.DeviceWriter(s.shape[1], s.shape[0])
    pb.transform(pb.DeviceSource(torch.from_numpy(s).cuda()), sp, tp, ref)
    for workers in (2, 4):
        sink = pb.ArrayWriter(s.shape[1], s.shape[0])
        pb.transform(pb.ArraySource(s), sp, tp, sink, strip_height=48, workers=workers)
        assert np.array_equal(sink.pixels, ref.pixels.cpu().numpy()), workers
    want = orc.run_transform(s, dict(i0=sp.i0, basis=sp.basis, p99=sp.stats.p99),
                             dict(i0=tp.i0, basis=tp.basis, p99=tp.stats.p99), workers=4)
    assert np.array_equal(sink.pixels, want)
