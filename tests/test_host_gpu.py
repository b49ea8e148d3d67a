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
    got = [None] * 6
    errs = []

    def work(i):
        try:
            s, t = pairs[i % 3]
            got[i] = pb.normalize(s, t)
        except Exception as exc:   # pragma: no cover
            errs.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for i in range(6):
        assert np.array_equal(got[i], ref[i % 3]), i
