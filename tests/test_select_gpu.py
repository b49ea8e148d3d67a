"""Exact percentile kernels: the cluster path (one large segment) and the
one-CTA-per-segment path agree with numpy's order statistics on awkward
distributions (ties, zeros, outliers far above the p99)."""
import numpy as np
import pytest

from oracle import spcn_oracle as orc

pytestmark = pytest.mark.gpu


def _cases(rng):
    n = 100_000
    yield rng.gamma(2.0, 0.4, (2, n))
    z = rng.gamma(1.5, 0.3, (2, n))
    z[:, rng.random(n) < 0.4] = 0.0                      # many exact zeros
    yield z
    t = np.round(rng.gamma(2.0, 0.4, (2, n)), 2)        # heavy ties
    yield t
    o = rng.gamma(2.0, 0.4, (2, n))
    o[:, :50] = 1e6                                     # outliers: the window misses
    yield o
    yield rng.gamma(2.0, 0.4, (2, 37))                  # tiny segment


def test_percentile_paths_match_numpy():
    import torch

    from paper_1901_03088_b200 import stats as dstats

    rng = np.random.default_rng(12)
    for k, h in enumerate(_cases(rng)):
        n = h.shape[1]
        ref = [orc.pct(h[0], 99.0), orc.pct(h[1], 99.0)]
        d = torch.from_numpy(np.ascontiguousarray(h)).cuda()
        one, _ = dstats.segment_percentiles(d, [0, n], 99.0)                # cluster path
        two = torch.from_numpy(np.ascontiguousarray(np.concatenate([h, h[:, ::-1]], axis=1))).cuda()
        many, _ = dstats.segment_percentiles(two, [0, n, 2 * n], 99.0)      # one CTA each
        assert one.cpu().numpy()[0].tolist() == ref, k
        assert many.cpu().numpy()[0].tolist() == ref, k
        assert many.cpu().numpy()[1].tolist() == ref, k
