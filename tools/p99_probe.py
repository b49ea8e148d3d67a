"""Time the sample-p99 step for one 100k-sample slide: k_p99_seg vs torch.sort."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_03088_b200 import stats as dstats  # noqa: E402

h = torch.rand((2, 100_000), dtype=torch.float64, device="cuda") * 2
seg = torch.tensor([0, 100_000], dtype=torch.int64, device="cuda")


def timed(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print(f"segment_percentiles: {timed(lambda: dstats.segment_percentiles(h, seg, 99.0)):.1f} us")
print(f"torch.sort(dim=1):   {timed(lambda: torch.sort(h, dim=1)):.1f} us")
print(f"torch.topk 1001:     {timed(lambda: torch.topk(h, 1001, dim=1)):.1f} us")
print(f"torch.kthvalue:      {timed(lambda: torch.kthvalue(h, 98_999, dim=1)):.1f} us")
