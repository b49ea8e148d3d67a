"""Single-slide fit pieces with and without the colour table (100 k samples)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import pipeline, snmf, synthetic, stats as dstats  # noqa: E402
from paper_1901_03088_b200.batch import _od_tables_exact  # noqa: E402

slide = synthetic.render_slide(8192, 8192, 1, tissue_fraction=0.6)
sample, meta = pipeline._sample_device(pb.DeviceSource(slide), pb.SamplePlan())
m = sample.shape[0]
i0 = np.array([[255.0, 255.0, 255.0]])
lut = _od_tables_exact(i0, "cuda")
flat = sample.reshape(-1)
off = torch.tensor([0, m], dtype=torch.int64, device="cuda")
cfg = pb.SnmfConfig()


def timed(fn, reps=20):
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


print("m", m)
print(f"snmf cluster=8 (no table): {timed(lambda: snmf.snmf_batched(flat, off, lut, cfg, cluster=8)):.1f} us")
print(f"snmf cluster=1 + table:    {timed(lambda: snmf.snmf_batched(flat, off, lut, cfg, cluster=1)):.1f} us")
r = snmf.snmf_batched(flat, off, lut, cfg, cluster=1)
print("distinct colours", int(r.table.view(torch.int32)[2 * m].item()))
print(f"code_samples:   {timed(lambda: snmf.code_samples(flat, off, lut, r.basis, 0.0, m)):.1f} us")
print(f"code_table:     {timed(lambda: snmf.code_table(r.table, off, lut, r.basis, 0.0, m, m)):.1f} us")
h = snmf.code_samples(flat, off, lut, r.basis, 0.0, m)
ht = snmf.code_table(r.table, off, lut, r.basis, 0.0, m, m)
print(f"p99 segments:   {timed(lambda: dstats.segment_percentiles(h, off, 99.0)):.1f} us")
print(f"p99 table:      {timed(lambda: snmf.percentile_table(ht, r.table, off, m, 99.0)):.1f} us")
a = dstats.segment_percentiles(h, off, 99.0)[0].cpu().numpy()
b = snmf.percentile_table(ht, r.table, off, m, 99.0)[0].cpu().numpy()
print("equal p99", np.array_equal(a, b))
