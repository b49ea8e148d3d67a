"""GPU timeline of one C2 batch step (fit_batch + transform_batch) under
torch.profiler: kernels with start offsets/durations and the idle gaps."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402

sys.argv = [sys.argv[0]]
args = bench.parse()
imgs = bench._batch_images(args, args.seed, args.batch, torch.device("cuda"))
out = torch.empty_like(imgs)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)))


def step():
    fits = pb.fit_batch(imgs)
    pb.transform_batch(imgs, fits, tgt, out)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = t0
idle = 0.0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = max(0.0, s - end)
    idle += gap
    print(f"{(s - t0) / 1e3:8.3f} ms  gap {gap:8.1f} us  dur {d:9.1f} us  {e.name[:70]}")
    end = max(end, e.time_range.end)
print(f"span {(end - t0) / 1e3:.3f} ms, idle {idle / 1e3:.3f} ms")
