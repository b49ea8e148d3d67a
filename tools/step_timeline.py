"""GPU timeline of the bench step (fit + transform, or the fused normalize) under torch.profiler:
per step, the kernels in order with their start offsets and durations, and the
idle gaps between them (host round trips).  python tools/step_timeline.py [side]"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
fused = os.environ.get("SPCN_FUSED", "1") != "0"   # step = pb.normalize (device-built params)
slide = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
tgt_img = synthetic.render_slide(2048, 2048, 2)
tgt = pb.fit(pb.DeviceSource(tgt_img))
if os.environ.get("SPCN_PAIR") == "1":   # C1: the target is an image fitted every step
    tgt = tgt_img
src = pb.DeviceSource(slide)
out = torch.empty_like(slide)


p99_mode = os.environ.get("SPCN_P99_MODE", "sample")


def step():
    if p99_mode != "sample":
        fp = pb.fit(src, p99_mode=p99_mode)
        pb.transform(src, fp, tgt, pb.DeviceWriter(side, side, out=out))
        return
    if fused:
        pb.normalize(slide, tgt, out=out)
        return
    fp = pb.fit(src)
    pb.transform(src, fp, tgt, pb.DeviceWriter(side, side, out=out))


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        with torch.profiler.record_function("STEP"):
            step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
steps = [e for e in prof.events() if e.name == "STEP"]
t0 = ev[0].time_range.start
prev_end = None
busy = 0.0
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = (s - prev_end) if prev_end is not None else 0.0
    busy += d
    print(f"{(s - t0) / 1e3:9.3f} ms  gap {gap:8.1f} us  dur {d:9.1f} us  {e.name[:80]}")
    prev_end = max(prev_end or 0, e.time_range.end)
span = (ev[-1].time_range.end - t0) / 1e3
print(f"span {span:.3f} ms for 3 steps, GPU busy {busy / 1e3:.3f} ms")
