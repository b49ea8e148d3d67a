"""normalize_batch_host (pinned host in/out) timing over chunk/stream settings."""
import os
import sys
import time
import warnings

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402
import bench  # noqa: E402


class A:
    batch, patch, seed = 4096, 512, 1


dev_imgs = bench._batch_images(A, 1, 4096, torch.device("cuda", 0))
host = dev_imgs.cpu().pin_memory()
out = torch.empty_like(host).pin_memory()
tgt = synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)
target = pb.fit(pb.DeviceSource(tgt))
warnings.simplefilter("ignore")
for chunk, streams in ((1024, 3), (512, 3), (256, 4), (512, 4), (256, 6)):
    pb.normalize_batch_host(host, target, out, chunk=chunk, streams=streams)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        pb.normalize_batch_host(host, target, out, chunk=chunk, streams=streams)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"chunk {chunk:5d} streams {streams}: {dt * 1e3:7.1f} ms  {4096 * 512 * 512 / dt / 1e9:6.2f} Gpx/s",
          flush=True)
# transfer-only ceiling: H2D + D2H of the whole batch on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d = torch.empty_like(dev_imgs)
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(host, non_blocking=True)
with torch.cuda.stream(s2):
    out.copy_(dev_imgs, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"duplex copy of 2 x {host.numel() / 1e9:.2f} GB: {dt * 1e3:.1f} ms")
