"""Host-visible breakdown of the batch step (fit_batch internals + transform)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402


class A:
    patch = 512
    seed = 1


n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
imgs = bench._batch_images(A, 1, n, torch.device("cuda", 0))
target = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2)))
out = torch.empty_like(imgs)
for _ in range(2):
    fits = pb.fit_batch(imgs)
    pb.transform_batch(imgs, fits, target, out)
torch.cuda.synchronize()
t0 = time.perf_counter()
fits = pb.fit_batch(imgs)
torch.cuda.synchronize()
t1 = time.perf_counter()
pb.transform_batch(imgs, fits, target, out)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"fit_batch {1e3 * (t1 - t0):.1f} ms  transform_batch {1e3 * (t2 - t1):.1f} ms")
pr = cProfile.Profile()
pr.enable()
fits = pb.fit_batch(imgs)
pb.transform_batch(imgs, fits, target, out)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
