"""Per-step device times of the batch workload (C2) + allocator counters,
to find run-to-run variance."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096


class A:
    batch, patch, seed = n, 512, 1


imgs = bench._batch_images(A, 1, n, torch.device("cuda", 0))
out = torch.empty_like(imgs)
tgt = synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)
target = pb.fit(pb.DeviceSource(tgt))
for k in range(12):
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    fits = pb.fit_batch(imgs)
    e1.record()
    pb.transform_batch(imgs, fits, target, out)
    e2.record()
    torch.cuda.synchronize()
    m1 = torch.cuda.memory_stats()
    print(f"step {k}: fit {e0.elapsed_time(e1):7.2f} ms  xform {e1.elapsed_time(e2):6.2f} ms  "
          f"wall {1e3 * (time.perf_counter() - t0):7.2f} ms  cudaMalloc "
          f"{m1.get('num_device_alloc', 0) - m0.get('num_device_alloc', 0)}  free "
          f"{m1.get('num_device_free', 0) - m0.get('num_device_free', 0)}  retries "
          f"{m1.get('num_alloc_retries', 0) - m0.get('num_alloc_retries', 0)}", flush=True)
