"""SNMF iteration statistics of the bench's batch workload (diagnostics)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_03088_b200 as pb  # noqa: E402


class A:
    patch = 512
    seed = 1


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
imgs = bench._batch_images(A, 1, n, torch.device("cuda", 0))
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = pb.fit_batch(imgs)
    torch.cuda.synchronize()
    print(f"fit_batch {1e3 * (time.perf_counter() - t0):.1f} ms")
it = f.iterations
print("samples per item: mean", f.count.mean(), "min", f.count.min(), "max", f.count.max())
print("iterations: mean %.1f median %d max %d  (hist %s)" % (
    it.mean(), np.median(it), it.max(), np.histogram(it, bins=[0, 10, 20, 40, 80, 160, 201])[0]))
print("converged", f.converged.mean(), "flags", np.bincount(f.warn_flags))
