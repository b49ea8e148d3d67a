"""Host-side timeline of normalize_batch_host: per chunk, when the host
enters/leaves fit_batch and transform_batch (ms since start)."""
import os
import sys
import time
import warnings

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import batch, synthetic  # noqa: E402
import bench  # noqa: E402


class A:
    batch, patch, seed = 4096, 512, 1


dev_imgs = bench._batch_images(A, 1, 4096, torch.device("cuda", 0))
host = dev_imgs.cpu().pin_memory()
out = torch.empty_like(host).pin_memory()
target = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)))
warnings.simplefilter("ignore")
log = []
t0 = [0.0]
of, ot = batch.fit_batch, batch.transform_batch


def fb(*a, **k):
    log.append(("fit+", time.perf_counter() - t0[0]))
    r = of(*a, **k)
    log.append(("fit-", time.perf_counter() - t0[0]))
    return r


def tb(*a, **k):
    r = ot(*a, **k)
    log.append(("xf-", time.perf_counter() - t0[0]))
    return r


batch.fit_batch, batch.transform_batch = fb, tb
for chunk in (256, 256, 256):
    torch.cuda.synchronize()
    log.clear()
    m0 = torch.cuda.memory_stats()
    t0[0] = time.perf_counter()
    pb.normalize_batch_host(host, target, out, chunk=chunk, streams=6)
    torch.cuda.synchronize()
    m1 = torch.cuda.memory_stats()
    print(f"chunk {chunk}: total {(time.perf_counter() - t0[0]) * 1e3:.1f} ms  cudaMalloc "
          f"{m1.get('num_device_alloc', 0) - m0.get('num_device_alloc', 0)} free "
          f"{m1.get('num_device_free', 0) - m0.get('num_device_free', 0)}")
    print("  " + " ".join(f"{k}{v * 1e3:.1f}" for k, v in log))
