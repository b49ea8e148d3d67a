"""normalize_batch_host (C2 e2e: 4096 x 512^2 from pinned host memory) per
chunk size / lookahead: wall time per batch, Gpx/s."""
import os
import sys
import time
import warnings

import torch

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402

warnings.simplefilter("ignore")


class A:
    batch, patch, seed = 4096, 512, 1


imgs = bench._batch_images(A, 1, 4096, torch.device("cuda", 0))
host = imgs.cpu().pin_memory()
out = torch.empty_like(host).pin_memory()
del imgs
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)))
for chunk in [int(x) for x in (sys.argv[1:] or ["256", "512", "1024"])]:
    for ahead in ("2", "3"):
        os.environ["SPCN_BATCH_AHEAD"] = ahead
        for _ in range(2):
            pb.normalize_batch_host(host, tgt, out, chunk=chunk)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            pb.normalize_batch_host(host, tgt, out, chunk=chunk)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 3
        print(f"chunk {chunk:5d} ahead {ahead}: {dt * 1e3:8.2f} ms  {4096 * 512 * 512 / dt / 1e9:6.2f} Gpx/s",
              flush=True)
