"""Host-side profile of the C1 call: pb.normalize(numpy 2048^2, numpy 2048^2)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402

s = synthetic.render_slide(2048, 2048, 1, tissue_fraction=0.6).cpu().numpy()
t = synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6).cpu().numpy()
for _ in range(3):
    pb.normalize(s, t)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    pb.normalize(s, t)
print(f"normalize(numpy, numpy): {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms")
sd, td = torch.from_numpy(s).cuda(), torch.from_numpy(t).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    pb.normalize(sd, td)
torch.cuda.synchronize()
print(f"normalize(cuda, cuda): {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    pb.normalize(s, t)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
