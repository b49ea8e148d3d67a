"""Wall time of normalize(numpy, numpy) for a 2048² tile (C1 e2e)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import synthetic
src = synthetic.render_slide(2048, 2048, 10, tissue_fraction=0.6).cpu().numpy()
tgt = synthetic.render_slide(2048, 2048, 11, tissue_fraction=0.6).cpu().numpy()
for _ in range(5):
    pb.normalize(src, tgt)
ts = []
for _ in range(30):
    a = time.perf_counter()
    pb.normalize(src, tgt)
    ts.append(time.perf_counter() - a)
ts.sort()
print(os.environ.get("SPCN_WHOLE_UPLOAD", "1"), "median %.3f ms" % (ts[15] * 1e3))
