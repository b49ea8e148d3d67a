"""Host wall time per normalize(image, image) call (C1) with and without a
final synchronize: separates host pacing from GPU time."""
import os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import synthetic
src = synthetic.render_slide(2048, 2048, 10, tissue_fraction=0.6)
tgt = synthetic.render_slide(2048, 2048, 11, tissue_fraction=0.6)
for _ in range(10):
    pb.normalize(src, tgt)
torch.cuda.synchronize()
for mode in ("nosync", "sync"):
    ts = []
    for _ in range(50):
        a = time.perf_counter()
        pb.normalize(src, tgt)
        if mode == "sync":
            torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    torch.cuda.synchronize()
    ts.sort()
    print(os.environ.get("SPCN_PAIR_SIDE", "1"), mode, "median %.1f us  p10 %.1f us" % (ts[25] * 1e6, ts[5] * 1e6))
