"""cProfile of the host side of the global-p99 step (fit(p99_mode=global) + transform)."""
import cProfile, os, pstats, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import synthetic
side = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
slide = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2)))
src = pb.DeviceSource(slide)
out = torch.empty_like(slide)
def step():
    fp = pb.fit(src, p99_mode="global")
    pb.transform(src, fp, tgt, pb.DeviceWriter(side, side, out=out))
for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
