"""cProfile of normalize(image, image) on resident 2048² tiles (C1)."""
import cProfile, os, pstats, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import synthetic
src = synthetic.render_slide(2048, 2048, 10, tissue_fraction=0.6)
tgt = synthetic.render_slide(2048, 2048, 11, tissue_fraction=0.6)
out = torch.empty_like(src)
for _ in range(20):
    pb.normalize(src, tgt, out=out)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    pb.normalize(src, tgt, out=out)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
