"""cProfile of the host side of one C2 step (fit_batch + transform_batch)."""
import cProfile, os, pstats, sys
import torch
sys.path.insert(0, os.getcwd())
import bench
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import synthetic
sys.argv = [sys.argv[0]]
args = bench.parse()
imgs = bench._batch_images(args, args.seed, args.batch, torch.device("cuda"))
out = torch.empty_like(imgs)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)))
def step():
    fits = pb.fit_batch(imgs)
    pb.transform_batch(imgs, fits, tgt, out)
for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
