"""Host time of batch._od_tables_exact on the bench batch's i0 values."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import bench
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import batch
sys.argv = [sys.argv[0]]
args = bench.parse()
imgs = bench._batch_images(args, args.seed, args.batch, torch.device("cuda"))
fits = pb.fit_batch(imgs)
i0 = fits.i0.cpu().numpy()
print("distinct i0 per channel", [len(np.unique(i0[:, c])) for c in range(3)])
torch.cuda.synchronize()
for _ in range(3):
    a = time.perf_counter(); t = batch._od_tables_exact(i0, imgs.device); b = time.perf_counter()
    torch.cuda.synchronize(); c = time.perf_counter()
    print("od_tables host %.1f us, +sync %.1f us" % ((b - a) * 1e6, (c - a) * 1e6))
ramp = np.arange(256, dtype=np.float64)
a = time.perf_counter()
for c in range(3):
    vals, inv = np.unique(i0[:, c], return_inverse=True)
b = time.perf_counter()
print("unique x3 %.1f us" % ((b - a) * 1e6))
