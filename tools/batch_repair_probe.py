"""Repair statistics of the EXACT batch transform on the bench's C2 batch:
pixels the analytic certification could not certify, per item group."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import _dev, _lib, synthetic  # noqa: E402

args = bench.parse()
n, P = args.batch, args.patch
imgs = bench._batch_images(args, args.seed, n, torch.device("cuda"))
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, args.seed + 1, tissue_fraction=0.6)))
fits = pb.fit_batch(imgs)
out, errors = pb.transform_batch(imgs, fits, tgt)
torch.cuda.synchronize()
per = P * P
ws_bytes = max(int(_lib.lib().spcn_xform_workspace_bytes(n * per)), 16 + 8 * (65536 + n * per // 8))
ws = _dev.workspace(ws_bytes)
G = min(n, torch.cuda.get_device_properties(0).multi_processor_count)
counts = ws[:8 * G].view(torch.int64).cpu().numpy()
seg = ws[8 * G:8 * G + 24 * n].view(torch.int64).view(n, 3).cpu().numpy()
rep = seg[:, 1] - seg[:, 0]
print("repaired pixels", int(counts.sum()), "of", n * per, f"({counts.sum() / (n * per):.4%})")
groups = 8
per_g = -(-n // groups)
for g in range(groups):
    r = rep[g * per_g:(g + 1) * per_g]
    print(f"group {g}: mean repaired/item {r.mean():9.1f} ({r.mean() / per:.3%}) max {r.max()}")
