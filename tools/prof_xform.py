"""Minimal driver for ncu: one fast and one calibrated-exact transform launch of ~400 Mpx."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402
from paper_1901_03088_b200.stain_sep import reference_basis  # noqa: E402

side = 20000
src = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
dst = torch.empty_like(src)
w = reference_basis()
rot = np.array([[0.58, 0.12], [0.74, 0.93], [0.33, 0.35]])
rot /= np.linalg.norm(rot, axis=0)
for prec in sys.argv[1:] or ["fast", "exact"]:
    plan = pb.XformPlan([255.0] * 3, w, 0.0, [1.2, 0.85], rot, [250.0, 246.0, 240.0], prec)
    if prec == "exact":
        plan.calibrate()
    for _ in range(2):
        plan.run(src, dst, side * side)
torch.cuda.synchronize()
print("ok")
