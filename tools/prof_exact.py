"""ncu driver: calibrated-EXACT transform launches (main + repair) on ~400 Mpx."""
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
rot = np.array([[0.58, 0.12], [0.74, 0.93], [0.33, 0.35]])
rot /= np.linalg.norm(rot, axis=0)
plan = pb.XformPlan([255.0] * 3, reference_basis(), 0.0, [1.2, 0.85], rot, [250.0, 246.0, 240.0],
                    "exact")
plan.calibrate()
for _ in range(3):
    plan.run(src, dst, side * side)
torch.cuda.synchronize()
print("ok", plan.repair_count())
