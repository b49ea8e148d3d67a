"""cProfile of the host side of fit + transform on a resident slide (which
Python/ctypes calls sit between the kernels)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402

side = 4096
slide = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2)))
src = pb.DeviceSource(slide)
out = torch.empty_like(slide)


def step():
    fp = pb.fit(src)
    pb.transform(src, fp, tgt, pb.DeviceWriter(side, side, out=out))


for _ in range(5):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
