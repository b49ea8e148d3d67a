"""cProfile of pb.fit + pb.transform host work on a device slide."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
slide = pb.DeviceSource(synthetic.render_slide(side, side, 1, tissue_fraction=0.6))
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2)))
out = torch.empty_like(slide.tensor)
for _ in range(5):
    fp = pb.fit(slide)
    pb.transform(slide, fp, tgt, pb.DeviceWriter(side, side, out=out))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    fp = pb.fit(slide)
    pb.transform(slide, fp, tgt, pb.DeviceWriter(side, side, out=out))
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
