import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import global_stats as gs, synthetic
from paper_1901_03088_b200.pipeline import slide_chunks
dev = synthetic.render_slide(20000, 20000, 1, tissue_fraction=0.6)
fp = pb.fit(pb.DeviceSource(dev))
for br in ([[1.87, 2.0], [1.867, 2.0]], [[1.5, 2.0], [1.5, 2.0]]):
    p99, n, info = gs.global_p99(slide_chunks(pb.DeviceSource(dev)), fp.i0, fp.basis, guess=np.array(br))
    print(br, info["mode"], "nonwhite", n, "table px", info["table_pixels"], f"{info['table_pixels']/n*100:.2f}%", "colours", info["colours"])
