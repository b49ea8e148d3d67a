"""Host-visible breakdown of one WSI step (fit stages + transform pieces)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import pipeline, snmf, synthetic  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
slide = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2)))
src = pb.DeviceSource(slide)
out = torch.empty_like(slide)


def t(label, fn, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn(*a, **k)
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - t0):8.3f} ms")
    return r


for rep in range(3):
    print("--- rep", rep)
    s, meta = t("sample (device)", pipeline._sample_device, src, pb.SamplePlan())
    fp = t("fit total", pb.fit, src)
    plan = t("XformPlan", pb.XformPlan, fp.i0, fp.basis, 0.0,
             pb.scale_factors(fp.stats, tgt.stats), tgt.basis, tgt.i0)
    t("calibrate", plan.calibrate)
    t("run (main + repair)", plan.run, slide, out, side * side)
    t("transform total", pb.transform, src, fp, tgt, pb.DeviceWriter(side, side, out=out))
