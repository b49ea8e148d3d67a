"""Small runs of every libspcn kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): TMA-ring recolour (exact, fast, strict,
calibration, repair), global-p99 passes (colour table + scan, histogram +
refine), sampling + SNMF + p99 fit, and the batch path.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import global_stats, synthetic  # noqa: E402

warnings.simplefilter("ignore")
side = int(os.environ.get("SANITIZE_SIDE", "1024"))
slide = synthetic.render_slide(side, side + 7, 1, tissue_fraction=0.6)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(512, 512, 2)))
src = pb.DeviceSource(slide)
fp = pb.fit(src)                                           # sampling, i0, SNMF, p99
for precision in ("exact", "fast", "strict"):
    out = pb.DeviceWriter(side, side + 7)
    pb.transform(src, fp, tgt, out, precision=precision)
plan = pb.XformPlan(fp.i0, fp.basis, 0.0, pb.scale_factors(fp.stats, tgt.stats), tgt.basis,
                    tgt.i0, "exact")
plan.calibrate()                                           # k_calibrate
plan.run(slide, torch.empty_like(slide), side * (side + 7))
g = pb.fit(src, p99_mode="global")                         # k_stats_table + k_table_scan
p99, nw, _ = global_stats.global_p99(lambda: iter([slide.reshape(-1)]), fp.i0, fp.basis)
imgs = torch.stack([synthetic.render_slide(128, 96, s, tissue_fraction=0.5) for s in range(6)])
o, errs, fits = pb.normalize_batch(imgs, tgt)              # batch sampling/SNMF/transform
torch.cuda.synchronize()
print("sanitize driver ok", np.round(fp.stats.p99, 4), np.round(g.stats.p99, 4),
      sum(e is None for e in errs))
