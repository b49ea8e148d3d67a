"""Quick device-resident timing of the recolor kernel per precision mode.

python tools/quick_xform_bench.py [--mpx 100]
Prints ms, Mpx/s, GB/s (6 B/px algorithmic) and the EXACT repair fraction.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402
from oracle import spcn_oracle as orc  # noqa: E402  (basis helper only)

ap = argparse.ArgumentParser()
ap.add_argument("--mpx", type=int, default=400)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()

side = int((args.mpx * 1e6) ** 0.5) // 16 * 16
src = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
dst = torch.empty_like(src)
npix = src.numel() // 3
w = orc.he_basis()
rot = np.array([[0.58, 0.12], [0.74, 0.93], [0.33, 0.35]])
rot /= np.linalg.norm(rot, axis=0)
ref = torch.empty_like(src)
pb.XformPlan([255.0] * 3, w, 0.0, [1.2, 0.85], np.array([[0.58, 0.12], [0.74, 0.93], [0.33, 0.35]])
             / np.linalg.norm([[0.58, 0.12], [0.74, 0.93], [0.33, 0.35]], axis=0),
             [250.0, 246.0, 240.0], "strict").run(src, ref, npix)
for prec, cal in (("fast", False), ("exact", False), ("exact", True), ("strict", False)):
    plan = pb.XformPlan([255.0] * 3, w, 0.0, [1.2, 0.85], rot, [250.0, 246.0, 240.0], prec)
    if cal:
        t0 = time.perf_counter()
        a = plan.calibrate()
        print(f"calibrated alpha = {a:.3e} in {1e3 * (time.perf_counter() - t0):.2f} ms "
              f"(analytic a0={plan.params.cert_alpha})", flush=True)
    for _ in range(3):
        plan.run(src, dst, npix)
    torch.cuda.synchronize()
    iters = args.iters if prec != "strict" else 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        plan.run(src, dst, npix)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    rep = plan.repair_count() if prec == "exact" else 0
    tag = prec + ("+cal" if cal else "")
    diff = int((dst != ref).sum().item())
    if prec != "fast" and diff:
        print(f"MISMATCH {tag}: {diff} bytes differ from the fp64 path", flush=True)
    print(f"{tag:10s} npix={npix} {ms:.3f} ms  {npix / ms / 1e3:.1f} Mpx/s  "
          f"{6 * npix / ms / 1e6:.1f} GB/s  repaired={rep} ({rep / npix:.5%})", flush=True)
