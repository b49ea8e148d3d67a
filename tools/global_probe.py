"""Diagnostics of the global-p99 passes on a GPU-rendered slide."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import global_stats as gs, synthetic  # noqa: E402
from paper_1901_03088_b200.pipeline import slide_chunks  # noqa: E402
from paper_1901_03088_b200.stain_sep import reference_basis  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
dev = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
fp = pb.fit(pb.DeviceSource(dev))
eng = gs.DeviceEngine(slide_chunks(pb.DeviceSource(dev)), fp.i0, fp.basis, 0.0, 220)
h0, c0 = eng.hist((0, 0), (gs.SHIFT0, gs.SHIFT0))
h0 = h0.cpu().numpy(); c0 = c0.cpu().numpy()
print("n", c0, "hist sums", h0.sum(axis=1))
for j in range(2):
    nz = np.nonzero(h0[j])[0]
    print(j, "bins used", nz.size, "first/last", nz[:3], nz[-3:], "bin0", h0[j][0])
try:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p99, n, info = gs.global_p99(slide_chunks(pb.DeviceSource(dev)), fp.i0, fp.basis)
    torch.cuda.synchronize()
    print("p99", p99, "n", n, "s", time.perf_counter() - t0)
    print(info)
except RuntimeError as e:
    print("ERR", e)

# per-pass device time
def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


npx = side * side
ms = timed(lambda: eng.hist((0, 0), (gs.SHIFT0, gs.SHIFT0)))
print(f"hist level0 {ms:.2f} ms  {npx / ms / 1e6:.1f} Mpx/s")
g = [1.9, 1.9]
ms = timed(lambda: eng.hist((gs._key_of(1.9), gs._key_of(1.9)), (8, 8)))
print(f"hist zoom   {ms:.2f} ms  {npx / ms / 1e6:.1f} Mpx/s")
ms = timed(lambda: eng.refine([1.95476, 1.94631], [1.95479, 1.94634], 1 << 20))
print(f"refine      {ms:.2f} ms  {npx / ms / 1e6:.1f} Mpx/s")

# whole fit, sample vs global mode (global seeded with the sample bracket)
_orig = gs.global_p99


def _traced(*a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = _orig(*a, **k)
    torch.cuda.synchronize()
    print(f"  global_p99 {1e3 * (time.perf_counter() - t0):.2f} ms passes {r[2]['passes']} "
          f"levels {r[2]['levels']} guess {k.get('guess')}")
    return r


gs.global_p99 = _traced
for mode in ("sample", "global"):
    src = pb.DeviceSource(dev)
    pb.fit(src, p99_mode=mode)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        pb.fit(src, p99_mode=mode)
    torch.cuda.synchronize()
    print(f"fit {mode}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms")
