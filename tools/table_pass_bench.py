"""Device time of the global-p99 one-pass table mode on a GPU-rendered slide:
the cell-class table pass (k_cube_class + k_stats_cube), the scan, and the
whole global_p99 (table mode), against the previous per-pixel table pass
(k_stats_table).  python tools/table_pass_bench.py [side]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import _lib, global_stats as gs, synthetic  # noqa: E402
from paper_1901_03088_b200.pipeline import slide_chunks  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
tissue = float(sys.argv[2]) if len(sys.argv) > 2 else 0.6
dev = synthetic.render_slide(side, side, 1, tissue_fraction=tissue)
npx = side * side
fp = pb.fit(pb.DeviceSource(dev))
chunks = slide_chunks(pb.DeviceSource(dev))
eng = gs.DeviceEngine(chunks, fp.i0, fp.basis, 0.0, 220)
from paper_1901_03088_b200 import fitcore, snmf  # noqa: E402

fb = fitcore.buffers(dev.device, 100_000, 200)
guess = None
# bracket from the fit's sample densities, as fit(p99_mode="global") does
m = fp.stats.sample_count
h = fb.h[:2 * m].view(2, m)
guess = gs.sample_bracket(h)
lo = [float(guess[0, 0]), float(guess[1, 0])]
print("bracket", guess.tolist())


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


L = gs._table_sig()
table = torch.zeros(1 << 24, dtype=torch.int64, device="cuda")
counts = torch.zeros(1, dtype=torch.int64, device="cuda")
cls = torch.empty((32 << 10) + (2 << 20), dtype=torch.uint8, device="cuda")
a = gs._F64x2(*lo)
x = dev.reshape(-1)
P = ctypes.byref(eng.plan.params)
st = _lib.stream_handle()
t_cls = timed(lambda: L.spcn_stats_cube_classes(P, 220, ctypes.byref(a), _lib.ptr(cls), st))
t_cube = timed(lambda: L.spcn_stats_table_cube(_lib.ptr(x), npx, P, 220, ctypes.byref(a),
                                               _lib.ptr(cls), _lib.ptr(table), _lib.ptr(counts), st))
t_old = timed(lambda: L.spcn_stats_table(_lib.ptr(x), npx, P, 220, ctypes.byref(a),
                                         _lib.ptr(table), _lib.ptr(counts), st))
c = np.bincount(cls[:1 << 15].cpu().numpy(), minlength=4)
print(f"cell classes white/below/mixed/candidate = {c.tolist()}")
for name, ms in (("cube classes", t_cls), ("cube table pass", t_cube), ("per-pixel table pass", t_old)):
    print(f"{name:22s} {ms:8.3f} ms  {npx / ms / 1e6:9.1f} Gpx/s  {3 * npx / ms / 1e6:8.1f} GB/s")
torch.cuda.synchronize()
t_all = timed(lambda: gs.global_p99(chunks, fp.i0, fp.basis, guess=guess), reps=3)
p99, n, info = gs.global_p99(chunks, fp.i0, fp.basis, guess=guess)
print(f"global_p99 (table mode) {t_all:.3f} ms  p99 {p99.tolist()} n {n} mode {info.get('mode')} "
      f"colours {info.get('colours')}")

# pixel fractions per cell class (a 4 Mpx sample of rows)
px = dev[:40].reshape(-1, 3).long()
cell = (px[:, 0] >> 3) | ((px[:, 1] >> 3) << 5) | ((px[:, 2] >> 3) << 10)
pc = torch.bincount(cls[:1 << 15].long()[cell], minlength=4).cpu().numpy()
print("pixel fractions white/below/mixed/candidate =", np.round(pc / pc.sum(), 4).tolist())
