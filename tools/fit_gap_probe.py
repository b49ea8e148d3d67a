import os, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import paper_1901_03088_b200 as pb
from paper_1901_03088_b200 import synthetic, _lib
side = 4096
slide = synthetic.render_slide(side, side, 1, tissue_fraction=0.6)
tgt = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2)))
src = pb.DeviceSource(slide)
out = torch.empty_like(slide)
L = _lib.lib()
stamps = []
def wrap(name):
    f = getattr(L, name)
    def g(*a):
        stamps.append((name + ">", time.perf_counter()))
        r = f(*a)
        stamps.append((name + "<", time.perf_counter()))
        return r
    setattr(L, name, g)
for n in ("spcn_stream_sync", "spcn_fit_sample_step", "spcn_fit_basis_step", "spcn_xform_rgb8"):
    wrap(n)
for _ in range(5):
    fp = pb.fit(src); pb.transform(src, fp, tgt, pb.DeviceWriter(side, side, out=out))
torch.cuda.synchronize()
acc = {}
for rep in range(30):
    stamps.clear(); stamps.append(("start", time.perf_counter()))
    fp = pb.fit(src)
    stamps.append(("fit<", time.perf_counter()))
    pb.transform(src, fp, tgt, pb.DeviceWriter(side, side, out=out))
    stamps.append(("tr<", time.perf_counter()))
    torch.cuda.synchronize()
    for (a, ta), (b, tb) in zip(stamps, stamps[1:]):
        acc.setdefault(f"{a} -> {b}", []).append((tb - ta) * 1e6)
for k, v in acc.items():
    print(f"{k:50s} median {np.median(v):8.1f} us")
