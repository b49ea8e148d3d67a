"""GPU-side timeline (CUDA events) of the batch host pipeline's stages."""
import os
import sys
import warnings

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_03088_b200 as pb  # noqa: E402
from paper_1901_03088_b200 import synthetic  # noqa: E402
from paper_1901_03088_b200.batch import _sliced_copy, fit_batch, transform_batch  # noqa: E402
import bench  # noqa: E402


class A:
    batch, patch, seed = 4096, 512, 1


dev_imgs = bench._batch_images(A, 1, 4096, torch.device("cuda", 0))
host = dev_imgs.cpu().pin_memory()
out = torch.empty_like(host).pin_memory()
target = pb.fit(pb.DeviceSource(synthetic.render_slide(2048, 2048, 2, tissue_fraction=0.6)))
warnings.simplefilter("ignore")
chunk, nst = 1024, 4
streams = [torch.cuda.Stream() for _ in range(nst)]
for rep in range(3):
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    base = E()
    base.record()
    marks = []
    starts = list(range(0, 4096, chunk))
    d_in = {}
    done = {}

    def upload(k):
        s = streams[k % nst]
        if k - nst in done:
            done[k - nst].synchronize()
        with torch.cuda.stream(s):
            e0, e1 = E(), E()
            e0.record()
            d_in[k] = torch.empty((chunk, 512, 512, 3), dtype=torch.uint8, device="cuda")
            _sliced_copy(d_in[k], host[starts[k]:starts[k] + chunk], True)
            e1.record()
        marks.append((f"h2d{k}", e0, e1))

    upload(0)
    for k in range(len(starts)):
        if k + 1 < len(starts):
            upload(k + 1)
        s = streams[k % nst]
        with torch.cuda.stream(s):
            e0, e1, e2, e3 = E(), E(), E(), E()
            e0.record()
            fits = fit_batch(d_in[k])
            e1.record()
            o, _ = transform_batch(d_in[k], fits, target)
            e2.record()
            _sliced_copy(out[starts[k]:starts[k] + chunk], o, True)
            e3.record()
            ev = torch.cuda.Event()
            ev.record()
            done[k] = ev
        marks += [(f"fit{k}", e0, e1), (f"xf{k}", e1, e2), (f"d2h{k}", e2, e3)]
    torch.cuda.synchronize()
    if rep == 2:
        for name, a, b in marks:
            print(f"{name:6s} {base.elapsed_time(a):7.1f} -> {base.elapsed_time(b):7.1f}  "
                  f"({a.elapsed_time(b):6.1f} ms)")
