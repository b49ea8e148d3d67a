"""Dump colors where EXACT != STRICT for a parameter set (diagnostics)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1901_03088_b200 as pb
from test_xform_gpu import PARAM_SETS, _resolve, _all_colors
for ps in PARAM_SETS:
    si0, sb, lam, f, tb, ti0 = _resolve(ps)
    px = _all_colors(torch)
    ex = torch.empty_like(px); st = torch.empty_like(px); fa = torch.empty_like(px)
    pb.XformPlan(si0, sb, lam, f, tb, ti0, precision="exact").run(px, ex, px.numel() // 3)
    pb.XformPlan(si0, sb, lam, f, tb, ti0, precision="strict").run(px, st, px.numel() // 3)
    pb.XformPlan(si0, sb, lam, f, tb, ti0, precision="fast").run(px, fa, px.numel() // 3)
    torch.cuda.synchronize()
    m = (ex != st).any(dim=-1).reshape(-1)
    idx = torch.nonzero(m).reshape(-1)
    fm = (fa != st).any(dim=-1).reshape(-1).sum().item()
    print(ps[0], "mismatch", idx.numel(), "fast-vs-strict", fm)
    np.savez(f"gpurun_out/mism_{ps[0]}.npz", idx=idx.cpu().numpy(),
             ex=ex.reshape(-1, 3)[idx].cpu().numpy(), st=st.reshape(-1, 3)[idx].cpu().numpy(),
             fa=fa.reshape(-1, 3)[idx].cpu().numpy(), si0=si0, sb=sb, lam=lam, f=f, tb=tb, ti0=ti0)
