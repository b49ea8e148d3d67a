#!/bin/bash
# one-off environment probe of the GPU box (host cores, RAM, GPU, PCIe copy rates)
set -x
nproc; free -g; lscpu | head -20; nvidia-smi; nvidia-smi -q | grep -iE 'pcie|link|bar1' | head -20
python - <<'PY'
import torch, time
x = torch.empty(2<<30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(2<<30, dtype=torch.uint8, device='cuda')
for _ in range(2):
    torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize(); h2d=time.perf_counter()-t
    t=time.perf_counter(); x.copy_(d, non_blocking=True); torch.cuda.synchronize(); d2h=time.perf_counter()-t
print("H2D GB/s", 2*2**30/h2d/1e9, "D2H GB/s", 2*2**30/d2h/1e9)
print(torch.cuda.get_device_properties(0))
PY
