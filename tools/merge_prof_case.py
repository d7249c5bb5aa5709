import torch
from paper_1812_07903_b200.order import argsort_device, merge_argsort_runs
from paper_1812_07903_b200 import _native as N
g = torch.Generator(device="cuda").manual_seed(0)
R=8; n1=1_000_000
s = torch.rand(R * n1, dtype=torch.float64, device="cuda", generator=g) ** 3
p = s / s.sum()
locs = [argsort_device(p[q * n1:(q + 1) * n1].contiguous(), True) for q in range(R)]
runs = torch.cat([o.to(torch.int32) for o in locs]); skeys = torch.cat([p[q * n1:(q + 1) * n1][locs[q]] for q in range(R)])
torch.cuda.synchronize()
merge_argsort_runs(skeys, runs, [n1]*R, True); torch.cuda.synchronize()
