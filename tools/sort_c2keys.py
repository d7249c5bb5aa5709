"""K7 on the C2 pipeline's actual probabilities (LVSK_SORT_TRACE=1 prints the phases)."""
import numpy as np
import torch

import bench
import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N

cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda")
X = bench.gen_x(cfg, 0, dev)
spec = P.SketchSpec("countsketch", eps=0.5, d=cfg["d"], seed=0, rows_override=cfg["k"])
res = P.leverage_sketched_trunc(X, spec, 1e-6, jl_dim=cfg["r"])
p = torch.from_numpy(np.ascontiguousarray(P.scores_to_distribution(res.scores))).cuda()
hi = (p.view(torch.int64) >> 32)
u, c = torch.unique(hi, return_counts=True)
print({"n": p.numel(), "distinct_hi32": u.numel(), "max_run": int(c.max()), "runs_gt1": int((c > 1).sum())})
L = N.lib()
out = torch.empty(p.numel(), dtype=torch.int64, device=dev)
ws = torch.empty(int(L.lvsk_argsort_workspace_bytes(p.numel())), dtype=torch.uint8, device=dev)
for _ in range(3):
    N.check(L.lvsk_argsort_f64(p.data_ptr(), p.numel(), 1, out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()))
torch.cuda.synchronize()
ref = np.argsort(-p.cpu().numpy(), kind="stable")
print({"exact": bool(np.array_equal(out.cpu().numpy(), ref))})
