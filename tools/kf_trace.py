import os, torch
import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N
for d, r in ((512, 64), (256, 64)):
    k = 4096
    sx = torch.randn(k, d, dtype=torch.float64, device="cuda")
    pi = P.leverage.jl_device(0, d, r)
    G = sx.T @ sx
    L = N.lib()
    ws = torch.empty(int(L.lvsk_chol_fold_workspace_bytes(d, r)), dtype=torch.uint8, device="cuda")
    M = torch.empty((d, r), dtype=torch.float64, device="cuda")
    diag = torch.empty(3, dtype=torch.float64, device="cuda")
    for _ in range(3):
        L.lvsk_chol_fold(G.data_ptr(), d, d, pi.data_ptr(), r, M.data_ptr(), diag.data_ptr(), 1e10, None, ws.data_ptr(), ws.numel(), N.stream_ptr())
    torch.cuda.synchronize()
