"""KF at C4's fold shape (d = 4096, r = 128): event time + one traced launch."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1812_07903_b200 as P  # noqa: E402
from paper_1812_07903_b200 import _native as N  # noqa: E402

for d, r in ((4096, 128), (2048, 128), (1024, 128)):
    g = torch.Generator(device="cuda").manual_seed(0)
    sx = torch.randn(4 * d, d, dtype=torch.float64, device="cuda", generator=g)
    pi = P.leverage.jl_device(0, d, r)
    G = sx.T @ sx
    L = N.lib()
    ws = torch.empty(int(L.lvsk_chol_fold_workspace_bytes(d, r)), dtype=torch.uint8, device="cuda")
    M = torch.empty((d, r), dtype=torch.float64, device="cuda")
    diag = torch.empty(3, dtype=torch.float64, device="cuda")

    def kf():
        N.check(L.lvsk_chol_fold(G.data_ptr(), d, d, pi.data_ptr(), r, M.data_ptr(), diag.data_ptr(), 1e10, None,
                                 ws.data_ptr(), ws.numel(), N.stream_ptr()), "kf")

    for _ in range(3):
        kf()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        kf()
    b.record()
    torch.cuda.synchronize()
    print(f"d={d} r={r}: KF {a.elapsed_time(b) / 10:.3f} ms", flush=True)
    os.environ["LVSK_KF_TRACE"] = "1"
    kf()
    torch.cuda.synchronize()
    del os.environ["LVSK_KF_TRACE"]
