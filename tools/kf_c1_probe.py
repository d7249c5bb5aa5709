"""KF at C1's shape (d = 256, r = 64): C1's own Gram vs a random one; event
timing, then one traced launch (LVSK_KF_TRACE chain breakdown)."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bench  # noqa: E402
import paper_1812_07903_b200 as P  # noqa: E402
from paper_1812_07903_b200 import _native as N  # noqa: E402

cfg = bench.configs()["c1"]
X = bench.gen_local("c1", 0, 0, cfg["n"], "cuda").float().contiguous()
spec = P.SketchSpec("gaussian", eps=0.5, d=256, seed=0, rows_override=1024)
pipe = P.LeveragePipeline(spec, X.shape[0], 256, torch.float32, sv_tol=1e-6, jl_dim=64)
pipe.run(X)
d, r = 256, 64
pi = P.leverage.jl_device(0, d, r)
L = N.lib()
ws = torch.empty(int(L.lvsk_chol_fold_workspace_bytes(d, r)), dtype=torch.uint8, device="cuda")
M = torch.empty((d, r), dtype=torch.float64, device="cuda")
diag = torch.empty(3, dtype=torch.float64, device="cuda")
for label, sx in (("c1", pipe.sx), ("randn", torch.randn(1024, d, dtype=torch.float64, device="cuda"))):
    G = sx.T @ sx
    def call():
        N.check(L.lvsk_chol_fold(G.data_ptr(), d, d, pi.data_ptr(), r, M.data_ptr(), diag.data_ptr(), 1e10, None,
                                 ws.data_ptr(), ws.numel(), N.stream_ptr()), "kf")
    for _ in range(5):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(label, "KF %.1f us" % (e0.elapsed_time(e1) / 50 * 1000), "diag", diag.tolist(), flush=True)
    os.environ["LVSK_KF_TRACE"] = "1"
    call()
    torch.cuda.synchronize()
    del os.environ["LVSK_KF_TRACE"]
