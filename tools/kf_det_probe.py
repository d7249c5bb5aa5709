"""KF determinism vs CTA count: lvsk_chol_fold at inflight 1 and 2 (24 CTAs) over d."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_1812_07903_b200 import _native as N  # noqa: E402
from paper_1812_07903_b200.leverage import _chol_body  # noqa: E402

for d in [256, 512, 576, 640, 768, 1024]:
    g = torch.Generator(device="cuda").manual_seed(d)
    sx = torch.randn(4 * d, d, device="cuda", dtype=torch.float64, generator=g)
    pi = torch.randn(d, 64, device="cuda", dtype=torch.float64, generator=g)
    outs = []
    for inf in (1, 2, 1, 2):
        N.lib().lvsk_set_inflight(inf)
        M, diag = _chol_body(sx, pi, 1e-6)
        torch.cuda.synchronize()
        outs.append((M.clone(), diag.clone()))
    N.lib().lvsk_set_inflight(1)
    same = [bool(torch.equal(outs[0][0], o[0])) for o in outs]
    dm = max(float((outs[0][0] - o[0]).abs().max()) for o in outs)
    print(d, "M equal to run 0:", same, "max diff %.3g" % dm, flush=True)
