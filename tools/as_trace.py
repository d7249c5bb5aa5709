"""K7 coop argsort phase trace (LVSK_SORT_TRACE) at small n for a few CTA counts."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_1812_07903_b200 import order as O  # noqa: E402

os.environ["LVSK_SORT_TRACE"] = "1"
for n in [20000]:
    p = torch.rand(n, device="cuda", dtype=torch.float64)
    p /= p.sum()
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    for mc in ["0", "512", "4096"]:
        os.environ["LVSK_AS_MIN_CHUNK"] = mc
        for _ in range(3):
            O.argsort_device(p, True, out)
            torch.cuda.synchronize()
