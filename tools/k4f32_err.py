"""Relative error of the fp32 Gaussian sketch (K4-TC stacked planes vs SIMT) against the fp64 oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1812_07903_b200 as P  # noqa: E402
from oracle import levsketch_oracle as O  # noqa: E402

for n, d, k in [(20000, 256, 1024), (3001, 100, 200), (700, 520, 64), (2100, 1000, 256), (100000, 256, 1024)]:
    x = np.random.default_rng(n).standard_normal((n, d)).astype(np.float32)
    X = torch.from_numpy(x).cuda()
    spec = P.SketchSpec("gaussian", eps=0.5, d=d, seed=4, rows_override=k)
    ref = O.gaussian_sketch(x.astype(np.float64), k, 4)
    tc = P.apply_sketch(X, spec).data
    os.environ["LVSK_NO_TC"] = "1"
    simt = P.apply_sketch(X, spec).data
    del os.environ["LVSK_NO_TC"]
    r = np.linalg.norm(ref)
    print(n, d, k, "tc %.3g" % (np.linalg.norm(tc - ref) / r), "simt %.3g" % (np.linalg.norm(simt - ref) / r), flush=True)
