"""Tiny tcgen05 K5 check (run first, under a short timeout): v1 and v2 kernels."""
import math
import sys

import torch

sys.path.insert(0, ".")
import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N

for n, d, r in ((300, 32, 64), (5000, 512, 64), (3000, 256, 128), (1000, 40, 30)):
    X = torch.randn(n, d, device="cuda", dtype=torch.float32)
    M = torch.randn(d, r, device="cuda", dtype=torch.float64) / math.sqrt(d)
    hi, lo = P.leverage.split_m_tf32(M)
    hb = hi.to(torch.bfloat16).contiguous()
    ref = ((X.double() @ M) ** 2).sum(1)
    for name, v in (("v1", None), ("v2", hb)):
        out = torch.full((n,), -1.0, dtype=torch.float64, device="cuda")
        fl = N.Flags()
        N.check(N.lib().lvsk_leverage_tf32x3(X.data_ptr(), n, d, d, hi.data_ptr(), lo.data_ptr(), N.ptr(v), r,
                                              out.data_ptr(), fl.p, N.stream_ptr()))
        torch.cuda.synchronize()
        rel = ((out - ref).abs() / ref).max().item()
        print(f"{name} n={n} d={d} r={r} max rel err {rel:.3e} flags={fl.read()} unset={(out < 0).sum().item()}",
              flush=True)
