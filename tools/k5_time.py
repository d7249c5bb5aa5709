"""Event-timed K5 (leverage pass) on the C2 shape: X fp32 1e6 x 512, r = 64."""
import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N


def main():
    n, d, r = 1_000_000, 512, 64
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(n, d, device="cuda", dtype=torch.float32, generator=g)
    M = torch.randn(d, r, device="cuda", dtype=torch.float64, generator=g) / 30
    ops = P.leverage.KernelOperands(M, X)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    flags = N.Flags()
    for _ in range(3):
        ops.run(X, out, flags.p)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        ops.run(X, out, flags.p)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    ref = ((X[:4096].double() @ M) ** 2).sum(1)
    err = ((out[:4096] - ref).abs() / ref).max().item()
    print({"k5_ms": round(ms, 4), "TBps": round(n * d * 4 / ms / 1e9, 3), "max_rel_err": err})


if __name__ == "__main__":
    main()
