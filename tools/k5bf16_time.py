"""Event-timed K5 bf16 (C5 leverage pass: X bf16 n x 1024, r = 128) for the
CTA-pair kernel and the 1-CTA kernel; bitwise agreement."""
import os
import sys

import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N


def run(ops, X, out, fl, reps=10):
    for _ in range(3):
        ops.run(X, out, fl.p)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ops.run(X, out, fl.p)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
    d, r = 1024, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.rand(n, d, device="cuda", generator=g).to(torch.bfloat16)
    M = torch.randn(d, r, device="cuda", dtype=torch.float64, generator=g) / 32
    ops = P.leverage.KernelOperands(M, X)
    fl = N.Flags()
    outs = {}
    for name, env in (("pair", None), ("single", "LVSK_K5_SINGLE_CTA")):
        if env:
            os.environ[env] = "1"
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        ms = run(ops, X, out, fl)
        if env:
            del os.environ[env]
        outs[name] = out
        print({"variant": name, "n": n, "ms": round(ms, 4), "TBps": round(n * (d * 2 + 8) / ms / 1e9, 3),
               "frac": round(n * (d * 2 + 8) / ms / 1e9 / 6553.6, 3)}, flush=True)
    print({"bitwise_equal": bool(torch.equal(outs["pair"], outs["single"]))})


if __name__ == "__main__":
    main()
