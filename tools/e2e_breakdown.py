"""Breaks the c2 end-to-end step (public API from pinned host memory) into its parts."""
import time

import numpy as np
import torch

import paper_1812_07903_b200 as P


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1000, out


def main():
    n, d = 1_000_000, 512
    Xd = torch.randn(n, d, device="cuda", dtype=torch.float32)
    Xh = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    Xh.copy_(Xd)
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=0, rows_override=4096)
    ms_h2d, _ = t(lambda: Xh.to("cuda", non_blocking=True))
    print({"h2d_ms": ms_h2d, "GBps": Xh.numel() * 4 / ms_h2d / 1e6})
    ms_lev, res = t(lambda: P.leverage_sketched_trunc(Xh, spec, 1e-6, jl_dim=64))
    ms_lev_dev, _ = t(lambda: P.leverage_sketched_trunc(Xd, spec, 1e-6, jl_dim=64))
    ms_dist, p = t(lambda: P.scores_to_distribution(res.scores))
    ms_plan, _ = t(lambda: P.make_plan(p, P.OrderingPolicy("dec")))
    print({"leverage_host_ms": ms_lev, "leverage_devX_ms": ms_lev_dev, "distribution_ms": ms_dist, "plan_ms": ms_plan})


if __name__ == "__main__":
    main()
