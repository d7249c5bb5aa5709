"""A/B of the c2 end-to-end step (public API, pinned host X): streamed vs whole-copy ingestion."""
import os
import time

import torch

import paper_1812_07903_b200 as P


def main():
    n, d = 1_000_000, 512
    Xd = torch.randn(n, d, device="cuda", dtype=torch.float32)
    Xh = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    Xh.copy_(Xd)
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=0, rows_override=4096)

    def step():
        res = P.leverage_sketched_trunc(Xh, spec, 1e-6, jl_dim=64)
        return P.make_plan(P.scores_to_distribution(res.scores), P.OrderingPolicy("dec")).indices

    for mode in ("0", "1", "0"):
        os.environ["LVSK_STREAM"] = "0" if mode == "1" else "1"
        step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print({"no_stream": mode, "ms": dt * 1000, "rows_per_s": n / dt})


if __name__ == "__main__":
    main()
