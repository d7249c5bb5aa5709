"""Singular values of the C5 sketch around the rank-100 cut (gap -> iterative top-k feasibility)."""
import torch

import bench
import paper_1812_07903_b200 as P


def main():
    cfg = bench.CONFIGS["c5"]
    X = bench.gen_x(cfg, 0, torch.device("cuda")).to(torch.bfloat16)
    spec = P.SketchSpec("gaussian", eps=0.5, d=cfg["d"], seed=0, rows_override=cfg["k"])
    sx = P.apply_sketch(X, spec).data_device
    s = torch.linalg.svdvals(sx).cpu().numpy()
    print("sigma_1", s[0], "sigma_2", s[1])
    for i in (90, 95, 98, 99, 100, 101, 102, 110, 128, 150, 200):
        print(i, s[i - 1], s[i - 1] / s[0])
    print("gap s100/s101", s[99] / s[100], "s100/s129", s[99] / s[128])


if __name__ == "__main__":
    main()
