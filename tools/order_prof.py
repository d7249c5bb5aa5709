"""cProfile of scores_to_distribution + make_plan('dec') on a 1e6 numpy score vector."""
import cProfile
import pstats
import time

import numpy as np
import torch

import paper_1812_07903_b200 as P

s = np.random.rand(1_000_000)
for _ in range(3):
    P.make_plan(P.scores_to_distribution(s), P.OrderingPolicy("dec"))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    p = P.scores_to_distribution(s)
t1 = time.perf_counter()
for _ in range(10):
    P.make_plan(p, P.OrderingPolicy("dec"))
t2 = time.perf_counter()
print({"dist_ms": (t1 - t0) * 100, "plan_ms": (t2 - t1) * 100})
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    P.make_plan(P.scores_to_distribution(s), P.OrderingPolicy("dec"))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
