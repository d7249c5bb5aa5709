"""C5 rank-capped fold: does the block subspace iteration still pass its
residual test with fewer Cholesky-QR rounds / power steps?  Times each
schedule on the real C5 sketch (synth.py generator, full 8e6 rows)."""
import time

import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import leverage as Lv
from paper_1812_07903_b200 import synth as S

X = S.gen_c5(0, "cuda")
spec = P.SketchSpec("gaussian", eps=0.5, d=X.shape[1], seed=0, rows_override=2048)
sx = P.apply_sketch(X, spec).data_device.contiguous()
del X
G = Lv.gram_full(sx)


def run(schedule, iters):
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = Lv._topk_gram(G, 100, rounds=1, iters=iters, schedule=schedule)
    torch.cuda.synchronize()
    return res, (time.perf_counter() - t) * 1e3


for sched, iters in (("2,2,1,1,1,2", 6), ("1,1,1,1,1,2", 6), ("1,1,1,1,2", 5), ("2,1,1,1,2", 5)):
    s = [int(v) for v in sched.split(",")]
    for _ in range(2):
        out, ms = run(s, iters)
    print({"schedule": sched, "iters": iters, "accepted": out is not None, "ms": round(ms, 3)}, flush=True)
