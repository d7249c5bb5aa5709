"""Stage timeline of BatchRunner passes (CUDA events on each slot's stream,
relative to one start event): which stages of consecutive passes overlap."""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bench  # noqa: E402
import paper_1812_07903_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.configs()[name]
dtype = {"f32": torch.float32, "bf16": torch.bfloat16}[cfg["dtype"]]
lo, hi, _ = bench.rows_of(name, cfg, 0, 1, None)
n = hi - lo
X = bench.gen_local(name, 0, lo, hi, "cuda")
X = X.to(dtype).contiguous()
Xs = [X] + [X.clone() for _ in range(slots - 1)]
spec = P.SketchSpec(cfg["family"], eps=0.5, d=cfg["d"], seed=0, rows_override=cfg["k"], osnap_s=cfg["s"])
R = P.BatchRunner(spec, n, cfg["d"], dtype, sv_tol=cfg["sv_tol"], jl_dim=cfg["r"], rank=cfg.get("rank"), slots=slots)
for i in range(6):
    R.submit(Xs[i % slots])
R.check()
torch.cuda.synchronize()
NP = 10
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(NP)]
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
for s in R.streams:
    s.wait_stream(torch.cuda.current_stream())
for i in range(NP):
    sl = i % slots
    p, st = R.pipes[sl], R.streams[sl]
    with torch.cuda.stream(st):
        x = Xs[sl]
        ev[i][0].record()
        p._sketch(x)
        ev[i][1].record()
        p._factor()
        ev[i][2].record()
        p._leverage(x)
        ev[i][3].record()
        p._order()
        ev[i][4].record()
R.drain()
torch.cuda.synchronize()
R.check()
names = ["sketch", "factor", "leverage", "order"]
for i in range(NP):
    t = [t0.elapsed_time(e) for e in ev[i]]
    print(f"pass {i} slot {i % slots}: " + "  ".join(f"{names[j]} {t[j]:.3f}-{t[j + 1]:.3f} ({t[j + 1] - t[j]:.3f})"
                                                   for j in range(4)))
print("per pass %.4f ms" % ((t0.elapsed_time(ev[NP - 1][4]) - t0.elapsed_time(ev[slots][0])) / (NP - slots)))
R.close()
