"""Serial vs two-stream pipelined passes (independent batches): does the
latency-bound fold / order of pass i overlap the HBM-bound sketch of pass i+1?"""
import os
import sys

import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bench  # noqa: E402
import paper_1812_07903_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.configs()[name]
dtype = {"f32": torch.float32, "bf16": torch.bfloat16}[cfg["dtype"]]
lo, hi, n_total = bench.rows_of(name, cfg, 0, 1, None)
n = hi - lo
X = bench.gen_local(name, 0, lo, hi, "cuda")
if not cfg.get("csr"):
    X = X.to(dtype).contiguous()
spec = P.SketchSpec(cfg["family"], eps=0.5, d=cfg["d"], seed=0, rows_override=cfg["k"], osnap_s=cfg["s"])
pipes = [P.LeveragePipeline(spec, n, cfg["d"], dtype, sv_tol=cfg["sv_tol"], jl_dim=cfg["r"], rank=cfg.get("rank"))
         for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]
K = 20
for p in pipes:
    for _ in range(3):
        p.run(X, check=False)
torch.cuda.synchronize()
for p in pipes:
    p.check()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def serial():
    for _ in range(K):
        pipes[0].run(X, check=False)


def piped():
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for i in range(K):
        with torch.cuda.stream(streams[i % 2]):
            pipes[i % 2].run(X, check=False)
    for s in streams:
        cur.wait_stream(s)


for rep in range(3):
    print(name, "serial %.4f ms/pass" % timed(serial), "two-stream %.4f ms/pass" % timed(piped), flush=True)
for p in pipes:
    p.check()
a, b = pipes[0].scores.clone(), pipes[1].scores.clone()
print("scores equal across instances:", bool(torch.equal(a, b)), bool(torch.equal(pipes[0].idx, pipes[1].idx)))
