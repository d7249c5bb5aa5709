"""Event-timed K2 (OSNAP s=4 sketch of CSR rows) on the C4 matrix (synth.py)
for the K2 v4 kernel, against the
bit-exact ordered kernel (LVSK_K2_DETERMINISTIC)."""
import os
import sys

import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import synth as S


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
    m = S.gen_c4(0, "cuda", 0, n)
    spec = P.SketchSpec("osnap", eps=0.5, d=4096, seed=0, rows_override=16384, osnap_s=4)
    res = {}
    shapes = [("v4", {})]
    for name, env in shapes + [("ordered_bitexact", {"LVSK_K2_DETERMINISTIC": "1"})]:
        os.environ.update(env)
        box = {}

        def run():
            box["st"] = P.apply_sketch(m, spec)

        ms = timed(run, reps=3 if "ordered" in name else 5)
        sx = box["st"].data_device.clone()
        for k_ in env:
            del os.environ[k_]
        res[name] = sx
        nbytes = m.nnz * 8 + 8 * (n + 1)
        print({"variant": name, "n": n, "ms": round(ms, 3), "alg_GBps": round(nbytes / ms / 1e6, 1)}, flush=True)
    ref = res["ordered_bitexact"]
    for k_, v in res.items():
        rel = float((v - ref).norm() / ref.norm())
        print({"variant": k_, "rel_vs_bitexact": rel, "bitwise": bool(torch.equal(v, ref))})


if __name__ == "__main__":
    main()
