"""Event-timed K6 (CSR leverage pass, r = 128) on the C4 matrix (synth.py):
tensor-core kernel vs SIMT kernel, and their agreement."""
import os
import sys

import torch

from paper_1812_07903_b200 import synth as S
from paper_1812_07903_b200.csr import csr_scores


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
    M = torch.randn(4096, 128, dtype=torch.float64, device="cuda") / 64
    out = {}
    for name, env in (("tc", None), ("simt", "LVSK_K6_SIMT")):
        if env:
            os.environ[env] = "1"
        box = {}

        def run():
            box["s"] = csr_scores(m, M)

        ms = timed(run)
        if env:
            del os.environ[env]
        out[name] = box["s"]
        nbytes = m.nnz * 8 + 8 * (n + 1) + 8 * n
        print({"variant": name, "n": n, "nnz": m.nnz, "ms": round(ms, 3), "alg_GBps": round(nbytes / ms / 1e6, 1)},
              flush=True)
    rel = ((out["tc"] - out["simt"]).abs() / out["simt"].abs().clamp_min(1e-30)).max().item()
    print({"max_rel_tc_vs_simt": rel})


if __name__ == "__main__":
    main()
