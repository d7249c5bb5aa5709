"""Event-timed K6-TC v2 (prepared hot window, csr_tc.cu) on the C4 matrix for
several hot-window widths, against v1 (128 resident hot columns) and a float64
recompute of a row sample."""
import os
import sys

import torch

from paper_1812_07903_b200 import _native as N
from paper_1812_07903_b200 import synth as S
from paper_1812_07903_b200.csr import csr_code, csr_prepare


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
    Mf = M.to(torch.float32).contiguous()
    L = N.lib()
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    # float64 recompute of the first rows
    ns = min(n, 20000)
    sub = m.rows(0, ns).to_dense().double()
    ref = ((sub @ Mf.double()) ** 2).sum(1)
    out = torch.empty(n, dtype=torch.float64, device="cuda")

    def v1():
        N.check(L.lvsk_rowsumsq_csr(m.indptr.data_ptr(), m.indices.data_ptr(), m.data.data_ptr(), csr_code(m), m.n,
                                    m.d, Mf.data_ptr(), 128, out.data_ptr(), flags.data_ptr(), N.stream_ptr()), "v1")

    os.environ["LVSK_K6_V1"] = "1"
    ms = timed(v1)
    del os.environ["LVSK_K6_V1"]
    err = ((out[:ns] - ref).abs() / ref.clamp_min(1e-30)).max().item()
    print({"variant": "v1", "ms": round(ms, 3), "max_rel_vs_f64": err}, flush=True)
    for nb in [int(a) for a in (sys.argv[2:] or ["2", "4", "8", "12", "16"])]:
        os.environ["LVSK_K6_HOTBLOCKS"] = str(nb)
        prep = csr_prepare(Mf)
        out.zero_()

        def v2():
            N.check(L.lvsk_rowsumsq_csr_prepared(m.indptr.data_ptr(), m.indices.data_ptr(), m.data.data_ptr(),
                                                 csr_code(m), m.n, m.d, Mf.data_ptr(), 128, prep.data_ptr(),
                                                 prep.numel(), out.data_ptr(), flags.data_ptr(), N.stream_ptr()), "v2")

        ms = timed(v2)
        err = ((out[:ns] - ref).abs() / ref.clamp_min(1e-30)).max().item()
        print({"variant": "v2", "hot_blocks": nb, "ms": round(ms, 3), "max_rel_vs_f64": err,
               "flags": int(flags.item())}, flush=True)


if __name__ == "__main__":
    main()
