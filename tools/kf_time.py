"""Event-timed KF (csrc/factor.cu) vs the cuSOLVER chain for the c2 / c3 / c4 fold shapes."""
import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000.0


def main():
    for k, d, r in ((4096, 512, 64), (4096, 256, 64), (16384, 4096, 128), (2048, 1024, 128)):
        g = torch.Generator(device="cuda").manual_seed(0)
        sx = torch.randn(k, d, dtype=torch.float64, device="cuda", generator=g)
        pi = P.leverage.jl_device(0, d, r)
        G = sx.T @ sx
        L = N.lib()
        ws = torch.empty(int(L.lvsk_chol_fold_workspace_bytes(d, r)), dtype=torch.uint8, device="cuda")
        M = torch.empty((d, r), dtype=torch.float64, device="cuda")
        diag = torch.empty(3, dtype=torch.float64, device="cuda")

        def kf():
            L.lvsk_chol_fold(G.data_ptr(), d, d, pi.data_ptr(), r, M.data_ptr(), diag.data_ptr(), 1e10, None, ws.data_ptr(),
                             ws.numel(), N.stream_ptr())

        def chol_torch():
            Lc, _ = torch.linalg.cholesky_ex(G)
            torch.linalg.solve_triangular(Lc.mT, pi, upper=True)

        print({"k": k, "d": d, "r": r, "gram_us": timeit(lambda: sx.T @ sx), "kf_us": timeit(kf),
               "cusolver_chol_trsm_us": timeit(chol_torch)}, flush=True)


if __name__ == "__main__":
    main()
