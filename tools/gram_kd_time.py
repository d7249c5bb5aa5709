"""Event-timed KD (lvsk_syrk_f64, DMMA block upper triangle) against cuBLAS
DGEMM SX^T SX for the fold shapes of C1, C2, C3, C5 (and the C5 Cholesky QR)."""
import torch

from paper_1812_07903_b200 import _native as N
from paper_1812_07903_b200.leverage import gram_workspace


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


for k, d in ((1024, 256), (4096, 512), (4096, 256), (2048, 1024), (1024, 136)):
    sx = torch.randn(k, d, dtype=torch.float64, device="cuda")
    ws = gram_workspace(k, d, "cuda")
    G = torch.empty(d, d, dtype=torch.float64, device="cuda")
    L = N.lib()
    f = lambda: L.lvsk_syrk_f64(sx.data_ptr(), k, d, d, G.data_ptr(), d, ws.data_ptr(), ws.numel(), N.stream_ptr())
    print({"k": k, "d": d, "kd_us": round(timeit(f), 1), "cublas_us": round(timeit(lambda: sx.T @ sx), 1)}, flush=True)
