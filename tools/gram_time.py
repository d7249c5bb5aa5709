"""KG (int8 Ozaki Gram) against torch float64 SX^T SX: accuracy on ragged /
scaled shapes, event timing on the config shapes."""
import sys

import torch

from paper_1812_07903_b200 import _native as N


def kg(sx):
    k, d = sx.shape
    L = N.lib()
    ws = torch.empty(int(L.lvsk_gram_workspace_bytes(k, d)), dtype=torch.uint8, device="cuda")
    G = torch.full((d, d), float("nan"), dtype=torch.float64, device="cuda")
    fl = N.Flags()

    def run():
        N.check(L.lvsk_gram_f64(sx.data_ptr(), k, d, sx.stride(0), G.data_ptr(), d, ws.data_ptr(), ws.numel(), fl.p,
                                N.stream_ptr()), "gram")

    return run, G


def upper_mask(d, tile=256):
    i = torch.arange(d, device="cuda")
    return (i[:, None] // tile) <= (i[None, :] // tile)


def check(k, d, scale_cols=False):
    g = torch.Generator(device="cuda").manual_seed(k + d)
    sx = torch.randn(k, d, dtype=torch.float64, device="cuda", generator=g)
    if scale_cols:
        sx *= torch.logspace(-6, 6, d, dtype=torch.float64, device="cuda")
    run, G = kg(sx)
    run()
    torch.cuda.synchronize()
    ref = sx.T @ sx
    m = upper_mask(d)
    diff = torch.where(m, (G - ref).abs(), torch.zeros_like(G))
    err = diff.max().item()
    # Ozaki bound: 2^(e_c + e_d) k 2^-49 with 2^e_c the column max scale
    cm = sx.abs().max(0).values
    bound = (cm[:, None] * cm[None, :]) * sx.shape[0] * 2.0**-49
    rel = (diff / bound).max().item()
    gemm = (sx.abs().T @ sx.abs()) * sx.shape[0] * 2.0**-53  # the float64 GEMM worst-case bound
    rel_gemm = (diff / gemm).max().item()
    print({"k": k, "d": d, "scaled": scale_cols, "max_abs_err": err, "err_over_ozaki_bound": rel,
           "err_over_dgemm_bound": rel_gemm,
           "nan_in_upper": bool(torch.isnan(G[m]).any())}, flush=True)


def timeit(k, d, reps=5):
    g = torch.Generator(device="cuda").manual_seed(1)
    sx = torch.randn(k, d, dtype=torch.float64, device="cuda", generator=g)
    run, G = kg(sx)
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    a.record()
    for _ in range(reps):
        sx.T @ sx
    b.record()
    torch.cuda.synchronize()
    ms_ref = a.elapsed_time(b) / reps
    print({"k": k, "d": d, "kg_ms": round(ms, 3), "cublas_dgemm_full_ms": round(ms_ref, 3)}, flush=True)


if __name__ == "__main__":
    for k, d in ((300, 100), (1000, 700), (4096, 512), (2048, 1024)):
        check(k, d)
    check(3000, 520, scale_cols=True)
    for k, d in ((4096, 512), (2048, 1024), (16384, 4096)):
        timeit(k, d)
