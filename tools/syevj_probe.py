"""Latency of cuSOLVER's Jacobi eigensolver (cusolverDnDsyevj) on a 128 x 128
SPD matrix against torch.linalg.eigh (syevd), called through ctypes on the
torch stream.  Probe only (not a product path)."""
import ctypes
import glob
import site

import torch

lib = None
for s in site.getsitepackages():
    for g in glob.glob(s + "/nvidia/cusolver/lib/libcusolver.so.11"):
        lib = ctypes.CDLL(g)
assert lib is not None
vp, ci = ctypes.c_void_p, ctypes.c_int


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000


def main():
    n = 128
    g = torch.Generator(device="cuda").manual_seed(0)
    Y = torch.randn(1024, n, dtype=torch.float64, device="cuda", generator=g)
    H = Y.T @ Y
    h = vp()
    assert lib.cusolverDnCreate(ctypes.byref(h)) == 0
    assert lib.cusolverDnSetStream(h, vp(torch.cuda.current_stream().cuda_stream)) == 0
    params = vp()
    assert lib.cusolverDnCreateSyevjInfo(ctypes.byref(params)) == 0
    lib.cusolverDnXsyevjSetTolerance(params, ctypes.c_double(1e-14))
    lib.cusolverDnXsyevjSetMaxSweeps(params, ci(15))
    A = H.clone()
    W = torch.empty(n, dtype=torch.float64, device="cuda")
    lw = ci()
    # jobz = CUSOLVER_EIG_MODE_VECTOR (1), uplo = CUBLAS_FILL_MODE_LOWER (0)
    assert lib.cusolverDnDsyevj_bufferSize(h, 1, 0, n, vp(A.data_ptr()), n, vp(W.data_ptr()), ctypes.byref(lw),
                                           params) == 0
    work = torch.empty(lw.value, dtype=torch.float64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")

    def run():
        A.copy_(H)
        lib.cusolverDnDsyevj(h, 1, 0, n, vp(A.data_ptr()), n, vp(W.data_ptr()), vp(work.data_ptr()), lw,
                             vp(info.data_ptr()), params)

    us = t(run)
    lam, V = torch.linalg.eigh(H)
    err_val = float((W - lam).abs().max() / lam.abs().max())
    res = float(torch.linalg.matrix_norm(H @ A - A * W) / torch.linalg.matrix_norm(H))
    print({"syevj_128_us": round(us, 1), "eigh_128_us": round(t(lambda: torch.linalg.eigh(H)), 1),
           "info": int(info.item()), "eigval_rel_err": err_val, "residual": res})


if __name__ == "__main__":
    main()
