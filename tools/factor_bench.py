"""Times the cuSOLVER building blocks a rank-capped fold could use (d = 1024, k = 2048, fp64)."""
import torch


def timeit(fn, reps=3):
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
    g = torch.Generator(device="cuda").manual_seed(0)
    for k, d in ((2048, 1024), (4096, 512), (16384, 4096)):
        sx = torch.randn(k, d, dtype=torch.float64, device="cuda", generator=g)
        G = sx.T @ sx
        R = torch.linalg.qr(sx, mode="r")[1]
        out = {"k": k, "d": d}
        out["gram_ms"] = timeit(lambda: sx.T @ sx)
        out["qr_r_ms"] = timeit(lambda: torch.linalg.qr(sx, mode="r"))
        out["eigh_ms"] = timeit(lambda: torch.linalg.eigh(G), 2)
        if d <= 1024:
            out["svd_gesvd_R_ms"] = timeit(lambda: torch.linalg.svd(R, full_matrices=False, driver="gesvd"), 1)
            out["svd_gesvdj_R_ms"] = timeit(lambda: torch.linalg.svd(R, full_matrices=False, driver="gesvdj"), 1)
        out["chol_ms"] = timeit(lambda: torch.linalg.cholesky_ex(G))
        print(out, flush=True)


if __name__ == "__main__":
    main()
