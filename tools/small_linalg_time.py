"""Latency of the small fp64 linear-algebra calls used by the subspace iteration."""
import torch


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps * 1000, 1)


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    G = torch.randn(1024, 1024, dtype=torch.float64, device="cuda", generator=g)
    G = G @ G.T
    Q = torch.randn(1024, 128, dtype=torch.float64, device="cuda", generator=g)
    B = Q.T @ Q
    L = torch.linalg.cholesky(B)
    print({"gemm_1024x1024x128_us": t(lambda: G @ Q), "gram_128_us": t(lambda: Q.T @ Q),
           "chol_128_us": t(lambda: torch.linalg.cholesky_ex(B)),
           "trsm_1024x128_us": t(lambda: torch.linalg.solve_triangular(L, Q.T, upper=False)),
           "eigh_128_us": t(lambda: torch.linalg.eigh(B)), "eigh_256_us": t(lambda: torch.linalg.eigh(G[:256, :256])),
           "eigh_1024_us": t(lambda: torch.linalg.eigh(G), 3),
           "svd_gesvdj_128_us": t(lambda: torch.linalg.svd(B, driver="gesvdj")),
           "svd_gesvd_128_us": t(lambda: torch.linalg.svd(B, driver="gesvd")),
           "svd_gesvda_128_us": t(lambda: torch.linalg.svd(B, driver="gesvda")),
           "eigvalsh_128_us": t(lambda: torch.linalg.eigvalsh(B)),
           "inv_ex_128_us": t(lambda: torch.linalg.inv_ex(B)),
           "qr_1024x128_us": t(lambda: torch.linalg.qr(Q)),
           "eigh_128_batched2_us": t(lambda: torch.linalg.eigh(torch.stack([B, B]))),
           "eigh_32_batched16_us": t(lambda: torch.linalg.eigh(B[:32, :32].expand(16, 32, 32).contiguous()))})


if __name__ == "__main__":
    main()
