"""cuSOLVER (torch.linalg.eigh) float64 timing against the matrix size: the
Rayleigh-Ritz block of the rank-capped fold (leverage._topk_gram) picks a
size on the fast side of cuSOLVER's n = 128 / 129 switch."""
import torch


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


g = torch.Generator(device="cuda").manual_seed(0)
for n in (96, 112, 120, 128, 129, 132, 136, 144, 152, 160, 176, 192):
    A = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    B = A @ A.T
    print(n, "eigh %.3f ms" % t(lambda: torch.linalg.eigh(B)), flush=True)
