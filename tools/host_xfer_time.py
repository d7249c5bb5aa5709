"""Times 8 MB float64 vector transfers: pageable vs pinned-backed numpy arrays."""
import time

import numpy as np
import torch


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / reps * 1000, 3)


n = 1_000_000
d = torch.rand(n, dtype=torch.float64, device="cuda")
page = np.random.rand(n)


def d2h_pinned():
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.copy_(d)
    return h.numpy()


pinned_np = d2h_pinned()


def h2d_staged(a):
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.copy_(torch.from_numpy(a))
    return h.to("cuda", non_blocking=True)


print({
    "d2h_pageable": t(lambda: d.cpu().numpy()),
    "d2h_pinned_alloc": t(d2h_pinned),
    "h2d_pageable": t(lambda: torch.from_numpy(page).to("cuda")),
    "h2d_from_pinned_numpy": t(lambda: torch.from_numpy(pinned_np).to("cuda")),
    "h2d_staged": t(lambda: h2d_staged(page)),
    "np_copy": t(lambda: page.copy()),
    "item": t(lambda: d[:1].item()),
})
