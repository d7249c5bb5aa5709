"""Event-timed K7 argsort (lvsk_argsort_f64): cooperative L2-resident kernel vs the
classic 3-kernel passes, with exactness against numpy's stable argsort."""
import os

import numpy as np
import torch

from paper_1812_07903_b200 import _native as N


def run(keys, desc=1, reps=30):
    n = keys.numel()
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    L = N.lib()
    ws = torch.empty(int(L.lvsk_argsort_workspace_bytes(n)), dtype=torch.uint8, device="cuda")

    def f():
        N.check(L.lvsk_argsort_f64(keys.data_ptr(), n, desc, out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()))

    f()
    torch.cuda.synchronize()
    kh = keys.cpu().numpy()
    ref = np.argsort(-kh if desc else kh, kind="stable")
    ok = bool(np.array_equal(out.cpu().numpy(), ref))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return ok, a.elapsed_time(b) / reps * 1000


g = torch.Generator(device="cuda").manual_seed(0)
for mode in ("coop", "classic"):
    os.environ.pop("LVSK_ARGSORT_CLASSIC", None)
    if mode == "classic":
        os.environ["LVSK_ARGSORT_CLASSIC"] = "1"
    for n in (1, 2, 1000, 100_000, 1_000_000, 4_000_000):
        keys = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) ** 3 * 1e-5
        ok, us = run(keys)
        ties = torch.round(keys * 1e8) / 1e8  # heavy ties
        ok2, _ = run(ties, reps=1)
        ok3, _ = run(ties, desc=0, reps=1)
        print({"mode": mode, "n": n, "exact": ok, "ties_desc": ok2, "ties_asc": ok3, "us": round(us, 1)}, flush=True)
    const = torch.full((5000,), 0.25, dtype=torch.float64, device="cuda")
    print({"mode": mode, "all_equal": run(const, reps=1)[0]})
