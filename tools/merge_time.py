"""Event-timed KM (lvsk_merge_argsort_runs: R sorted runs -> global stable
order) against K7 on all keys — the rank-0 cost of the multi-rank "dec"
order at N = 2, 4, 8 with 1e6 keys per rank."""
import torch

from paper_1812_07903_b200.order import argsort_device, merge_argsort_runs


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000.0


g = torch.Generator(device="cuda").manual_seed(0)
for R in (2, 4, 8):
    n1 = 1_000_000
    s = torch.rand(R * n1, dtype=torch.float64, device="cuda", generator=g) ** 3
    p = s / s.sum()
    locs = [argsort_device(p[q * n1:(q + 1) * n1].contiguous(), True) for q in range(R)]
    runs = torch.cat([o.to(torch.int32) for o in locs])
    skeys = torch.cat([p[q * n1:(q + 1) * n1][locs[q]] for q in range(R)])
    counts = [n1] * R
    out = torch.empty(R * n1, dtype=torch.int64, device="cuda")
    from paper_1812_07903_b200 import _native as N
    ws = torch.empty(int(N.lib().lvsk_merge_runs_workspace_bytes(R * n1, R)), dtype=torch.uint8, device="cuda")
    fl = N.Flags()
    merged = merge_argsort_runs(skeys, runs, counts, True, out, ws, fl)
    assert torch.equal(merged, argsort_device(p, True))
    print({"runs": R, "n": R * n1, "merge_us": round(timeit(lambda: merge_argsort_runs(skeys, runs, counts, True, out, ws, fl)), 1),
           "local_sort_1e6_us": round(timeit(lambda: argsort_device(p[:n1].contiguous(), True)), 1),
           "full_sort_us": round(timeit(lambda: argsort_device(p, True)), 1)}, flush=True)
