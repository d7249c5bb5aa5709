"""Event-timed K4-TC (Gaussian sketch) on the C5 shape (bf16 X n x 1024,
k = 2048) for each kernel variant, plus bitwise agreement between them.
Usage: python tools/k4_time.py [n]"""
import os
import sys

import torch

from paper_1812_07903_b200 import _native as N


def run(X, k, reps=10):
    n, d = X.shape
    L = N.lib()
    ws = torch.empty(int(L.lvsk_gaussian_workspace_bytes(n, d, k, N.LVSK_BF16)), dtype=torch.uint8, device="cuda")
    SX = torch.empty((k, d), dtype=torch.float64, device="cuda")
    flags = N.Flags()

    def once():
        N.check(L.lvsk_gaussian_sketch(X.data_ptr(), N.LVSK_BF16, n, d, d, 0, 0, k, SX.data_ptr(), 0, ws.data_ptr(),
                                       ws.numel(), flags.p, N.stream_ptr()), "k4")

    for _ in range(3):
        once()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        once()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, SX.clone()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    d, k = 1024, 2048
    X = torch.rand(n, d, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0)).to(torch.bfloat16)
    res = {}
    for name, env in (("pair_shared_z", "3"), ("shared_z_cluster2", "2"), ("x_multicast", "1")):
        os.environ["LVSK_K4_VARIANT"] = env
        ms, sx = run(X, k)
        tf = 2.0 * k * n * d / (ms / 1e3) / 1e12
        res[name] = (ms, sx)
        print({"variant": name, "n": n, "ms": round(ms, 4), "TFLOPs": round(tf, 1)}, flush=True)
    ref = res["x_multicast"][1]
    for nm, (_, sx) in res.items():
        print({"variant": nm, "bitwise_equal_to_x_multicast": bool(torch.equal(sx, ref))})


if __name__ == "__main__":
    main()
