"""Time K3 (SRHT) at C3 and compare the one-pass sampled kernel with the
two-pass kernels (LVSK_SRHT_V2=1) on the same inputs.

  python tools/srht_time.py [n_log2=21] [d=256] [k=4096]
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_07903_b200 as P  # noqa: E402
from paper_1812_07903_b200 import _native as N  # noqa: E402
from paper_1812_07903_b200.sketch import srht_signs_and_sample  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 21
d = int(sys.argv[2]) if len(sys.argv) > 2 else 256
k = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
n = m = 1 << L
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((n, d), device="cuda", generator=g) / torch.sqrt(torch.arange(1, d + 1, device="cuda").float())
signs, sample = srht_signs_and_sample(0, m, k)
sg = torch.from_numpy(signs.astype(np.int8)).cuda()
sm = torch.from_numpy(sample.astype(np.int64)).cuda()
lib = N.lib()


def run(out):
    ws = N.workspace(lib.lvsk_srht_workspace_bytes(m, d, N.LVSK_F32, k))
    flags = N.Flags()
    st = N.stream_ptr()
    def call():
        N.check(lib.lvsk_srht(X.data_ptr(), N.LVSK_F32, n, d, X.stride(0), m, sg.data_ptr(), sm.data_ptr(), k,
                              math.sqrt(k), out.data_ptr(), ws.data_ptr(), ws.numel(), flags.p, st), "srht")
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    assert flags.read() == 0, flags.read()
    return e0.elapsed_time(e1) / reps


res = {}
for mode in ("v3", "v2"):
    if mode == "v2":
        os.environ["LVSK_SRHT_V2"] = "1"
    else:
        os.environ.pop("LVSK_SRHT_V2", None)
    out = torch.empty((k, d), dtype=torch.float64, device="cuda")
    ms = run(out)
    res[mode] = out.cpu().numpy()
    gbs = n * d * 4 / ms / 1e6
    print(f"{mode}: {ms:.3f} ms  {gbs:.0f} GB/s  ({gbs / 6553.6:.1%} of HBM copy peak)")
rel = np.linalg.norm(res["v3"] - res["v2"]) / np.linalg.norm(res["v2"])
print(f"v3 vs v2 rel diff {rel:.3e}")
# exact check of a few sampled rows in float64
xs = X[:, :].double()
sgd = sg.double()
idx = torch.arange(n, device="cuda", dtype=torch.int64)
for t in (0, 1, k // 2, k - 1):
    p = int(sample[t])
    par = torch.zeros(n, dtype=torch.int64, device="cuda")
    v = idx & p
    while bool(v.any()):
        par ^= v & 1
        v >>= 1
    ref = ((1 - 2 * par).double() * sgd) @ xs / math.sqrt(k)
    err = float((torch.from_numpy(res["v3"][t]).cuda() - ref).norm() / ref.norm())
    print(f"row {t} (p={p}): rel err vs fp64 {err:.2e}")
