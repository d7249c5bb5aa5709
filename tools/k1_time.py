"""Event-timed K1 (lvsk_hashed_sketch) on the c2 shape, outside the pipeline."""
import torch

import paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N


def main():
    n, d, k = 1_000_000, 512, 4096
    X = torch.randn(n, d, device="cuda", dtype=torch.float32)
    spec = P.SketchSpec("countsketch", eps=0.5, d=d, seed=0, rows_override=k)
    st = P.SketchState(spec, n)
    L = N.lib()
    ws = torch.empty(int(L.lvsk_hashed_workspace_bytes(n, 1, k)), dtype=torch.uint8, device="cuda")
    flags = N.Flags()

    def run():
        N.check(L.lvsk_hashed_sketch(X.data_ptr(), N.LVSK_F32, n, d, d, 0, st._blocks, 1, st._scale,
                                     st._hi.data_ptr(), st._lo.data_ptr(), st._hi.data_ptr(), st._lo.data_ptr(), k,
                                     ws.data_ptr(), ws.numel(), flags.p, N.stream_ptr()), "k1")

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        run()
    b.record()
    torch.cuda.synchronize()
    print({"k1_sketch_ms": a.elapsed_time(b) / 20})


if __name__ == "__main__":
    main()
