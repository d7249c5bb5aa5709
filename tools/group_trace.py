import torch
import paper_1812_07903_b200 as P
X = torch.randn(1_000_000, 512, device="cuda")
spec = P.SketchSpec("countsketch", eps=0.5, d=512, seed=0, rows_override=4096)
for _ in range(3):
    P.apply_sketch(X, spec)
torch.cuda.synchronize()
