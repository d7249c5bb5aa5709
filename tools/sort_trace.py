import torch
from paper_1812_07903_b200 import _native as N
for n in (1_000_000, 2_097_152, 4_000_000):
    keys = torch.rand(n, dtype=torch.float64, device="cuda") ** 3 * 1e-5
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    L = N.lib()
    ws = torch.empty(int(L.lvsk_argsort_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        N.check(L.lvsk_argsort_f64(keys.data_ptr(), n, 1, out.data_ptr(), ws.data_ptr(), ws.numel(), N.stream_ptr()))
    torch.cuda.synchronize()
