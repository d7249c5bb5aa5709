cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobi or c5_shaped or jl_fold" 2>&1 | tail -3
cat > /tmp/e1.py <<'PY'
import torch, time
from paper_1812_07903_b200.leverage import small_eigh_desc
n=128
A=torch.randn(n,n,dtype=torch.float64,device="cuda"); A=A@A.T
for f in (lambda: small_eigh_desc(A), lambda: torch.linalg.eigh(A)):
    f(); torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize(); print("ms", a.elapsed_time(b)/10)
PY
timeout 300 python /tmp/e1.py
timeout 600 python -m pytest tests/test_gpu_configs.py -q -x -k "c5" 2>&1 | tail -2
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"factor_ms": [0-9.]*'
