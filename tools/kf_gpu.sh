cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chol or kf or jl_fold or fold_cert or uncertified or pipeline" 2>&1 | tail -3
timeout 300 python tools/kf_time.py 2>&1 | tail -5
LVSK_KF_TRACE=1 timeout 120 python -c "
import torch, paper_1812_07903_b200 as P
from paper_1812_07903_b200 import _native as N
for d in (512, 4096):
    k=4*d if d<4096 else 16384; r=64 if d<4096 else 128
    sx=torch.randn(k,d,dtype=torch.float64,device='cuda'); G=sx.T@sx; pi=P.leverage.jl_device(0,d,r)
    L=N.lib(); ws=torch.empty(int(L.lvsk_chol_fold_workspace_bytes(d,r)),dtype=torch.uint8,device='cuda')
    M=torch.empty((d,r),dtype=torch.float64,device='cuda'); dg=torch.empty(3,dtype=torch.float64,device='cuda')
    L.lvsk_chol_fold(G.data_ptr(),d,d,pi.data_ptr(),r,M.data_ptr(),dg.data_ptr(),1e10,None,ws.data_ptr(),ws.numel(),N.stream_ptr()); torch.cuda.synchronize()
" 2>&1 | tail -8
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-900
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-1200
