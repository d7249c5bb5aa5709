import torch
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize(); return round(a.elapsed_time(b)/reps,3)
g=torch.Generator(device="cuda").manual_seed(0)
for d in (512, 1024, 4096):
    SX=torch.randn(4*d,d,dtype=torch.float64,device="cuda",generator=g)
    G=SX.T@SX
    L,_=torch.linalg.cholesky_ex(G)
    I=torch.eye(d,dtype=torch.float64,device="cuda")
    Pi=torch.randn(d,128,dtype=torch.float64,device="cuda",generator=g)
    print(d, {"gram_ms": t(lambda: SX.T@SX), "potrf_ms": t(lambda: torch.linalg.cholesky_ex(G)),
       "trsm_Pi_ms": t(lambda: torch.linalg.solve_triangular(L, Pi, upper=False)),
       "trsm_I_ms": t(lambda: torch.linalg.solve_triangular(L, I, upper=False))})
