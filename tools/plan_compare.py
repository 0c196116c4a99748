import sys, os, time, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n=16384
a=torch.randn(n,n,device="cuda",dtype=torch.float64); b=torch.randn(n,n,device="cuda",dtype=torch.float64); c=torch.empty_like(a)
A,B,C=pk.Matrix(a),pk.Matrix(b),pk.Matrix(c)
pol=pk.BasePolicy.naive_cutoff(4096)
for plan in ("breadth-first","hybrid","depth-first","hybrid"):
    pk.set_plan(plan)
    pk.winograd_block_mul(A,B,C,pol); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): pk.winograd_block_mul(A,B,C,pol)
    e1.record(); torch.cuda.synchronize()
    print(plan, e0.elapsed_time(e1)/3, pk.last_stats().workspace_bytes/2**30)
pk.set_plan()
