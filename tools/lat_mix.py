import json, os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
def run(n, cut, reps=10):
    a = torch.randint(-8, 9, (n, n), device="cuda").double(); b = torch.randint(-8, 9, (n, n), device="cuda").double()
    c = torch.empty_like(a); A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c); pol = pk.BasePolicy.naive_cutoff(cut)
    for _ in range(3): pk.winograd_block_mul(A, B, C, pol)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(reps): pk.winograd_block_mul(A, B, C, pol)
    e1.record(); torch.cuda.synchronize()
    print(n, cut, "gpu", round(e0.elapsed_time(e1)/reps,3), "wall", round((time.perf_counter()-t0)/reps*1e3,3), "reserved GB", round(torch.cuda.memory_reserved()/2**30,2), flush=True)
run(4096, 512); run(1024, 64); run(4096, 512); run(256, 32); run(4096, 512)
