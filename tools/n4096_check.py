import sys, os, time, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n, cut = 4096, 512
a = torch.randint(-8, 9, (n, n), device="cuda").double(); b = torch.randint(-8, 9, (n, n), device="cuda").double()
c = torch.empty_like(a)
A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)
pol = pk.BasePolicy.naive_cutoff(cut)
for _ in range(3): pk.winograd_block_mul(A, B, C, pol)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(10): pk.winograd_block_mul(A, B, C, pol)
    e1.record(); torch.cuda.synchronize(); t = time.perf_counter() - t0
    print("events", e0.elapsed_time(e1) / 10, "wall", t / 10 * 1e3, "ws", pk.last_stats().workspace_bytes / 2**20)
