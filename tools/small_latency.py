"""Per-call latency of small products through the API (device-resident): where launch and
planning overheads dominate. Dev tool."""
import json, os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
for n, cut in ((256, 32), (1024, 64), (1024, 256), (2048, 256), (4096, 512)):
    a = torch.randint(-8, 9, (n, n), device="cuda").double(); b = torch.randint(-8, 9, (n, n), device="cuda").double()
    c = torch.empty_like(a)
    A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)
    pol = pk.BasePolicy.naive_cutoff(cut)
    for _ in range(3):
        pk.winograd_block_mul(A, B, C, pol)
    torch.cuda.synchronize()
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        pk.winograd_block_mul(A, B, C, pol)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pk.winograd_block_mul(A, B, C, pol)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"n": n, "cutoff": cut, "levels": pk.last_stats().levels, "wall_ms": round(wall, 3),
                      "gpu_ms": round(e0.elapsed_time(e1) / reps, 3)}))
