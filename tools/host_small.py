"""Host-side cost of a small call (n = 256, cutoff 32, device-resident): wall time per call with
and without synchronising, and a cProfile of 300 calls. Dev tool."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk  # noqa: E402

n, cut = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (256, 32)
a = torch.randint(-8, 9, (n, n), device="cuda").double()
b = torch.randint(-8, 9, (n, n), device="cuda").double()
c = torch.empty_like(a)
A, B, C, pol = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(cut)
for _ in range(10):
    pk.winograd_block_mul(A, B, C, pol)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(300):
    pk.winograd_block_mul(A, B, C, pol)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"n={n} cut={cut}: enqueue {1e3 * (t1 - t0) / 300:.3f} ms/call, with drain {1e3 * (t2 - t0) / 300:.3f} ms/call", flush=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    pk.winograd_block_mul(A, B, C, pol)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
