"""Host time to enqueue one bench-config call (device-resident operands), per phase."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk  # noqa: E402

n = 16384
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty(n, n, dtype=torch.float64, device="cuda")
A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)
pol = pk.BasePolicy.naive_cutoff(4096)
for _ in range(3):
    pk.winograd_block_mul(A, B, C, pol)
torch.cuda.synchronize()
for i in range(4):
    t0 = time.perf_counter()
    pk.winograd_block_mul(A, B, C, pol)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"call {i}: enqueue {1e3 * (t1 - t0):.2f} ms, total {1e3 * (t2 - t0):.2f} ms", flush=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
pk.winograd_block_mul(A, B, C, pol)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(15)
