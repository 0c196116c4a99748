"""Breadth-first calls at small orders (device-resident operands): ms per call of winograd_block_mul
for the order / cutoff pairs below, with the current environment (TAG labels the line; A/B with
MK_PIPELINE=0/1, MK_PDL=0/1). Dev tool."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk  # noqa: E402

res = {"tag": os.environ.get("TAG", "")}
ev = lambda: torch.cuda.Event(enable_timing=True)
for n, cut in ((256, 32), (512, 64), (1024, 64), (1024, 128), (2048, 128), (2048, 256), (4096, 256), (4096, 512), (8192, 512)):
    a = torch.randint(-8, 9, (n, n), device="cuda").double()
    b = torch.randint(-8, 9, (n, n), device="cuda").double()
    c = torch.empty_like(a)
    A, B, C, pol = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(cut)
    for _ in range(3):
        pk.winograd_block_mul(A, B, C, pol)
    torch.cuda.synchronize()
    assert torch.equal(c, a @ b), (n, cut)
    reps = 20
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps):
        pk.winograd_block_mul(A, B, C, pol)
    e1.record()
    torch.cuda.synchronize()
    res[f"n{n}_c{cut}"] = round(e0.elapsed_time(e1) / reps, 3)
print(json.dumps(res), flush=True)
