"""Rectangular products at mid sizes (device-resident operands): ms per multiply() call, to place
the pipelined plan's size thresholds (A/B with MK_PIPELINE=0/1/2; TAG labels the line). Dev tool."""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk  # noqa: E402

res = {"tag": os.environ.get("TAG", "")}
ev = lambda: torch.cuda.Event(enable_timing=True)
for (m, k, n), cut in (((1200, 1400, 1000), 128), ((3000, 3500, 2500), 128), ((3000, 3500, 2500), 256), ((3000, 3500, 2500), 512),
                       ((6000, 7000, 5000), 256), ((6000, 7000, 5000), 512), ((6000, 7000, 5000), 1024)):
    a = torch.randint(-6, 7, (m, k), device="cuda").double()
    b = torch.randint(-6, 7, (k, n), device="cuda").double()
    v = pk.get_variant("winograd-mod2", cutoff=cut)
    A, B = pk.Matrix(a), pk.Matrix(b)
    for _ in range(2):
        c = pk.multiply(A, B, v)
    torch.cuda.synchronize()
    assert torch.equal(c.arr if isinstance(c.arr, torch.Tensor) else torch.from_numpy(c.arr).cuda(), a @ b), (m, k, n, cut)
    reps = 5
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps):
        pk.multiply(A, B, v)
    e1.record()
    torch.cuda.synchronize()
    res[f"{m}x{k}x{n}_c{cut}"] = round(e0.elapsed_time(e1) / reps, 3)
print(json.dumps(res), flush=True)
