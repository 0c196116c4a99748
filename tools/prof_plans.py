"""One workload through the public API, warm, then ONE profiled call (cudaProfilerStart/Stop) for
`ncu --profile-from-start off` launch lists. Also prints the CUDA-event time of that call.

  python tools/prof_plans.py cfg5|inplace8192|twotemp8192|cfg3|bench [plan]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_00628_b200 as pk  # noqa: E402

w = sys.argv[1]
if len(sys.argv) > 2:
    pk.set_plan(sys.argv[2])
r = np.random.default_rng(1)
if w == "cfg5":
    a = torch.from_numpy(r.uniform(-1, 1, (12000, 14000))).cuda()
    b = torch.from_numpy(r.uniform(-1, 1, (14000, 10000))).cuda()
    spec = pk.VariantSpec("winograd-block", pk.BasePolicy.naive_cutoff(512))
    call = lambda: pk.multiply(pk.Matrix(a), pk.Matrix(b), spec)  # noqa: E731
else:
    n = 16384 if w == "bench" else 8192
    cut = {"bench": 4096}.get(w, 1024)
    a = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
    b = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
    c = torch.empty_like(a)
    pol = pk.BasePolicy.naive_cutoff(cut)
    if w == "inplace8192":
        a2, b2 = a.clone(), b.clone()
        call = lambda: pk.in_place_winograd(pk.Matrix(a2), pk.Matrix(b2), pk.Matrix(c), pol)  # noqa: E731
    elif w == "twotemp8192":
        call = lambda: pk.two_temp_winograd(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol)  # noqa: E731
    else:
        call = lambda: pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol)  # noqa: E731
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record()
call()
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"{w}: {e0.elapsed_time(e1):.3f} ms, workspace {pk.last_stats().workspace_bytes / 2**30:.2f} GiB")
