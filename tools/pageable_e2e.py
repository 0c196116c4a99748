"""Drop-in usage timing: plain (pageable) numpy operands through the public API at n=16384,
winograd-block cutoff 4096 (vs the pinned overlapped path). Dev tool."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
rng = np.random.default_rng(1)
a, b = rng.standard_normal((n, n)), rng.standard_normal((n, n))
c = np.empty((n, n))
pol = pk.BasePolicy.naive_cutoff(4096)
A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pk.winograd_block_mul(A, B, C, pol)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(json.dumps({"rep": i, "pageable_e2e_ms": round(t * 1e3, 1), "tflops": round(2 * n ** 3 / t / 1e12, 2),
                      "path": pk.last_stats().path}), flush=True)
# copy bandwidths
x = torch.from_numpy(a)
for label, src in (("pageable", x), ("pinned", x.pin_memory())):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = src.to("cuda", non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter() - t0
    t0 = time.perf_counter(); h = d.cpu(); t2 = time.perf_counter() - t0
    print(json.dumps({"h2d": label, "GBps": round(a.nbytes / t / 1e9, 1), "d2h_to_pageable_GBps": round(a.nbytes / t2 / 1e9, 1)}))
print(json.dumps({"cpus": os.cpu_count()}))
