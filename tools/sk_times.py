"""Stream-K A/B: device-resident times of launch-tail-bound workloads with MK_STREAMK on / off
(the engine reads the variable once per process, so run this twice:
    MK_STREAMK=0 python tools/sk_times.py; python tools/sk_times.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_00628_b200 as pk  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tag = "streamk=" + os.environ.get("MK_STREAMK", "1")
r = np.random.default_rng(5)
out = []
for n in (1024, 2048, 3072, 4096, 8192):
    a = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
    b = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
    c = torch.empty_like(a)
    t = timed(lambda: pk.naive_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)), reps=10)
    err = float((c - a @ b).abs().max())
    out.append(f"dgemm n={n}: {t:.3f} ms {2 * n ** 3 / t / 1e9:.2f} TF/s err {err:.1e}")
n = 8192
a = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
b = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
c = torch.empty_like(a)
pol = pk.BasePolicy.naive_cutoff(1024)
a2, b2 = a.clone(), b.clone()
out.append(f"in-place n=8192 L=3: {timed(lambda: pk.in_place_winograd(pk.Matrix(a2), pk.Matrix(b2), pk.Matrix(c), pol), 3, 1):.3f} ms")
out.append(f"two-temp n=8192 L=3: {timed(lambda: pk.two_temp_winograd(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol), 3, 1):.3f} ms")
out.append(f"wino n=8192 L=3: {timed(lambda: pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol), 5, 2):.3f} ms")
pk.set_plan("depth-first")
out.append(f"wino dfs n=8192 L=3: {timed(lambda: pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol), 3, 1):.3f} ms")
pk.set_plan()
del a, b, c, a2, b2
n = 16384
a = torch.from_numpy(r.standard_normal((n, n))).cuda()
b = torch.from_numpy(r.standard_normal((n, n))).cuda()
c = torch.empty_like(a)
for g in (7, 4, 3):
    pk.set_plan(group=g)
    t = timed(lambda: pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(4096)), 5, 2)
    out.append(f"wino n=16384 L=2 group {g}: {t:.3f} ms ({pk.last_stats().workspace_bytes / 2**30:.2f} GiB)")
pk.set_plan()
out.append(f"wino n=16384 L=1: {timed(lambda: pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(8192)), 3, 1):.3f} ms")
out.append(f"in-place n=16384 L=2: {timed(lambda: pk.in_place_winograd(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(4096)), 2, 1):.3f} ms")
for line in out:
    print(tag, line, flush=True)
ar = torch.from_numpy(r.uniform(-1, 1, (12000, 14000))).cuda()
br = torch.from_numpy(r.uniform(-1, 1, (14000, 10000))).cuda()
spec = pk.VariantSpec("winograd-block", pk.BasePolicy.naive_cutoff(512))
t = timed(lambda: pk.multiply(pk.Matrix(ar), pk.Matrix(br), spec), 3, 2)
print(tag, f"cfg5 L=5: {t:.3f} ms ({pk.last_stats().workspace_bytes / 2**30:.2f} GiB)", flush=True)
