"""Breadth-first plan: time and workspace vs top-level products per pass (set_plan(group=g)),
device-resident, CUDA events. Also two-temp literal vs breadth-first tail.

  python tools/group_times.py
"""
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


r = np.random.default_rng(3)
cases = {}
for n in (16384, 8192):
    a = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
    b = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
    cases[n] = (a, b, torch.empty_like(a))
ar = torch.from_numpy(r.uniform(-1, 1, (12000, 14000))).cuda()
br = torch.from_numpy(r.uniform(-1, 1, (14000, 10000))).cuda()
spec = pk.VariantSpec("winograd-block", pk.BasePolicy.naive_cutoff(512))
work = [
    ("wino n16384 L2", lambda: pk.winograd_block_mul(*(pk.Matrix(x) for x in cases[16384]), pk.BasePolicy.naive_cutoff(4096))),
    ("strassen n16384 L2", lambda: pk.strassen_mul(*(pk.Matrix(x) for x in cases[16384]), pk.BasePolicy.naive_cutoff(4096))),
    ("wino n16384 L3", lambda: pk.winograd_block_mul(*(pk.Matrix(x) for x in cases[16384]), pk.BasePolicy.naive_cutoff(2048))),
    ("wino n8192 L3", lambda: pk.winograd_block_mul(*(pk.Matrix(x) for x in cases[8192]), pk.BasePolicy.naive_cutoff(1024))),
    ("cfg5 L5", lambda: pk.multiply(pk.Matrix(ar), pk.Matrix(br), spec)),
]
groups = [int(x) for x in os.environ.get("GROUPS", "7,4,3,2,1").split(",")]
for name, fn in work:
    row = []
    for g in groups:
        pk.set_plan(group=g)
        t = timed(fn, reps=3 if "cfg5" in name or "L3" in name else 5)
        row.append(f"g{g}: {t:8.3f} ms {pk.last_stats().workspace_bytes / 2**30:6.2f} GiB")
        pk.release_workspaces() if hasattr(pk, "release_workspaces") else None
        torch.cuda.empty_cache()
    print(f"{name:20s} " + " | ".join(row), flush=True)
pk.set_plan()
for n, cut in ((16384, 4096), (8192, 1024)):
    row = []
    for tail in (False, True):
        pk.set_plan(two_temp_tail=tail)
        t = timed(lambda: pk.two_temp_winograd(*(pk.Matrix(x) for x in cases[n]), pk.BasePolicy.naive_cutoff(cut)), reps=3)
        row.append(f"tail={tail}: {t:8.3f} ms {pk.last_stats().workspace_bytes / 2**30:6.2f} GiB")
    print(f"two-temp n{n} " + " | ".join(row), flush=True)
pk.set_plan()
