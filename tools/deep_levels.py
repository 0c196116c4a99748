"""Recursions deeper than the level policy's former clamp (5 levels, leaf order >= 32): exactness
on integer data against an int64 matmul, and times. Dev tool."""
import sys

import torch

sys.path.insert(0, "tools")
from quick_gpu import lib, strassen, timeit  # noqa: E402

NAMES = {1: "strassen", 2: "winograd-block", 3: "winograd-knuth", 4: "knuth-8call", 5: "two-temp", 6: "in-place"}


def case(algo, n, levels, time_it=False):
    g = torch.Generator(device="cuda").manual_seed(n * 31 + levels)
    ai = torch.randint(-8, 9, (n, n), device="cuda", generator=g, dtype=torch.int64)
    bi = torch.randint(-8, 9, (n, n), device="cuda", generator=g, dtype=torch.int64)
    a, b = ai.double(), bi.double()
    ref = (a @ b)  # exact on these integers (|c| <= 64 n)
    c = torch.full((n, n), float("nan"), device="cuda", dtype=torch.float64)
    a2, b2 = a.clone(), b.clone()
    try:
        ws = strassen(algo, a2, b2, c, levels)
    except RuntimeError as e:
        print(f"{NAMES[algo]:15s} n={n:6d} L={levels} leaf={n >> levels}: ERROR {e}", flush=True)
        return
    torch.cuda.synchronize()
    ok = bool(torch.equal(c, ref))
    ms = timeit(lambda: strassen(algo, a2, b2, c, levels), reps=2) if time_it and algo != 6 else float("nan")
    print(f"{NAMES[algo]:15s} n={n:6d} L={levels} leaf={n >> levels:4d}: exact={ok} ws={ws / 2**20:9.1f} MiB {ms:8.2f} ms",
          flush=True)


for algo in range(1, 7):
    case(algo, 256, 6)
    case(algo, 256, 7)
    case(algo, 512, 6)
    case(algo, 1024, 6)
    case(algo, 1024, 7)
for L in (5, 6, 7):
    case(2, 4096, L, True)
for L in (5, 6):
    case(2, 16384, L, True)
