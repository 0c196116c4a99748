"""DMMA vs INT8 (Ozaki) leaves on the BASELINE configs' shapes (device-resident, CUDA events)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


r = np.random.default_rng(20240901)
MIN_WORK = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 29  # the library default
cases = [("cfg1 n=256 cut32", 256, 256, 256, 32), ("cfg2 n=1024 cut64", 1024, 1024, 1024, 64),
         ("cfg3 n=8192 cut1024", 8192, 8192, 8192, 1024), ("cfg5 12000x14000x10000 cut512", 12000, 14000, 10000, 512),
         ("cfg5 cut2048", 12000, 14000, 10000, 2048), ("n=8192 cut512", 8192, 8192, 8192, 512),
         ("n=4096 cut256", 4096, 4096, 4096, 256), ("n=16384 cut2048", 16384, 16384, 16384, 2048)]
for name, m, k, n, cut in cases:
    a = torch.from_numpy(r.uniform(-1, 1, (m, k))).cuda()
    b = torch.from_numpy(r.uniform(-1, 1, (k, n))).cuda()
    A, B = pk.Matrix(a), pk.Matrix(b)
    spec = pk.VariantSpec("winograd-block", pk.BasePolicy.naive_cutoff(cut))
    out = {}
    for leaf in ("dmma", "ozaki"):
        pk.set_leaf(leaf, 8, min_work=MIN_WORK) if leaf == "ozaki" else pk.set_leaf("dmma")
        if m == k == n:
            c = pk.Matrix.zeros(m, n, device="cuda")
            t = timed(lambda: pk.winograd_block_mul(A, B, c, pk.BasePolicy.naive_cutoff(cut)))
        else:
            t = timed(lambda: pk.multiply(A, B, spec))
        out[leaf] = t
    pk.set_leaf("dmma")
    f = 2.0 * m * n * k
    print(f"{name}: dmma {out['dmma']:.2f} ms ({f / out['dmma'] / 1e9:.1f} TF/s)  "
          f"ozaki {out['ozaki']:.2f} ms ({f / out['ozaki'] / 1e9:.1f} TF/s)", flush=True)
