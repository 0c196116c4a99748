"""Bench config (n=16384 winograd-block cutoff 4096) with INT8 leaves at 6/7/8 slices: time and
error against the naive DMMA product (the cfg4 gate: <= 5.1e-12, the reference CPU's own)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk  # noqa: E402
from paper_2309_00628_b200.metrics import baseline_operands  # noqa: E402

a, b = baseline_operands(4)
da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
del a, b
A, B = pk.Matrix(da), pk.Matrix(db)
cn = pk.Matrix.zeros(16384, 16384, device="cuda")
pk.naive_mul(A, B, cn)
c = pk.Matrix.zeros(16384, 16384, device="cuda")
pol = pk.BasePolicy.naive_cutoff(4096)
for s in (8, 7, 6):
    pk.set_leaf("ozaki", s)
    pk.winograd_block_mul(A, B, c, pol)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        pk.winograd_block_mul(A, B, c, pol)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3
    err = float((c.arr - cn.arr).abs().max())
    print(f"slices {s}: {t:.1f} ms, {2 * 16384 ** 3 / t / 1e9:.1f} TF/s effective, max|C - C_naive| = {err:.3e}",
          flush=True)
pk.set_leaf("dmma")
