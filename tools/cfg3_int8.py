"""BASELINE cfg3 (n=8192 uniform, winograd-block cutoff 1024 -> 343 leaves of 1024^3) with INT8
leaves, twice (the second for ncu launch lists)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk  # noqa: E402

r = np.random.default_rng(20240901)
a = torch.from_numpy(r.uniform(-1, 1, (8192, 8192))).cuda()
b = torch.from_numpy(r.uniform(-1, 1, (8192, 8192))).cuda()
c = pk.Matrix.zeros(8192, 8192, device="cuda")
pk.set_leaf("ozaki", 8)
for _ in range(2):
    pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), c, pk.BasePolicy.naive_cutoff(1024))
torch.cuda.synchronize()
