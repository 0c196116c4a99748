"""One bench-config product (n=16384, winograd-block, cutoff 4096) with Ozaki leaves, for ncu launch lists."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk  # noqa: E402

n = 16384
rng = np.random.default_rng(20240901)
a = torch.from_numpy(rng.standard_normal((n, n))).cuda()
b = torch.from_numpy(rng.standard_normal((n, n))).cuda()
c = torch.empty((n, n), dtype=torch.float64, device="cuda")
pk.set_leaf("ozaki", int(sys.argv[1]) if len(sys.argv) > 1 else 8)
A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)
pol = pk.BasePolicy.naive_cutoff(4096)
pk.winograd_block_mul(A, B, C, pol)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pk.winograd_block_mul(A, B, C, pol)
e1.record()
torch.cuda.synchronize()
print("step ms", e0.elapsed_time(e1), file=sys.stderr)
