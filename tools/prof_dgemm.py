"""One naive_mul (mk_dgemm) of order n after warm-up, between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures.   python tools/prof_dgemm.py 1024"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_00628_b200 as pk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
r = np.random.default_rng(1)
a = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
b = torch.from_numpy(r.uniform(-1, 1, (n, n))).cuda()
c = torch.empty_like(a)
for _ in range(3):
    pk.naive_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c))
torch.cuda.synchronize()
torch.cuda.profiler.start()
pk.naive_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", n)
