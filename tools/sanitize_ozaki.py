"""Small INT8 (Ozaki) workload touching every Ozaki kernel (single, persistent, batched splits,
grouped launches, ragged shapes, K chunks, slabs), for compute-sanitizer."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk  # noqa: E402
from paper_2309_00628_b200 import _lib, multigpu as mg  # noqa: E402

lib = _lib.load()
r = np.random.default_rng(5)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for (m, n, k) in [(130, 70, 33), (64, 64, 4500), (1, 1, 1)]:
    a = torch.from_numpy(r.integers(-8, 9, (m, k)).astype(np.float64)).cuda()
    b = torch.from_numpy(r.integers(-8, 9, (k, n)).astype(np.float64)).cuda()
    c = torch.empty((m, n), dtype=torch.float64, device="cuda")
    wsb = lib.mk_ozaki_workspace_bytes(m, n, k, 8)
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device="cuda")
    assert lib.mk_ozaki_dgemm(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0), m, n,
                              k, 8, ws.data_ptr(), wsb, st) == 0
    torch.cuda.synchronize()
    assert torch.equal(c, a @ b), (m, n, k)
pk.set_leaf("ozaki", 8, min_work=0)
n = 256
a = r.integers(-8, 9, (n, n)).astype(np.float64)
b = r.integers(-8, 9, (n, n)).astype(np.float64)
c = pk.Matrix.zeros(n, n)
pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), c, pk.BasePolicy.naive_cutoff(64))  # grouped, batched splits
assert np.array_equal(c.arr, a @ b)
pk.strassen_mul(pk.Matrix(a), pk.Matrix(b), c, pk.BasePolicy.naive_cutoff(128))
assert np.array_equal(c.arr, a @ b)
ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
slabs = [torch.zeros((n // 2, n), dtype=torch.float64, device="cuda") for _ in range(2)]
total = mg.leaf_count("winograd-block", 1) * 8
for rank in range(2):
    f, cnt = mg.shard_range(total, 2, rank)
    mg.partial_product_slabs("winograd-block", ta, tb, slabs, 1, f, cnt)
torch.cuda.synchronize()
assert torch.equal(torch.cat(slabs), ta @ tb)
pk.set_leaf("dmma")
print("sanitize_ozaki ok")
