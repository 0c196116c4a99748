"""One in-place (default) or two-temp (ALGO=5) product at n = 8192, 3 levels, for ncu launch lists."""
import os
import sys

import torch

sys.path.insert(0, "tools")
import quick_gpu as q  # noqa: E402

n, L, algo = 8192, 3, int(os.environ.get("ALGO", "6"))
a = torch.rand(n, n, device="cuda", dtype=torch.float64)
b = torch.rand(n, n, device="cuda", dtype=torch.float64)
c = torch.empty_like(a)
q.strassen(algo, a, b, c, L)
torch.cuda.synchronize()
print("done")
