"""Per-operation timeline of a literal schedule (MK_HOST_TRACE=1): in-place at n = 4096, L = 2
(leaves of 1024^3, as at n = 8192 L = 3). Dev tool."""
import os
import sys

import torch

sys.path.insert(0, "tools")
import quick_gpu as q  # noqa: E402

n, L = int(os.environ.get("N", "4096")), int(os.environ.get("L", "2"))
algo = int(os.environ.get("ALGO", "6"))
a = torch.randint(-8, 9, (n, n), device="cuda").double()
b = torch.randint(-8, 9, (n, n), device="cuda").double()
c = torch.empty_like(a)
for _ in range(2):  # the second timeline is the warm one
    print("---- call ----", file=sys.stderr, flush=True)
    q.strassen(algo, a.clone(), b.clone(), c, L)
    torch.cuda.synchronize()
