"""One warm mk_ozaki_dgemm call for ncu (n, slices from argv)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from ozaki_probe import oz  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
s = int(sys.argv[2]) if len(sys.argv) > 2 else 8
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.empty(n, n, dtype=torch.float64, device="cuda")
oz(a, b, s, c)
torch.cuda.synchronize()
oz(a, b, s, c)
torch.cuda.synchronize()
