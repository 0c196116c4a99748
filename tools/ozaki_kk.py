import sys
sys.path.insert(0, "."); sys.path.insert(0, "tools")
import torch
from ozaki_probe import oz
for k in (256, 4096):
    a = torch.randn(4096, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, 4096, dtype=torch.float64, device="cuda")
    c = torch.empty(4096, 4096, dtype=torch.float64, device="cuda")
    oz(a, b, 8, c); torch.cuda.synchronize()
