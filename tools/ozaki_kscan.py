"""Per-tile fixed cost vs per-k rate of the Ozaki product: time m=n=4096 products over K."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from ozaki_probe import oz  # noqa: E402

m = n = 4096
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for k in (256, 512, 1024, 2048, 4096):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c = torch.empty(m, n, dtype=torch.float64, device="cuda")
    oz(a, b, S, c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        oz(a, b, S, c)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5
    print(f"S={S} k={k}: {t:.3f} ms, {2 * m * n * k / t / 1e9:.1f} TF/s eq", flush=True)
