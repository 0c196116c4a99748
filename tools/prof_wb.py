"""Run one Winograd/Strassen call (for ncu launch lists / full captures)."""
import sys, torch
sys.path.insert(0, "tools")
import quick_gpu as q
algo, n, L, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 1
a = torch.randn(n, n, device="cuda", dtype=torch.float64)
b = torch.randn(n, n, device="cuda", dtype=torch.float64)
c = torch.empty_like(a)
for _ in range(reps):
    q.strassen(algo, a, b, c, L)
torch.cuda.synchronize()
print("done")
