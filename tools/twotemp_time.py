"""two-temp / in-place time and workspace at n=16384 (L=1,2) and n=8192 (L=3), literal tail on/off. Dev tool."""
import json, os, sys
import torch
sys.path.insert(0, "tools")
import quick_gpu as q
for n, Ls in ((16384, (1, 2)), (8192, (2, 3))):
    a = torch.randn(n, n, device="cuda", dtype=torch.float64)
    b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    c = torch.empty_like(a)
    for L in Ls:
        for algo in (5, 6):
            if algo == 6:
                a2, b2 = a.clone(), b.clone()
                ms = q.timeit(lambda: q.strassen(6, a2, b2, c, L), reps=2)
            else:
                ms = q.timeit(lambda: q.strassen(5, a, b, c, L), reps=2)
            ws = q.lib.mk_workspace_bytes(algo, q.I64(n), L)
            q.out(tag=os.environ.get("TAG", ""), algo={5: "two-temp", 6: "in-place"}[algo], n=n, L=L, ms=round(ms, 2),
                  ws_gib=round(ws / 2**30, 3))
