"""In-place / two-temp literal schedules at n=8192 L=3 (and n=4096 L=2): device time, exactness on
integer data (dev A/B tool; TAG labels the line)."""
import json, os, sys
import torch
sys.path.insert(0, "tools")
import quick_gpu as q
res = {"tag": os.environ.get("TAG", "")}
for n, L in ((8192, 3), (4096, 2)):
    a = torch.randint(-8, 9, (n, n), device="cuda").double()
    b = torch.randint(-8, 9, (n, n), device="cuda").double()
    ref = a @ b
    c = torch.empty_like(a)
    for algo in (6, 5):
        name = {5: "two_temp", 6: "in_place"}[algo]
        if algo == 6:
            a2, b2 = a.clone(), b.clone()
            q.strassen(6, a2, b2, c, L)
            torch.cuda.synchronize()
            ok = bool(torch.equal(c, ref))
            ms = q.timeit(lambda: q.strassen(6, a2, b2, c, L), reps=3)
        else:
            q.strassen(5, a, b, c, L)
            torch.cuda.synchronize()
            ok = bool(torch.equal(c, ref))
            ms = q.timeit(lambda: q.strassen(5, a, b, c, L), reps=3)
        res[f"{name}_n{n}_L{L}_ms"] = round(ms, 2)
        res[f"{name}_n{n}_L{L}_exact"] = ok
print(json.dumps(res), flush=True)
