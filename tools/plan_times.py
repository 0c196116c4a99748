"""Device-resident timings of the main plans (dev A/B tool): winograd n=16384 L=2 (bench) and
L=1, n=8192 L=3 (cfg3), cfg5 rectangular L=5 and L=3, plus a max-error check vs mk_dgemm."""
import ctypes, json, os, sys
import torch
sys.path.insert(0, "tools")
import quick_gpu as q

torch.manual_seed(0)
tag = os.environ.get("TAG", "")
res = {"tag": tag}
for n, L in ((16384, 2), (16384, 1), (8192, 3)):
    a = torch.randn(n, n, device="cuda", dtype=torch.float64)
    b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    c = torch.empty_like(a)
    ms = q.timeit(lambda: q.strassen(2, a, b, c, L), reps=3 if n > 8192 else 10, warm=1)
    res[f"n{n}_L{L}_ms"] = round(ms, 2)
    if n == 8192:
        ref = torch.empty_like(a)
        q.dgemm(a, b, ref)
        res["n8192_L3_maxdiff_vs_dgemm"] = float((c - ref).abs().max())
    del a, b, c
m_, k_, n_ = 12000, 14000, 10000
a = torch.rand(m_, k_, device="cuda", dtype=torch.float64)
b = torch.rand(k_, n_, device="cuda", dtype=torch.float64)
c = torch.empty(m_, n_, device="cuda", dtype=torch.float64)
for L in (5, 3):
    ws_b = q.lib.mk_rect_workspace_bytes(2, q.I64(m_), q.I64(n_), q.I64(k_), L)
    ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device="cuda")
    f = lambda: q.lib.mk_multiply_rect(2, q.VP(a.data_ptr()), q.I64(k_), q.VP(b.data_ptr()), q.I64(n_),  # noqa: E731
                                       q.VP(c.data_ptr()), q.I64(n_), q.I64(m_), q.I64(n_), q.I64(k_), L,
                                       q.VP(ws.data_ptr()), ctypes.c_size_t(ws_b), q.stream())
    res[f"rect_L{L}_ms"] = round(q.timeit(f, reps=3, warm=1), 2)
print(json.dumps(res), flush=True)
