"""cfg5 (12000x14000 . 14000x10000, L=5 and L=3) device-resident time and max error against
mk_dgemm (dev A/B tool: MK_LIB selects an engine variant, TAG labels the line)."""
import ctypes, hashlib, json, os, sys
import torch
sys.path.insert(0, "tools")
import quick_gpu as q

torch.manual_seed(0)
res = {"tag": os.environ.get("TAG", ""), "lib": os.environ.get("MK_LIB", "default")}
m_, k_, n_ = 12000, 14000, 10000
a = torch.rand(m_, k_, device="cuda", dtype=torch.float64) * 2 - 1
b = torch.rand(k_, n_, device="cuda", dtype=torch.float64) * 2 - 1
c = torch.empty(m_, n_, device="cuda", dtype=torch.float64)
ref = torch.empty_like(c)
q.dgemm(a, b, ref)
for L in [int(x) for x in os.environ.get("LEVELS", "5").split(",")]:
    ws_b = q.lib.mk_rect_workspace_bytes(2, q.I64(m_), q.I64(n_), q.I64(k_), L)
    ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device="cuda")
    f = lambda: q.lib.mk_multiply_rect(2, q.VP(a.data_ptr()), q.I64(k_), q.VP(b.data_ptr()), q.I64(n_),  # noqa: E731
                                       q.VP(c.data_ptr()), q.I64(n_), q.I64(m_), q.I64(n_), q.I64(k_), L,
                                       q.VP(ws.data_ptr()), ctypes.c_size_t(ws_b), q.stream())
    res[f"rect_L{L}_ms"] = round(q.timeit(f, reps=int(os.environ.get("REPS", "5")), warm=2), 2)
    res[f"rect_L{L}_maxdiff"] = float((c - ref).abs().max())
    res[f"rect_L{L}_sha"] = hashlib.sha256(c.cpu().numpy().tobytes()).hexdigest()[:16]
    res[f"rect_L{L}_ws_gib"] = round(ws_b / 2**30, 2)
    del ws
print(json.dumps(res), flush=True)
