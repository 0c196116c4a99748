"""Host planning cost of the cfg5 L=5 rectangular product: dry sizing time, and host-side time of
the real call (enqueue) against its GPU time. Dev tool."""
import ctypes, json, os, sys, time
import torch
sys.path.insert(0, "tools")
import quick_gpu as q
m_, k_, n_ = 12000, 14000, 10000
a = torch.rand(m_, k_, device="cuda", dtype=torch.float64); b = torch.rand(k_, n_, device="cuda", dtype=torch.float64)
c = torch.empty(m_, n_, device="cuda", dtype=torch.float64)
for L in (3, 5):
    t0 = time.perf_counter(); ws_b = q.lib.mk_rect_workspace_bytes(2, q.I64(m_), q.I64(n_), q.I64(k_), L); t_dry = time.perf_counter() - t0
    ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device="cuda")
    f = lambda: q.lib.mk_multiply_rect(2, q.VP(a.data_ptr()), q.I64(k_), q.VP(b.data_ptr()), q.I64(n_), q.VP(c.data_ptr()), q.I64(n_), q.I64(m_), q.I64(n_), q.I64(k_), L, q.VP(ws.data_ptr()), ctypes.c_size_t(ws_b), q.stream())
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter(); f(); t_enq = time.perf_counter() - t0; torch.cuda.synchronize(); t_all = time.perf_counter() - t0
    print(json.dumps({"L": L, "dry_ms": round(t_dry * 1e3, 2), "enqueue_ms": round(t_enq * 1e3, 2), "total_ms": round(t_all * 1e3, 2)}))
