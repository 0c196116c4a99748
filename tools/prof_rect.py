import sys, ctypes, torch
sys.path.insert(0, "tools")
import quick_gpu as q
m_, k_, n_ = 12000, 14000, 10000
L = int(sys.argv[1]) if len(sys.argv) > 1 else 5
a = torch.rand(m_, k_, device="cuda", dtype=torch.float64)
b = torch.rand(k_, n_, device="cuda", dtype=torch.float64)
c = torch.empty(m_, n_, device="cuda", dtype=torch.float64)
ws_b = q.lib.mk_rect_workspace_bytes(2, q.I64(m_), q.I64(n_), q.I64(k_), L)
ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device="cuda")
rc = q.lib.mk_multiply_rect(2, q.VP(a.data_ptr()), q.I64(k_), q.VP(b.data_ptr()), q.I64(n_), q.VP(c.data_ptr()), q.I64(n_),
                            q.I64(m_), q.I64(n_), q.I64(k_), L, q.VP(ws.data_ptr()), ctypes.c_size_t(ws_b), q.stream())
assert rc == 0
torch.cuda.synchronize()
print("done")
