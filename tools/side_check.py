"""Pipelined plan check (dev tool): small rectangular products whose leaves take narrow tiles, on
integer data (exact), against torch; prints max error and a hash (compare across MK_PIPELINE /
MK_SIDE_ATTACH settings, which must agree bit for bit)."""
import ctypes, hashlib, json, os, sys
import torch
sys.path.insert(0, "tools")
import quick_gpu as q

torch.manual_seed(0)
out = {"pipe": os.environ.get("MK_PIPELINE", "1"), "attach": os.environ.get("MK_SIDE_ATTACH", "1")}
for (m_, k_, n_, L) in ((256, 256, 256, 3), (1200, 1400, 1000, 3), (3000, 3500, 2500, 4), (12000, 14000, 10000, 5)):
    a = torch.randint(-4, 5, (m_, k_), device="cuda").double()
    b = torch.randint(-4, 5, (k_, n_), device="cuda").double()
    c = torch.empty(m_, n_, device="cuda", dtype=torch.float64)
    ws_b = q.lib.mk_rect_workspace_bytes(2, q.I64(m_), q.I64(n_), q.I64(k_), L)
    ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device="cuda")
    rc = q.lib.mk_multiply_rect(2, q.VP(a.data_ptr()), q.I64(k_), q.VP(b.data_ptr()), q.I64(n_), q.VP(c.data_ptr()),
                                q.I64(n_), q.I64(m_), q.I64(n_), q.I64(k_), L, q.VP(ws.data_ptr()), ctypes.c_size_t(ws_b),
                                q.stream())
    assert rc == 0, q.lib.mk_last_error()
    torch.cuda.synchronize()
    ref = a @ b
    out[f"{m_}x{k_}x{n_}_L{L}"] = {"maxerr": float((c - ref).abs().max()),
                                    "sha": hashlib.sha256(c.cpu().numpy().tobytes()).hexdigest()[:12],
                                    "ws_gib": round(ws_b / 2**30, 3)}
    del a, b, c, ws, ref
print(json.dumps(out), flush=True)
