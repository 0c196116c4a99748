import cProfile, pstats, sys, os, time, ctypes
import torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
from paper_2309_00628_b200 import _lib
n, cut = 1024, 256
a = torch.randint(-8, 9, (n, n), device="cuda").double(); b = torch.randint(-8, 9, (n, n), device="cuda").double()
c = torch.empty_like(a)
A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix(c)
pol = pk.BasePolicy.naive_cutoff(cut)
for _ in range(5): pk.winograd_block_mul(A, B, C, pol)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(50): pk.winograd_block_mul(A, B, C, pol)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(18)
# raw ABI call time
lib = _lib.load()
ws_b = lib.mk_workspace_bytes(2, n, 2); ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
t0 = time.perf_counter()
for _ in range(50):
    lib.mk_strassen(2, ctypes.c_void_p(a.data_ptr()), n, ctypes.c_void_p(b.data_ptr()), n, ctypes.c_void_p(c.data_ptr()), n, n, 2, ctypes.c_void_p(ws.data_ptr()), ws_b, s)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("raw mk_strassen host time per call (ms):", (t1 - t0) / 50 * 1e3)
