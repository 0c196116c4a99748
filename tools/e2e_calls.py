import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n = 16384
rng = np.random.default_rng(1)
ha = torch.from_numpy(rng.standard_normal((n, n))).pin_memory(); hb = torch.from_numpy(rng.standard_normal((n, n))).pin_memory()
hc = torch.empty((n, n), dtype=torch.float64).pin_memory()
A, B, C = pk.Matrix(ha.numpy()), pk.Matrix(hb.numpy()), pk.Matrix(hc.numpy())
pol = pk.BasePolicy.naive_cutoff(4096)
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pk.winograd_block_mul(A, B, C, pol)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"call {i}: {t*1e3:.1f} ms", flush=True)
