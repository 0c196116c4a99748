"""Largest square order on one B200 through the public API (device-resident, integer-valued FP64):
n = 32768 at 3 levels (exact check against mk_dgemm on a row band) and the workspace plan chosen. Dev tool."""
import json, sys, time, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cut = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randint(-8, 9, (n, n), device="cuda", generator=g).double()
b = torch.randint(-8, 9, (n, n), device="cuda", generator=g).double()
c = torch.empty((n, n), dtype=torch.float64, device="cuda")
free0 = torch.cuda.mem_get_info()[0]
torch.cuda.synchronize(); t0 = time.perf_counter()
pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pk.BasePolicy.naive_cutoff(cut))
torch.cuda.synchronize(); t = time.perf_counter() - t0
st = pk.last_stats()
band = slice(n // 3, n // 3 + 256)
ref = a[band] @ b
ok = bool(torch.equal(c[band], ref))
print(json.dumps({"n": n, "cutoff": cut, "levels": st.levels, "s": round(t, 3), "eff_tflops": round(2 * n ** 3 / t / 1e12, 2),
                  "workspace_gib": round(st.workspace_bytes / 2 ** 30, 2), "free_gib_before": round(free0 / 2 ** 30, 1),
                  "row_band_exact": ok}))
