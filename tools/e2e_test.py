import os, sys, time, json, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
n = 16384
rng = np.random.default_rng(1)
ha = torch.from_numpy(rng.standard_normal((n, n))).pin_memory(); hb = torch.from_numpy(rng.standard_normal((n, n))).pin_memory()
hc = torch.empty((n, n), dtype=torch.float64).pin_memory()
A, B, C = pk.Matrix(ha.numpy()), pk.Matrix(hb.numpy()), pk.Matrix(hc.numpy())
pol = pk.BasePolicy.naive_cutoff(4096)
# reference: device-resident result
dC = pk.Matrix.zeros(n, n, device="cuda")
pk.winograd_block_mul(pk.Matrix(ha.cuda()), pk.Matrix(hb.cuda()), dC, pol)
want = dC.arr.cpu()
for mode in ("1", "0"):
    os.environ["MK_PIPELINE"] = mode
    for panels in (["-"]):
        os.environ["MK_PIPELINE_PANELS"] = panels if panels != "-" else "4"
        pk.winograd_block_mul(A, B, C, pol); torch.cuda.synchronize()
        t = []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            pk.winograd_block_mul(A, B, C, pol); torch.cuda.synchronize()
            t.append(time.perf_counter() - t0)
        err = float((torch.from_numpy(C.arr) - want).abs().max())
        ms = 1e3 * min(t)
        print(json.dumps({"pipeline": mode, "panels": panels, "ms": round(ms, 1), "e2e_tflops": round(2 * n**3 / ms / 1e9, 2), "maxdiff_vs_device_path": err, "stats": pk.last_stats().__dict__}), flush=True)
