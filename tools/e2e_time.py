"""e2e (pinned host operands through the public API) vs device-resident timing at n=16384,
winograd-block cutoff 4096, plus agreement of the two results. Dev tool."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cut = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
rng = np.random.default_rng(1)
ha = torch.from_numpy(rng.standard_normal((n, n))).pin_memory()
hb = torch.from_numpy(rng.standard_normal((n, n))).pin_memory()
hc = torch.empty((n, n), dtype=torch.float64).pin_memory()
pol = pk.BasePolicy.naive_cutoff(cut)
da, db = ha.cuda(), hb.cuda()
dc = pk.Matrix.zeros(n, n, device="cuda")


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t_dev = timed(lambda: pk.winograd_block_mul(pk.Matrix(da), pk.Matrix(db), dc, pol))
t_e2e = timed(lambda: pk.winograd_block_mul(pk.Matrix(ha.numpy()), pk.Matrix(hb.numpy()), pk.Matrix(hc.numpy()), pol))
path = pk.last_stats().path
diff = float((hc - dc.arr.cpu()).abs().max())
f = 2 * n ** 3 / 1e9
print(json.dumps({"n": n, "cutoff": cut, "device_ms": round(t_dev, 2), "device_tflops": round(f / t_dev, 2),
                  "e2e_ms": round(t_e2e, 2), "e2e_tflops": round(f / t_e2e, 2), "path": path, "maxdiff": diff}))
