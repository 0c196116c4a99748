"""cfg5 (12000x14000 . 14000x10000, winograd-block cutoff 512) through multiply() with plain numpy
host arrays: staged copies vs torch's pageable copies. Dev tool."""
import json, sys, time, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk
from paper_2309_00628_b200 import device
rng = np.random.default_rng(20240901)
a = rng.uniform(-1, 1, (12000, 14000)); b = rng.uniform(-1, 1, (14000, 10000))
spec = pk.VariantSpec("winograd-block", pk.BasePolicy.naive_cutoff(512))
for label, thr in (("staged", 8 << 20), ("torch", 1 << 62)):
    device._STAGED_MIN_BYTES = thr
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        c = pk.multiply(pk.Matrix(a), pk.Matrix(b), spec)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(json.dumps({"copies": label, "rep": rep, "ms": round(t * 1e3, 1), "eff_tflops": round(2 * 12000 * 14000 * 10000 / t / 1e12, 2)}), flush=True)
