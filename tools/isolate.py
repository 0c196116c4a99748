import subprocess, sys, json
cases = [("dgemm_like", 2, 256, 0), ("wb", 2, 256, 1), ("str", 1, 256, 1), ("str", 1, 2, 1), ("wb", 2, 2, 1), ("str", 1, 16, 1), ("wb", 2, 1024, 2), ("tt", 5, 256, 2), ("ip", 6, 256, 2)]
code = r'''
import sys, torch, ctypes
sys.path.insert(0, "tools")
import quick_gpu as q
algo, n, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = torch.randint(-8, 9, (n, n), device="cuda").double(); b = torch.randint(-8, 9, (n, n), device="cuda").double()
ref = a @ b; c = torch.full((n, n), float("nan"), dtype=torch.float64, device="cuda")
try:
    q.strassen(algo, a.clone(), b.clone(), c, L); torch.cuda.synchronize()
    print("OK maxerr", float((c - ref).abs().max()))
except Exception as e:
    print("ERR", str(e)[:300])
'''
for name, algo, n, L in cases:
    r = subprocess.run([sys.executable, "-c", code, str(algo), str(n), str(L)], capture_output=True, text=True, env={**__import__("os").environ, "MK_DEBUG_SYNC": "1"}, timeout=120)
    print(name, algo, n, L, "->", (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
