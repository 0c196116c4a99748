import sys, torch
sys.path.insert(0, ".")
import paper_2309_00628_b200 as pk
n = 16384
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
A, B, C = pk.Matrix(a), pk.Matrix(b), pk.Matrix.zeros(n, n, device="cuda")
for leaf in ("dmma", "ozaki"):
    pk.set_leaf(leaf, 8) if leaf == "ozaki" else pk.set_leaf("dmma")
    for name, fn in (("naive", lambda: pk.naive_mul(A, B, C)), ("wino L1", lambda: pk.winograd_block_mul(A, B, C, pk.BasePolicy.naive_cutoff(8192)))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); fn(); e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 2
        print(leaf, name, round(t, 2), "ms", round(2 * n ** 3 / t / 1e9, 1), "TF/s", flush=True)
