"""Randomised correctness sweep (dev tool, not part of the suite): many shapes / presets /
cutoffs / operand placements / entry points, integer data, exact against numpy."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2309_00628_b200 as pk

r = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 400
presets = pk.preset_names()
fns = {"strassen": pk.strassen_mul, "winograd-block": pk.winograd_block_mul, "winograd-knuth": pk.winograd_knuth_mul,
       "two-temp": pk.two_temp_winograd, "in-place": pk.in_place_winograd}
t0 = time.time()
fails = 0
for case in range(N):
    kind = r.integers(0, 3)
    try:
        if kind == 0:  # rectangular multiply
            m, k, n = (int(x) for x in r.integers(1, 1500, 3))
            spec = pk.get_variant(presets[int(r.integers(0, len(presets)))], cutoff=int(r.choice([8, 32, 64, 100, 128, 256])))
            a = r.integers(-8, 9, (m, k)).astype(np.float64); b = r.integers(-8, 9, (k, n)).astype(np.float64)
            dev = bool(r.integers(0, 2))
            A = pk.Matrix(torch.from_numpy(a).cuda()) if dev else pk.Matrix(a)
            B = pk.Matrix(torch.from_numpy(b).cuda()) if dev else pk.Matrix(b)
            got = pk.multiply(A, B, spec).numpy()
            want = a @ b
            tag = ("multiply", m, k, n, spec.kernel, dev)
        else:  # square entry points on (possibly windowed) views
            n = int(2 ** r.integers(0, 11))
            name = list(fns)[int(r.integers(0, len(fns)))]
            pol = pk.BasePolicy.naive_cutoff(int(r.choice([1, 2, 8, 32, 64, 128, 512])))
            pad = int(r.integers(0, 5))
            big = [r.integers(-8, 9, (n + 2 * pad, n + 3 * pad)).astype(np.float64) for _ in range(3)]
            dev = kind == 2
            mats = [pk.Matrix(torch.from_numpy(x).cuda()) if dev else pk.Matrix(x) for x in big]
            views = [pk.MatrixView(mm, pad, 2 * pad, n, n) for mm in mats]
            a = big[0][pad:pad + n, 2 * pad:2 * pad + n].copy(); b = big[1][pad:pad + n, 2 * pad:2 * pad + n].copy()
            fns[name](views[0], views[1], views[2], pol)
            c = mats[2].numpy() if dev else big[2]
            got = c[pad:pad + n, 2 * pad:2 * pad + n]
            want = a @ b
            tag = (name, n, pad, dev)
        if not np.array_equal(got, want):
            fails += 1
            print("MISMATCH", case, tag, float(np.abs(got - want).max()), flush=True)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print("ERROR", case, type(e).__name__, e, flush=True)
print(f"fuzz: {N} cases, {fails} failures, {time.time() - t0:.1f} s", flush=True)
