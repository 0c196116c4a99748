"""Ozaki-scheme INT8 tensor-core FP64 product (mk_ozaki_dgemm): exactness, accuracy, speed.

Run on the B200:  python tools/ozaki_probe.py [--quick]
"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_00628_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def oz(a, b, slices, c=None):
    m, k = a.shape
    n = b.shape[1]
    if c is None:
        c = torch.empty((m, n), dtype=torch.float64, device=dev)
    wsb = lib.mk_ozaki_workspace_bytes(m, n, k, slices)
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device=dev)
    rc = lib.mk_ozaki_dgemm(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0),
                            m, n, k, slices, ws.data_ptr(), wsb, st)
    if rc:
        raise RuntimeError(lib.mk_last_error().decode())
    return c


def dg(a, b, c=None):
    m, k = a.shape
    n = b.shape[1]
    if c is None:
        c = torch.empty((m, n), dtype=torch.float64, device=dev)
    rc = lib.mk_dgemm(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0), m, n, k, st)
    if rc:
        raise RuntimeError(lib.mk_last_error().decode())
    return c


def main():
    rng = np.random.default_rng(20240901)
    # 1. exactness on integer data (the reference's [-8, 8] fixtures), ragged shapes
    for (m, n, k) in [(128, 64, 32), (256, 256, 256), (300, 200, 260), (1000, 1030, 1017), (64, 64, 1)]:
        a = torch.from_numpy(rng.integers(-8, 9, (m, k)).astype(np.float64)).to(dev)
        b = torch.from_numpy(rng.integers(-8, 9, (k, n)).astype(np.float64)).to(dev)
        ref = a @ b
        for s in (4, 8):
            c = oz(a, b, s)
            torch.cuda.synchronize()
            bad = (c != ref).sum().item()
            print(f"int m={m} n={n} k={k} S={s}: mismatches {bad}  max|d| {(c - ref).abs().max().item():.3g}",
                  flush=True)
    # 2. accuracy on reals against an extended-precision reference
    n = 512
    for dist in ("uniform", "normal"):
        an = rng.uniform(-1, 1, (n, n)) if dist == "uniform" else rng.standard_normal((n, n))
        bn = rng.uniform(-1, 1, (n, n)) if dist == "uniform" else rng.standard_normal((n, n))
        exact = np.matmul(an.astype(np.longdouble), bn.astype(np.longdouble))
        a, b = torch.from_numpy(an).to(dev), torch.from_numpy(bn).to(dev)
        scale = np.abs(an).max() * np.abs(bn).max()
        res = {"dmma": dg(a, b), "cublas": a @ b, "numpy": None}
        for s in (5, 6, 7, 8):
            res[f"oz{s}"] = oz(a, b, s)
        torch.cuda.synchronize()
        for name, c in res.items():
            cn = np.matmul(an, bn) if c is None else c.cpu().numpy()
            err = np.abs(cn.astype(np.longdouble) - exact).max()
            print(f"{dist} n={n} {name:7s} max err {float(err):.3e}  / (u|A||B|) {float(err) / (2**-53 * scale):.1f}",
                  flush=True)
    if "--quick" in sys.argv:
        return
    # 3. speed
    for n in (4096, 8192, 16384):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        c = torch.empty(n, n, dtype=torch.float64, device=dev)
        fl = 2.0 * n ** 3

        def timeit(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps

        t = timeit(lambda: dg(a, b, c))
        print(f"n={n} dmma {t:.2f} ms {fl / t / 1e9:.1f} TF/s", flush=True)
        for s in (6, 7, 8):
            t = timeit(lambda: oz(a, b, s, c))
            pairs = s * (s + 1) // 2
            print(f"n={n} ozaki S={s} {t:.2f} ms {fl / t / 1e9:.1f} TF/s (FP64-equivalent); "
                  f"int8 {pairs * fl / t / 1e12:.2f} POP/s", flush=True)


if __name__ == "__main__":
    main()
