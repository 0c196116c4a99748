"""Quick GPU bring-up check of libmk_strassen.so through its C ABI (ctypes + torch memory).

Correctness vs torch's fp64 matmul (exact on integer-valued inputs) across algorithms and
level counts, then CUDA-event timings. Dev tool; the real tests live in tests/.
"""
import ctypes
import json
import os
import sys
import time

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.environ.get("MK_LIB") or os.path.join(HERE, "..", "paper_2309_00628_b200", "libmk_strassen.so"))
lib.mk_last_error.restype = ctypes.c_char_p
lib.mk_workspace_bytes.restype = ctypes.c_size_t
lib.mk_rect_workspace_bytes.restype = ctypes.c_size_t
I64, VP = ctypes.c_int64, ctypes.c_void_p


def stream():
    return VP(torch.cuda.current_stream().cuda_stream)


def dgemm(a, b, c):
    m, k = a.shape
    n = b.shape[1]
    rc = lib.mk_dgemm(VP(a.data_ptr()), I64(a.stride(0)), VP(b.data_ptr()), I64(b.stride(0)),
                      VP(c.data_ptr()), I64(c.stride(0)), I64(m), I64(n), I64(k), stream())
    if rc:
        raise RuntimeError(f"mk_dgemm rc={rc}: {lib.mk_last_error().decode()}")


def strassen(algo, a, b, c, levels):
    n = a.shape[0]
    ws_bytes = lib.mk_workspace_bytes(algo, I64(n), levels)
    ws = torch.empty(max(ws_bytes, 8), dtype=torch.uint8, device="cuda")
    rc = lib.mk_strassen(algo, VP(a.data_ptr()), I64(a.stride(0)), VP(b.data_ptr()), I64(b.stride(0)),
                         VP(c.data_ptr()), I64(c.stride(0)), I64(n), levels, VP(ws.data_ptr()),
                         ctypes.c_size_t(ws_bytes), stream())
    if rc:
        raise RuntimeError(f"mk_strassen rc={rc}: {lib.mk_last_error().decode()}")
    return ws_bytes


def timeit(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def out(**kw):
    print(json.dumps(kw), flush=True)


def main():
    torch.manual_seed(0)
    fuse = int(os.environ.get("MK_FUSE", "0"))
    lib.mk_set_option(1, fuse)
    out(mode="fuse_preadds" if fuse else "materialised_preadds")
    dev = "cuda"
    # ---- correctness: dgemm, integer-valued, odd shapes ----
    for (m, n, k) in [(8, 8, 4), (128, 128, 16), (256, 256, 256), (1000, 777, 555), (130, 3, 17), (1, 1, 1)]:
        a = torch.randint(-8, 9, (m, k + (k % 2)), device=dev).double()[:, :k]
        b = torch.randint(-8, 9, (k, n + (n % 2)), device=dev).double()[:, :n]
        c = torch.full((m, n), float("nan"), dtype=torch.float64, device=dev)
        dgemm(a, b, c)
        torch.cuda.synchronize()
        ref = a @ b
        out(check="dgemm", m=m, n=n, k=k, maxerr=float((c - ref).abs().max()))
    # ---- correctness: algorithms x levels on integer data ----
    names = {1: "strassen", 2: "winograd_block", 3: "winograd_knuth", 4: "knuth8", 5: "two_temp", 6: "in_place"}
    for n, levels in [(4, 1), (16, 1), (16, 3), (64, 3), (256, 1), (256, 2), (1024, 1), (1024, 2), (1024, 3), (512, 4)][: (99 if not os.environ.get("MK_QUICK") else 0)]:
        a = torch.randint(-8, 9, (n, n), device=dev).double()
        b = torch.randint(-8, 9, (n, n), device=dev).double()
        ref = a @ b
        for algo in range(1, 7):
            aa, bb = a.clone(), b.clone()
            c = torch.full((n, n), float("nan"), dtype=torch.float64, device=dev)
            try:
                ws = strassen(algo, aa, bb, c, levels)
                torch.cuda.synchronize()
                err = float((c - ref).abs().max())
                clob = bool((aa != a).any()) if algo == 6 else None
                out(check=names[algo], n=n, levels=levels, maxerr=err, ws_bytes=ws, a_clobbered=clob)
            except Exception as e:  # noqa: BLE001
                out(check=names[algo], n=n, levels=levels, error=str(e))
    # float accuracy
    n = 2048
    a = torch.rand(n, n, device=dev, dtype=torch.float64) * 2 - 1
    b = torch.rand(n, n, device=dev, dtype=torch.float64) * 2 - 1
    ref = a @ b
    for algo in (0, 2):
        c = torch.empty_like(a)
        if algo == 0:
            dgemm(a, b, c)
        else:
            strassen(algo, a, b, c, 2)
        torch.cuda.synchronize()
        out(check="float", algo=algo, n=n, maxerr=float((c - ref).abs().max()))
    # ---- timing ----
    # rectangular cfg5 and small-leaf plans
    m_, k_, n_ = 12000, 14000, 10000
    a = torch.rand(m_, k_, device=dev, dtype=torch.float64) * 2 - 1
    b = torch.rand(k_, n_, device=dev, dtype=torch.float64) * 2 - 1
    c = torch.empty(m_, n_, device=dev, dtype=torch.float64)
    ref = a @ b
    for L in (1, 2, 3, 5):
        ws_b = lib.mk_rect_workspace_bytes(2, I64(m_), I64(n_), I64(k_), L)
        ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device=dev)
        def run():
            rc = lib.mk_multiply_rect(2, VP(a.data_ptr()), I64(k_), VP(b.data_ptr()), I64(n_), VP(c.data_ptr()),
                                      I64(n_), I64(m_), I64(n_), I64(k_), L, VP(ws.data_ptr()), ctypes.c_size_t(ws_b),
                                      stream())
            if rc:
                raise RuntimeError(lib.mk_last_error().decode())
        ms = timeit(run, reps=2)
        out(time="rect_cfg5", levels=L, ms=round(ms, 3), eff_tflops=round(2 * m_ * n_ * k_ / ms / 1e9, 3),
            maxerr=float((c - ref).abs().max()), ws_gib=round(ws_b / 2**30, 2))
    del a, b, c, ref
    for n in (8192, 16384):
        a = torch.randn(n, n, device=dev, dtype=torch.float64)
        b = torch.randn(n, n, device=dev, dtype=torch.float64)
        c = torch.empty_like(a)
        ms = timeit(lambda: dgemm(a, b, c), reps=2 if n == 16384 else 3)
        out(time="mk_dgemm", n=n, ms=round(ms, 3), tflops=round(2 * n**3 / ms / 1e9, 3))
        ms = timeit(lambda: torch.matmul(a, b, out=c), reps=2 if n == 16384 else 3)
        out(time="cublas", n=n, ms=round(ms, 3), tflops=round(2 * n**3 / ms / 1e9, 3))
        for algo in (2, 1, 5, 6):
            for levels in ((1, 2, 3) if n == 8192 else (1, 2)):
                if algo == 6:  # in-place clobbers: give it copies
                    a2, b2 = a.clone(), b.clone()
                    ms = timeit(lambda: strassen(algo, a2, b2, c, levels), reps=2)
                    L = levels
                    out(time=names[algo], n=n, levels=L, ms=round(ms, 3), eff_tflops=round(2 * n**3 / ms / 1e9, 3))
                    continue
                ms = timeit(lambda: strassen(algo, a, b, c, levels), reps=2)
                L = levels
                n0 = n >> L
                actual = 7**L * 2 * n0**3
                out(time=names[algo], n=n, levels=L, ms=round(ms, 3), eff_tflops=round(2 * n**3 / ms / 1e9, 3),
                    actual_tflops=round(actual / ms / 1e9, 3))


if __name__ == "__main__":
    main()
