"""Probe (build: tools/build_variant.py cowork -DMK_COWORK_PROBE): a long narrow-tile mk_dgemm
alone, the same with an HBM-bound elementwise job (c = a +/- b) streamed by the leaf kernel's idle
producer warps, and the job alone through mk_block_combine -- DMMA slowdown vs side bandwidth."""
import ctypes, json, os, sys
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.environ.get("MK_LIB") or os.path.join(HERE, "..", "paper_2309_00628_b200", "libmk_strassen.so"))
I64, VP = ctypes.c_int64, ctypes.c_void_p
st = lambda: VP(torch.cuda.current_stream().cuda_stream)  # noqa: E731
M, N, K = 148 * 128, 320, 14016
a = torch.rand(M, K, device="cuda", dtype=torch.float64)
b = torch.rand(K, N, device="cuda", dtype=torch.float64)
c = torch.empty(M, N, device="cuda", dtype=torch.float64)
flops = 2.0 * M * N * K


def gemm():
    assert lib.mk_dgemm(VP(a.data_ptr()), I64(K), VP(b.data_ptr()), I64(N), VP(c.data_ptr()), I64(N),
                        I64(M), I64(N), I64(K), st()) == 0


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
pass
t0 = timed(gemm)
out["gemm_alone_ms"] = round(t0, 3)
out["gemm_alone_tflops"] = round(flops / t0 / 1e9, 2)
# main-loop rate of the two layouts (long K) and the per-tile cost at cfg5's K (438)
for (m, n, k, label) in ((148 * 128, 320, 14016, "narrow_longK"), (148 * 128, 384, 14016, "wide_longK"),
                         (148 * 128 * 4, 320, 438, "narrow_K438_20waves"), (148 * 128 * 4, 320, 448, "narrow_K448_20waves"),
                         (148 * 128 * 4, 384, 448, "wide_K448_12waves")):
    aa = torch.rand(m, k, device="cuda", dtype=torch.float64)
    bb = torch.rand(k, n, device="cuda", dtype=torch.float64)
    cc = torch.empty(m, n, device="cuda", dtype=torch.float64)
    f = lambda: lib.mk_dgemm(VP(aa.data_ptr()), I64(k), VP(bb.data_ptr()), I64(n), VP(cc.data_ptr()), I64(n),  # noqa: E731
                             I64(m), I64(n), I64(k), st())
    t = timed(f)
    out[label] = {"ms": round(t, 3), "tflops": round(2.0 * m * n * k / t / 1e9, 2)}
    del aa, bb, cc
print(json.dumps(out), flush=True)
