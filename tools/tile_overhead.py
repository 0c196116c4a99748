"""Per-tile fixed cost vs main-loop rate of the leaf kernel (through mk_dgemm): grids of exactly
148*w tiles (whole waves), K swept; time(K) = waves * (t0 + K/16 * t_stage). Dev tool."""
import sys
import torch
sys.path.insert(0, "tools")
import quick_gpu as q

torch.manual_seed(0)
SM = torch.cuda.get_device_properties(0).multi_processor_count
for waves in (1, 4):
    M, N = SM * 128, waves * 128
    rows = []
    for K in (256, 512, 1024, 2048, 4096, 8192, 16384):
        a = torch.randn(M, K, device="cuda", dtype=torch.float64)
        b = torch.randn(K, N, device="cuda", dtype=torch.float64)
        c = torch.empty(M, N, device="cuda", dtype=torch.float64)
        ms = q.timeit(lambda: q.dgemm(a, b, c), reps=10, warm=3)
        rows.append((K, ms))
        q.out(waves=waves, K=K, ms=round(ms, 4), tflops=round(2 * M * N * K / ms / 1e9, 2))
    # least squares on the two largest K: slope per stage, intercept per wave
    import numpy as np
    ks = np.array([r[0] for r in rows], float); ts = np.array([r[1] for r in rows])
    A = np.vstack([ks, np.ones_like(ks)]).T
    sl, ic = np.linalg.lstsq(A[2:], ts[2:], rcond=None)[0]
    flop_per_wave_per_k = 2 * M * N
    q.out(waves=waves, slope_ms_per_k=sl, intercept_ms=ic, intercept_us_per_wave=ic / waves * 1e3,
          mainloop_tflops=flop_per_wave_per_k / sl / 1e9)
