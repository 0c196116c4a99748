"""Per-CTA timeline of the leaf kernel (trace build, tools/build_trace.py): fill latency, main
loop, epilogue and the gap between consecutive CTAs on an SM. Dev tool."""
import ctypes, json, os, statistics, sys
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libmk_trace.so"))
I64, VP = ctypes.c_int64, ctypes.c_void_p
SM = torch.cuda.get_device_properties(0).multi_processor_count


def run(M, N, K, label):
    a = torch.randn(M, K, device="cuda", dtype=torch.float64)
    b = torch.randn(K, N, device="cuda", dtype=torch.float64)
    c = torch.empty(M, N, device="cuda", dtype=torch.float64)
    st = VP(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        assert lib.mk_dgemm(VP(a.data_ptr()), I64(K), VP(b.data_ptr()), I64(N), VP(c.data_ptr()), I64(N),
                            I64(M), I64(N), I64(K), st) == 0
    torch.cuda.synchronize()
    ntiles = ((M + 127) // 128) * ((N + 127) // 128)
    buf = (ctypes.c_ulonglong * (5 * ntiles))()
    assert lib.mk_trace_read(buf, ntiles) == 0
    rows = [tuple(buf[5 * i:5 * i + 5]) for i in range(ntiles)]
    t0 = min(r[1] for r in rows)
    fill = [r[2] - r[1] for r in rows]
    loop = [r[3] - r[2] for r in rows]
    epi = [r[4] - r[3] for r in rows]
    by_sm = {}
    for r in rows:
        by_sm.setdefault(r[0], []).append(r)
    gaps = []
    for v in by_sm.values():
        v.sort(key=lambda r: r[1])
        gaps += [v[i + 1][1] - v[i][4] for i in range(len(v) - 1)]
    end = max(r[4] for r in rows)
    med = lambda x: statistics.median(x) / 1e3 if x else None  # noqa: E731
    print(json.dumps({"case": label, "tiles": ntiles, "sms": len(by_sm), "span_us": (end - t0) / 1e3,
                      "fill_us": med(fill), "loop_us": med(loop), "epi_us": med(epi), "gap_us": med(gaps),
                      "first_entry_spread_us": (max(v[0][1] for v in by_sm.values()) - t0) / 1e3}))


run(SM * 128, 4 * 128, 4096, "4 waves K=4096")
run(SM * 128, 4 * 128, 512, "4 waves K=512")
run(4096, 4096, 4096, "4096^3 (6.9 waves)")
