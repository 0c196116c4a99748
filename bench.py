"""Benchmark: effective FP64 TFLOP/s (2 n^3 / t) of Strassen-Winograd on B200.

Workload (BASELINE.json config 4, the north-star target): n = 16384, A and B standard
normal from np.random.default_rng(20240901) (A then B), winograd-block with
naive_cutoff(4096) -> 2 recursion levels, 49 DMMA leaf GEMMs of 4096^3. One "step" is one
full multiplication C = A B. Inputs (2 GiB each) exceed the 126 MB L2, so no L2 flush is
needed between steps.

  python bench.py [--gpus N --steps K --warmup W]   # our engine; N > 1 self-launches N ranks
  python bench.py --impl reference [...]            # the reference CPU path (oracle port)

value     = whole-job 2n^3 / t, inputs resident in HBM, CUDA events, max over ranks.
e2e       = the same metric through the public API with pinned HOST buffers: per step
            H2D of A and B, the product, D2H of C.
roofline  = the dominant kernel (DMMA leaf product): algorithmic flops per launch /
            CUDA-event launch time inside the timed region, against the FP64 tensor roofline
            measured in the same run by a DMMA-only microbenchmark (mk_fp64_peak).
cpu_baseline / --impl reference = the oracle (numpy restatement of the reference, bit-identical
            to it: tests/test_oracle_golden.py) on the host cores at the SAME configuration
            (n = 16384, naive_cutoff(4096)), one full product per step.
legs      = (N = 1) BASELINE cfg3 (n = 8192, 3 levels), cfg5 (12000x14000 . 14000x10000,
            cutoff 512, 5 levels), cuBLAS DGEMM (torch.matmul, comparison only), the memory-lean
            plans, other cutoffs and the opt-in INT8 (Ozaki) leaf.
N > 1     = strong scaling of one product: the 49 leaves, split into 8 row panels each, sharded
            evenly over ranks; partial C sum-reduced to rank 0 over NVLink (NCCL). Reported
            beside it: compute and exchange time, exchange bytes against the measured peer
            bandwidth, the fused reduce-scatter leg, and an e2e leg whose A and B start on GPU 0
            (subgroup broadcasts of only the quadrants each rank reads) and whose C ends there.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective FP64 TFLOP/s (2n^3/t) of Strassen-Winograd, n={n}"
UNIT = "TFLOP/s"
PEER_GBS = 770.0  # measured NVLink peer copy per direction per GPU (B200_PROFILING.md)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--order", dest="n", type=int, default=16384)
    p.add_argument("--cutoff", type=int, default=4096)
    p.add_argument("--algo", default="winograd-block")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only for 1-GPU plumbing checks")
    p.add_argument("--fused-reduce", action="store_true",
                   help="N > 1: headline uses the fused reduce-scatter (leaf epilogues add into the owning "
                        "rank's C row slab over peer memory) instead of partial C + NCCL reduce")
    p.add_argument("--alt", default="8192,2048", help="extra cutoffs to report (comma list, '' for none)")
    p.add_argument("--legs", default="cfg3,cfg5,cublas,lean",
                   help="extra N=1 legs (comma list of cfg3, cfg5, cublas, lean; '' for none)")
    p.add_argument("--ozaki-slices", type=int, default=8,
                   help="also time the same workload with INT8 tensor-core (Ozaki) leaves, 0 = skip")
    return p.parse_args()


def config(args, levels, world=1):
    c = {
        "workload": f"BASELINE cfg4: n={args.n} standard-normal FP64, {args.algo}, naive_cutoff({args.cutoff}) "
                    f"-> {levels} levels ({7 ** levels} DMMA leaf GEMMs)",
        "n": args.n, "cutoff": args.cutoff, "levels": levels, "algo": args.algo,
        "l2": (f"inputs {args.n * args.n * 8 / 2 ** 30:g} GiB each > 126 MB L2 (no flush needed)"
               if args.n * args.n * 8 > 126e6 else "inputs fit in L2 (non-default order: no flush between steps)"),
    }
    if world > 1:
        c["parallelism"] = (f"leaf row panels over {world} ranks; " +
                            ("fused reduce-scatter into owner row slabs over peer memory, slabs pulled to rank 0"
                             if args.fused_reduce else "partial C per rank + NCCL reduce to rank 0"))
    return c


def levels_for(n, cutoff):
    lv = 0
    while n > cutoff and n > 1:
        n //= 2
        lv += 1
    return lv


def actual_flops(n, levels, algo):
    """Flops the algorithm executes: 7^L leaf GEMMs + the block additions of every level."""
    adds = {"strassen": 18, "winograd-block": 15, "winograd-knuth": 16}.get(algo, 15)
    n0 = n >> levels
    f = 7 ** levels * 2.0 * n0 ** 3
    for lvl in range(levels):
        f += adds * 7 ** lvl * (n >> (lvl + 1)) ** 2
    return f


def rect_actual_flops(m, n, k, levels, algo="winograd-block"):
    """Same for the engine's rectangular recursion (mk_multiply_rect pads m, k to multiples of
    2^(L+1) and n to 2^(L+2)). Block additions per node: A side / B side / post-additions =
    4 / 4 / 7 for winograd-block (kernels.py:96-119), 5 / 5 / 8 for strassen (kernels.py:66-92)."""
    ra, rb, rc = {"strassen": (5, 5, 8)}.get(algo, (4, 4, 7))
    mp = -(-m // (2 << levels)) * (2 << levels)
    kp = -(-k // (2 << levels)) * (2 << levels)
    np_ = -(-n // (4 << levels)) * (4 << levels)
    f = 7 ** levels * 2.0 * (mp >> levels) * (np_ >> levels) * (kp >> levels)
    for lvl in range(levels):
        s = lvl + 1
        f += 7 ** lvl * (ra * (mp >> s) * (kp >> s) + rb * (kp >> s) * (np_ >> s) + rc * (mp >> s) * (np_ >> s))
    return f


def tf(flops, ms):
    return flops / (ms * 1e-3) / 1e12


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"mk_clocks_{os.getpid()}.csv")
        self.skip = 0

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
            # let nvidia-smi finish starting up (NVML init) before the timed region begins: its
            # start-up must not land inside a timed step
            t0 = time.time()
            while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
                time.sleep(0.05)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def mark(self):
        """Start of the timed region: samples written before this are not summarised."""
        if self.proc is not None:
            self.fh.flush()
            self.skip = os.path.getsize(self.path)

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            fh.seek(self.skip)
            lines = fh.read().splitlines()
        for line in lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        try:
            os.remove(self.path)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ----------------------------------------------------------------------------- CPU legs
def all_host_threads():
    """Context raising the BLAS pool to every host core: torchrun exports OMP_NUM_THREADS=1 to
    its ranks, and the reference's CPU path should still use the whole host."""
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")
    except Exception:  # pragma: no cover
        import contextlib

        return contextlib.nullcontext()


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"), default=1)
    except Exception:
        return os.cpu_count() or 1


def cpu_operands(n):
    """The workload's operands (cfg4 generator at order n): standard normal, A then B from one
    seeded generator -- shared by the GPU arm and the CPU legs."""
    from paper_2309_00628_b200.metrics import BASELINE_SEED

    rng = np.random.default_rng(BASELINE_SEED)
    return rng.standard_normal((n, n)), rng.standard_normal((n, n))


def cpu_product_seconds(a, b, cutoff, algo):
    """One oracle (reference restatement, bit-identical to it) product on the host."""
    from oracle import strassen_oracle as o

    kernel = algo if algo in o.TABLES else "winograd-block"
    t0 = time.perf_counter()
    o.product(kernel, a, b, o.policy("naive-cutoff", cutoff))
    return time.perf_counter() - t0


def cpu_sample_text(args, levels, cores, what):
    return (f"oracle (numpy restatement of matmulkit, bit-identical to it) {args.algo} n={args.n} "
            f"naive_cutoff({args.cutoff}) = the full {levels}-level workload ({7 ** levels} OpenBLAS leaves on "
            f"{cores} threads, block adds single-threaded as in the reference); {what}")


def cpu_baseline(args, levels):
    """One full product of the stated configuration on the host (rank 0, N = 1)."""
    a, b = cpu_operands(args.n)
    with all_host_threads():
        cpu_product_seconds(a[:512, :512].copy(), b[:512, :512].copy(), 128, args.algo)  # warm numpy/BLAS
        t = cpu_product_seconds(a, b, args.cutoff, args.algo)
        cores = blas_threads()
    return {
        "value": round(2.0 * args.n ** 3 / t / 1e12, 4), "unit": UNIT, "cores": cores, "kind": "port",
        "sample": cpu_sample_text(args, levels, cores, f"one product, {t:.2f} s"),
        "seconds": round(t, 3),
    }


def run_reference(args):
    """--impl reference: the reference's CPU path at the stated config, one full product per step.
    Warm-up: one product (a CPU run has no JIT or cache state beyond first-touch page faults,
    which the first product takes); the K timed steps follow."""
    levels = levels_for(args.n, args.cutoff)
    if int(os.environ.get("RANK", "0")) != 0:
        return
    a, b = cpu_operands(args.n)
    warm = min(args.warmup, 1)
    with all_host_threads():
        for _ in range(warm):
            cpu_product_seconds(a, b, args.cutoff, args.algo)
        ts = [cpu_product_seconds(a, b, args.cutoff, args.algo) for _ in range(args.steps)]
        cores = blas_threads()
    ms = 1e3 * sum(ts) / len(ts)
    value = tf(2.0 * args.n ** 3, ms)
    line = {
        "metric": METRIC.format(n=args.n), "value": round(value, 4), "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": warm, "warmup_requested": args.warmup,
        "ms_per_step": round(ms, 2), "higher_is_better": True,
        "step_ms": {"median": round(1e3 * statistics.median(ts), 2), "best": round(1e3 * min(ts), 2),
                    "worst": round(1e3 * max(ts), 2)},
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded standard normal)",
        "config": config(args, levels),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": cpu_sample_text(args, levels, cores, "one full product per step (host cores only)")},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- helpers
def event_timer(torch, stream):
    def timed(fn, reps=3, warm=1):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(reps):
            fn()
        g1.record(stream)
        torch.cuda.synchronize()
        return g0.elapsed_time(g1) / reps
    return timed


def step_stats(ms_list):
    return {"median": round(statistics.median(ms_list), 3), "best": round(min(ms_list), 3),
            "worst": round(max(ms_list), 3)}


# ----------------------------------------------------------------------------- Ozaki leg
def ozaki_leg(args, pk, lib, _lib, torch, A, B, C, dc, host_a, host_b, policy, stream, local):
    """The same workload with every leaf product on the INT8 tensor cores (Ozaki scheme I,
    set_leaf("ozaki", S)): value / e2e like the headline, the leaf launches' int8 roofline, and
    the max difference from the DMMA (FP64 tensor-core) result of the same inputs. Opt-in
    arithmetic beyond the north star's FP64 tensor-core leaf: never the headline."""
    n, S = args.n, args.ozaki_slices
    call = {"winograd-block": pk.winograd_block_mul, "strassen": pk.strassen_mul,
            "winograd-knuth": pk.winograd_knuth_mul}[args.algo]
    pk.set_leaf("dmma")
    call(A, B, C, policy)
    ref = dc.clone()
    timed = event_timer(torch, stream)
    try:
        pk.set_leaf("ozaki", S)
        with ClockSampler(local) as clk:
            for _ in range(max(args.warmup, 3)):
                call(A, B, C, policy)
            torch.cuda.synchronize()
            clk.mark()
            _lib.check(lib.mk_timing_begin(), "mk_timing_begin")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
            e0.record(stream)
            for i in range(args.steps):
                call(A, B, C, policy)
                if i < args.steps - 1:
                    marks[i].record(stream)
            e1.record(stream)
            torch.cuda.synchronize()
        kms, kcnt, kfl = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
        _lib.check(lib.mk_timing_end(ctypes.byref(kms), ctypes.byref(kcnt), ctypes.byref(kfl)), "mk_timing_end")
        ms = e0.elapsed_time(e1) / args.steps
        bounds = [e0] + marks + [e1]
        step_ms = [bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps)]
        diff = float((dc - ref).abs().max())
        scale = float(torch.linalg.vector_norm(ref, ord=float("inf")))
        host_c = torch.empty((n, n), dtype=torch.float64).pin_memory()
        hA, hB, hC = pk.Matrix(host_a.numpy()), pk.Matrix(host_b.numpy()), pk.Matrix(host_c.numpy())
        ems = timed(lambda: call(hA, hB, hC, policy), reps=args.steps)
        alts = []
        for cut in [int(x) for x in args.alt.split(",") if x]:  # same extra cutoffs as the DMMA leg
            pol = pk.BasePolicy.naive_cutoff(cut)
            ams = timed(lambda: call(A, B, C, pol), reps=3, warm=2)
            alts.append({"cutoff": cut, "levels": levels_for(n, cut), "ms_per_step": round(ams, 3),
                         "value": round(tf(2.0 * n ** 3, ams), 4)})
    finally:
        pk.set_leaf("dmma")
    pairs = S * (S + 1) // 2
    peak, src = 4500.0, "nominal 4500 TOPS dense INT8 (B200 datasheet)"
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        if mp.get("bf16_tflops"):
            peak = 2.0 * float(mp["bf16_tflops"])
            src = "2 x MEASURED_PEAKS.json bf16_tflops (burst; the tensor pipe's 8-bit rate is twice its 16-bit rate)"
    except Exception:
        pass
    achieved = pairs * kfl.value / (kms.value * 1e-3) / 1e12 if kms.value > 0 else None
    lv = levels_for(n, args.cutoff)
    return {
        "slices": S, "digit_bits": 7 + 8 * (S - 1), "int8_products_per_leaf": pairs,
        "extra_workspace_bytes": 2 * int(lib.mk_ozaki_workspace_bytes(n >> lv, n >> lv, n >> lv, S)),
        "value": round(tf(2.0 * n ** 3, ms), 4), "unit": UNIT, "ms_per_step": round(ms, 3),
        "step_ms": step_stats(step_ms),
        "e2e": {"value": round(tf(2.0 * n ** 3, ems), 4), "unit": UNIT, "ms_per_step": round(ems, 2),
                "h2d_bytes_per_step": 2 * n * n * 8, "d2h_bytes_per_step": n * n * 8},
        "max_abs_diff_vs_dmma_result": diff, "result_max_abs": scale,
        "roofline": {"bound": "tensor", "achieved": round(achieved, 1) if achieved else None, "peak": round(peak, 1),
                     "unit": "TOPS (int8)", "frac": round(achieved / peak, 4) if achieved else None,
                     "kernel": "mk::oz::ozaki_product_kernel + digit splitting (per leaf, CUDA events)",
                     "peak_source": src},
        "clocks": clk.summary(),
        "alt_cutoffs": alts,
        "dtype": "f64 operands/results; int8 x int8 -> int32 tensor-core products (Ozaki scheme I)",
    }


# ----------------------------------------------------------------------------- N = 1 legs
def baseline_legs(args, pk, lib, _lib, torch, stream, peak_tflops, legs):
    """BASELINE cfg3 and cfg5 on their seeded inputs, and cuBLAS DGEMM as a comparison point
    (torch.matmul on FP64 CUDA tensors; never on the product path)."""
    from paper_2309_00628_b200.metrics import baseline_operands

    timed = event_timer(torch, stream)
    out = {}
    if "cfg3" in legs:
        a, b = baseline_operands(3)
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        c = torch.empty_like(da)
        pol = pk.BasePolicy.naive_cutoff(1024)
        fn = lambda: pk.winograd_block_mul(pk.Matrix(da), pk.Matrix(db), pk.Matrix(c), pol)  # noqa: E731
        ms = timed(fn, reps=5, warm=3)
        f_act = actual_flops(8192, 3, "winograd-block")
        out["cfg3"] = {"workload": "BASELINE cfg3: n=8192 uniform[-1,1), winograd-block, naive_cutoff(1024) -> 3 levels "
                                   "(343 leaves of 1024^3)",
                       "ms_per_step": round(ms, 3), "value": round(tf(2.0 * 8192 ** 3, ms), 4),
                       "actual_tflops": round(tf(f_act, ms), 4), "frac_of_fp64_peak_actual": round(tf(f_act, ms) / peak_tflops, 4),
                       "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS["winograd-block"], 8192, 3))}
        a2, b2 = da.clone(), db.clone()
        ms_ip = timed(lambda: pk.in_place_winograd(pk.Matrix(a2), pk.Matrix(b2), pk.Matrix(c), pol), reps=3, warm=1)
        out["cfg3"]["in_place"] = {"ms_per_step": round(ms_ip, 3), "value": round(tf(2.0 * 8192 ** 3, ms_ip), 4),
                                   "workspace_bytes": 0}
        ms_tt = timed(lambda: pk.two_temp_winograd(pk.Matrix(da), pk.Matrix(db), pk.Matrix(c), pol), reps=3, warm=1)
        out["cfg3"]["two_temp"] = {"ms_per_step": round(ms_tt, 3), "value": round(tf(2.0 * 8192 ** 3, ms_tt), 4),
                                   "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS["two-temp"], 8192, 3))}
        del da, db, c, a2, b2
        torch.cuda.empty_cache()
    if "cfg5" in legs:
        a, b = baseline_operands(5)
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        m, k = a.shape
        n = b.shape[1]
        spec = pk.VariantSpec("winograd-block", pk.BasePolicy.naive_cutoff(512))
        fn = lambda: pk.multiply(pk.Matrix(da), pk.Matrix(db), spec)  # noqa: E731
        ms = timed(fn, reps=5, warm=3)
        lv = pk.last_stats().levels
        f_act = rect_actual_flops(m, n, k, lv)
        out["cfg5"] = {"workload": "BASELINE cfg5: 12000x14000 . 14000x10000 uniform[-1,1), multiply(winograd-block, "
                                   f"naive_cutoff(512)) -> {lv} levels on even-quadrant padding",
                       "ms_per_step": round(ms, 3), "value": round(tf(2.0 * m * n * k, ms), 4), "levels": lv,
                       "actual_tflops": round(tf(f_act, ms), 4), "frac_of_fp64_peak_actual": round(tf(f_act, ms) / peak_tflops, 4),
                       "workspace_bytes": int(pk.last_stats().workspace_bytes)}
        del da, db
        torch.cuda.empty_cache()
    if "cublas" in legs:
        res = {}
        for nn in (8192, 16384):
            x = torch.randn((nn, nn), dtype=torch.float64, device="cuda")
            y = torch.randn((nn, nn), dtype=torch.float64, device="cuda")
            z = torch.empty_like(x)
            ms = timed(lambda: torch.matmul(x, y, out=z), reps=3, warm=2)
            dmma = timed(lambda: pk.naive_mul(pk.Matrix(x), pk.Matrix(y), pk.Matrix(z)), reps=3, warm=2)
            res[str(nn)] = {"cublas_dgemm_ms": round(ms, 3), "cublas_dgemm_tflops": round(tf(2.0 * nn ** 3, ms), 4),
                            "mk_dgemm_ms": round(dmma, 3), "mk_dgemm_tflops": round(tf(2.0 * nn ** 3, dmma), 4)}
            del x, y, z
        torch.cuda.empty_cache()
        out["cublas_dgemm"] = {"note": "torch.matmul FP64 (cuBLAS DGEMM) as a comparison point only; mk_dgemm = our "
                                       "naive_mul leaf kernel", **res}
    return out


# ----------------------------------------------------------------------------- N > 1 helpers
class Multi:
    """Sharded product pieces for N ranks: NCCL reduce of partial C (headline), the fused
    reduce-scatter leg, and the GPU-0-resident e2e leg with subgroup broadcasts."""

    def __init__(self, args, torch, dist, multigpu, world, rank, dev, levels):
        self.args, self.torch, self.dist, self.mg = args, torch, dist, multigpu
        self.world, self.rank, self.dev, self.levels = world, rank, dev, levels
        self.gloo = args.dist_backend == "gloo"
        total = multigpu.leaf_count(args.algo, levels) * multigpu.PANELS
        self.first, self.count = multigpu.shard_range(total, world, rank)
        # quadrant subgroups for the GPU-0 e2e leg: the ranks whose units read quadrant q of A (B)
        self.groups = {}
        for side in (0, 1):
            for q in range(4):
                members = [0]
                for r in range(world):
                    f, c = multigpu.shard_range(total, world, r)
                    qa, qb = multigpu.operand_quadrants(args.algo, levels, f, c)
                    if q in (qa if side == 0 else qb) and r != 0:
                        members.append(r)
                grp = dist.new_group(members) if len(members) > 1 else None  # every rank calls new_group
                self.groups[(side, q)] = (members, grp)

    def _collective(self, fn, t, *a, **kw):
        """gloo on one GPU (plumbing checks only): collectives on host copies."""
        if self.gloo and t.is_cuda:
            h = t.cpu()
            fn(h, *a, **kw)
            t.copy_(h)
        else:
            fn(t, *a, **kw)

    def reduce_step(self, da, db, dc, ws, ev=None):
        """This rank's leaf row panels into a zeroed partial C, then the reduce to rank 0."""
        dc.zero_()
        if self.count:
            self.mg.partial_product(self.args.algo, da, db, dc, self.levels, self.first, self.count, ws=ws)
        if ev is not None:
            ev.record(self.torch.cuda.current_stream())
        self._collective(self.dist.reduce, dc, dst=0, op=self.dist.ReduceOp.SUM)

    def broadcast_operands(self, da, db, stage):
        """A and B on GPU 0 -> every rank that reads a quadrant gets it (one broadcast per quadrant
        inside the subgroup of its readers). Quadrant views are strided, so they travel through a
        contiguous stage buffer."""
        n = da.shape[0]
        h = n // 2
        moved = 0
        for side, src in ((0, da), (1, db)):
            for q in range(4):
                members, grp = self.groups[(side, q)]
                if grp is None or self.rank not in members:
                    continue
                view = src[(q >> 1) * h:(q >> 1) * h + h, (q & 1) * h:(q & 1) * h + h]
                if self.rank == 0:
                    stage.copy_(view)
                self._collective(self.dist.broadcast, stage, src=0, group=grp)
                if self.rank != 0:
                    view.copy_(stage)
                    moved += h * h * 8
        return moved


def run_multi(args, pk, lib, _lib, torch, dist, multigpu, world, rank, local, levels, da, db, dc, host_a, host_b,
              clk_ctx):
    """N > 1: timed NCCL-reduce steps (headline) with compute / exchange split; fused leg; e2e legs."""
    n = args.n
    dev = da.device
    stream = torch.cuda.current_stream()
    need = int(lib.mk_partial_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels))
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    M = Multi(args, torch, dist, multigpu, world, rank, dev, levels)
    ex = multigpu.SlabExchange(n)

    def fused_step():
        multigpu.fused_sharded_multiply(args.algo, da, db, levels, ex, out=dc if rank == 0 else None, ws=ws)

    def barrier():
        dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        M._collective(dist.all_reduce, t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        t = torch.tensor([int(x)], dtype=torch.int64, device=dev)
        M._collective(dist.all_reduce, t, op=dist.ReduceOp.SUM)
        return int(t.item())

    headline_fused = args.fused_reduce
    res = {}
    with clk_ctx as clk:
        # ---- headline leg (NCCL reduce, or --fused-reduce)
        for _ in range(max(args.warmup, 3)):
            fused_step() if headline_fused else M.reduce_step(da, db, dc, ws)
        torch.cuda.synchronize()
        launches0 = lib.mk_launch_count()
        barrier()
        torch.cuda.synchronize()
        clk.mark()
        _lib.check(lib.mk_timing_begin(), "mk_timing_begin")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        e0.record(stream)
        for i in range(args.steps):
            if headline_fused:
                fused_step()
            else:
                M.reduce_step(da, db, dc, ws, ev=mids[i])
            marks[i].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    clocks = clk.summary()
    kms, kcnt, kfl = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
    _lib.check(lib.mk_timing_end(ctypes.byref(kms), ctypes.byref(kcnt), ctypes.byref(kfl)), "mk_timing_end")
    launches = lib.mk_launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    bounds = [e0] + marks
    step_ms = [bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps)]
    res["ms"] = max_over_ranks(ms)
    res["step_ms"] = step_stats(step_ms)
    res["launches"] = sum_over_ranks(launches)
    res["kernel"] = (kms.value, kcnt.value, kfl.value)
    res["clocks"] = clocks
    if not headline_fused:
        comp = [bounds[i].elapsed_time(mids[i]) for i in range(args.steps)]
        exch = [mids[i].elapsed_time(marks[i]) for i in range(args.steps)]
        res["compute_ms"] = max_over_ranks(statistics.median(comp))
        ex_med = statistics.median(exch)
        res["exchange_ms"] = max_over_ranks(ex_med)
        res["compute_ms_min_rank"] = -max_over_ranks(-statistics.median(comp))
    # ---- the other reduce leg (fused if the headline was NCCL, else NCCL)
    timed = event_timer(torch, stream)
    if headline_fused:
        other = timed(lambda: M.reduce_step(da, db, dc, ws), reps=3, warm=1)
        res["other_leg"] = {"exchange": "partial C + NCCL reduce", "ms_per_step": round(max_over_ranks(other), 3)}
    else:
        other = timed(fused_step, reps=3, warm=1)
        res["other_leg"] = {"exchange": "fused reduce-scatter (leaf epilogues add into the owner's row slab over "
                                        "CUDA-IPC peer memory; no partial C, no collective)",
                            "ms_per_step": round(max_over_ranks(other), 3)}
    res["other_leg"]["value"] = round(tf(2.0 * n ** 3, res["other_leg"]["ms_per_step"]), 4)
    barrier()
    # ---- e2e (headline): pinned host operands, each rank uploads the quadrants its shard reads
    if not args.no_e2e:
        host_c = torch.empty((n, n), dtype=torch.float64).pin_memory() if rank == 0 else None
        moved = [0]

        def e2e_step():
            moved[0] = multigpu.upload_operands(args.algo, levels, host_a, host_b, da, db)
            M.reduce_step(da, db, dc, ws)
            if rank == 0:
                host_c.copy_(dc, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        e2e_step()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1) / args.steps)
        res["e2e"] = {"value": round(tf(2.0 * n ** 3, ems), 4), "unit": UNIT,
                      "h2d_bytes_per_step": sum_over_ranks(moved[0]), "d2h_bytes_per_step": n * n * 8,
                      "ms_per_step": round(ems, 2),
                      "how": "pinned host A, B; every rank uploads only the operand quadrants its leaves read; "
                             "partial C NCCL-reduced to rank 0; C downloaded from GPU 0"}
        # ---- e2e from GPU 0: A and B resident on GPU 0 only, C ends on GPU 0
        h = n // 2
        stage = torch.empty((h, h), dtype=torch.float64, device=dev)
        bmoved = [0]

        def gpu0_step():
            bmoved[0] = M.broadcast_operands(da, db, stage)
            M.reduce_step(da, db, dc, ws)

        gpu0_step()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            gpu0_step()
        g1.record(stream)
        torch.cuda.synchronize()
        barrier()
        gms = max_over_ranks(g0.elapsed_time(g1) / args.steps)
        res["e2e_from_gpu0"] = {
            "value": round(tf(2.0 * n ** 3, gms), 4), "unit": UNIT, "ms_per_step": round(gms, 2),
            "broadcast_bytes_per_step": sum_over_ranks(bmoved[0]),
            "how": "A, B resident on GPU 0; one NCCL broadcast per operand quadrant inside the subgroup of the ranks "
                   "that read it; partial C NCCL-reduced to GPU 0 (C ends on GPU 0)"}
        del stage
    del ws
    return res


# ----------------------------------------------------------------------------- GPU arm
def self_launch(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-run this script as N ranks."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def nccl_env():
    """NCCL's init report (ranks, NVLS / channels) on stderr, keeping stdout for the JSON line."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and args.dist_backend == "nccl":
        nccl_env()

    import torch
    import torch.distributed as dist

    import paper_2309_00628_b200 as pk
    from paper_2309_00628_b200 import _lib, multigpu
    from paper_2309_00628_b200.device import require_engine

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    lib = require_engine()
    n = args.n
    levels = levels_for(n, args.cutoff)
    policy = pk.BasePolicy.naive_cutoff(args.cutoff)
    dev = torch.device("cuda", local)

    peak = ctypes.c_double(0.0)
    _lib.check(lib.mk_fp64_peak(ctypes.byref(peak), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "mk_fp64_peak")
    peak_tflops = float(peak.value)

    host_a, host_b = (torch.from_numpy(x).pin_memory() for x in cpu_operands(n))
    da, db = host_a.to(dev), host_b.to(dev)
    dc = torch.empty((n, n), dtype=torch.float64, device=dev)
    A, B, C = pk.Matrix(da), pk.Matrix(db), pk.Matrix(dc)
    stream = torch.cuda.current_stream()
    torch.cuda.reset_peak_memory_stats(dev)
    mem0 = torch.cuda.memory_allocated(dev)

    if world > 1:
        r = run_multi(args, pk, lib, _lib, torch, dist, multigpu, world, rank, local, levels, da, db, dc, host_a,
                      host_b, ClockSampler(local))
        peak_mem = torch.cuda.max_memory_allocated(dev) - mem0
        gpus_active = len({int(x) for x in _gather_devices(torch, dist, dev, args.dist_backend == "gloo")})
        dist.barrier()
        if rank != 0:
            dist.destroy_process_group()
            return
        ms = r["ms"]
        kms, kcnt, kfl = r["kernel"]
        achieved = kfl / (kms * 1e-3) / 1e12 if kms > 0 else None
        f_act = actual_flops(n, levels, args.algo)
        exch_bytes = (world - 1) * n * n * 8
        line = {
            "metric": METRIC.format(n=n), "value": round(tf(2.0 * n ** 3, ms), 4), "unit": UNIT, "n_gpus": world,
            "gpus_active": gpus_active, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 3),
            "higher_is_better": True, "step_ms": r["step_ms"], "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded standard normal)", "config": config(args, levels, world),
            "actual_tflops": round(tf(f_act, ms), 4),
            "frac_of_fp64_peak_actual": round(tf(f_act, ms) / (peak_tflops * world), 4),
            "workspace_bytes_per_rank": int(lib.mk_partial_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels)),
            "peak_mem_delta_bytes_rank0": int(peak_mem),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3) if achieved else None,
                         "peak": round(peak_tflops, 3), "unit": "TFLOP/s",
                         "frac": round(achieved / peak_tflops, 4) if achieved else None, "traffic": None,
                         "kernel": "mk::persistent_product_kernel (rank 0's leaf launches)",
                         "peak_source": "measured in this run: DMMA-only microbenchmark (mk_fp64_peak)"},
            "clocks": r["clocks"], "gpu_launches": r["launches"], "e2e": r.get("e2e"),
            "e2e_from_gpu0": r.get("e2e_from_gpu0"), "other_exchange_leg": r["other_leg"],
        }
        if "compute_ms" in r:
            t_ex = r["exchange_ms"]
            moved = exch_bytes * 1.0 / world  # per-GPU bytes of a pipelined reduce: S (N-1)/N
            line["exchange"] = {
                "compute_ms": round(r["compute_ms"], 3), "compute_ms_fastest_rank": round(r["compute_ms_min_rank"], 3),
                "exchange_ms": round(t_ex, 3),
                "bytes_per_step": exch_bytes,
                "note": "exchange = NCCL reduce of one n x n FP64 partial C per rank to rank 0; exchange_ms is the "
                        "slowest rank's reduce time (includes waiting for the slowest compute); per-GPU link bytes of a "
                        "pipelined reduce = S (N-1)/N, S = n^2 * 8",
                "link_gbs": round(moved / (t_ex * 1e-3) / 1e9, 1) if t_ex > 0 else None,
                "peer_peak_gbs": PEER_GBS, "frac_of_peer_peak": round(moved / (t_ex * 1e-3) / 1e9 / PEER_GBS, 4)
                if t_ex > 0 else None,
            }
        print(json.dumps(line), flush=True)
        dist.destroy_process_group()
        return

    # ---------------- N = 1
    def step():
        {"winograd-block": pk.winograd_block_mul, "strassen": pk.strassen_mul,
         "winograd-knuth": pk.winograd_knuth_mul}[args.algo](A, B, C, policy)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the clock sampler starts before the warm-up steps so that nvidia-smi's own start-up work
    # is over before the timed region; only samples taken after mark() are summarised
    with ClockSampler(local) as clk:
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        peak_mem = torch.cuda.max_memory_allocated(dev) - mem0
        launches0 = lib.mk_launch_count()
        torch.cuda.synchronize()
        clk.mark()
        _lib.check(lib.mk_timing_begin(), "mk_timing_begin")
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
        e0.record(stream)
        for i in range(args.steps):
            step()
            if i < args.steps - 1:
                marks[i].record(stream)  # per-step boundaries (median / best below)
        e1.record(stream)
        torch.cuda.synchronize()
    kms, kcnt, kfl = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
    _lib.check(lib.mk_timing_end(ctypes.byref(kms), ctypes.byref(kcnt), ctypes.byref(kfl)), "mk_timing_end")
    launches = lib.mk_launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    bounds = [e0] + marks + [e1]
    step_ms = [bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps)]
    value = tf(2.0 * n ** 3, ms)
    clocks = clk.summary()
    timed = event_timer(torch, stream)

    # -------- e2e: public API with pinned host buffers (H2D A, B; product; D2H C) --------
    e2e = None
    if not args.no_e2e:
        host_c = torch.empty((n, n), dtype=torch.float64).pin_memory()
        hA, hB, hC = pk.Matrix(host_a.numpy()), pk.Matrix(host_b.numpy()), pk.Matrix(host_c.numpy())
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fmarks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
        pk.winograd_block_mul(hA, hB, hC, policy)
        torch.cuda.synchronize()
        f0.record(stream)
        for i in range(args.steps):
            pk.winograd_block_mul(hA, hB, hC, policy)
            if i < args.steps - 1:
                fmarks[i].record(stream)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / args.steps
        fb = [f0] + fmarks + [f1]
        e2e = {"value": round(tf(2.0 * n ** 3, ems), 4), "unit": UNIT,
               "h2d_bytes_per_step": 2 * n * n * 8, "d2h_bytes_per_step": n * n * 8,
               "step_ms": step_stats([fb[i].elapsed_time(fb[i + 1]) for i in range(args.steps)]),
               "ms_per_step": round(ems, 2)}

    achieved = kfl.value / (kms.value * 1e-3) / 1e12 if kms.value > 0 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dominant_kernel", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {
        "bound": "tensor", "achieved": round(achieved, 3) if achieved else None, "peak": round(peak_tflops, 3),
        "unit": "TFLOP/s", "frac": round(achieved / peak_tflops, 4) if achieved else None, "traffic": traffic,
        "kernel": "mk::persistent_product_kernel (DMMA leaf product, K1/K3)",
        "launches_timed": kcnt.value // max(args.steps, 1) if kcnt.value else 0,
        "peak_source": "measured in this run: DMMA-only microbenchmark on all SMs (mk_fp64_peak); "
                       "MEASURED_PEAKS.json has no FP64 figure",
    }
    f_act = actual_flops(n, levels, args.algo)
    line = {
        "metric": METRIC.format(n=n), "value": round(value, 4), "unit": UNIT, "n_gpus": 1, "gpus_active": 1,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 3), "higher_is_better": True,
        "step_ms": step_stats(step_ms),
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded standard normal)",
        "config": config(args, levels),
        "actual_tflops": round(tf(f_act, ms), 4),
        "frac_of_fp64_peak_actual": round(tf(f_act, ms) / peak_tflops, 4),
        "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels)),
        "peak_mem_delta_bytes": int(peak_mem),
        "roofline": roofline, "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e,
    }
    legs = {x for x in args.legs.split(",") if x}
    if args.alt:
        alts = []
        for cut in [int(x) for x in args.alt.split(",") if x]:
            pol = pk.BasePolicy.naive_cutoff(cut)
            lv = levels_for(n, cut)
            ams = timed(lambda: pk.winograd_block_mul(A, B, C, pol), reps=3, warm=2)
            alts.append({"cutoff": cut, "levels": lv, "ms_per_step": round(ams, 3),
                         "value": round(tf(2.0 * n ** 3, ams), 4),
                         "actual_tflops": round(tf(actual_flops(n, lv, args.algo), ams), 4),
                         "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, lv))})
        line["alt_cutoffs"] = alts
    if "lean" in legs:
        # peak-workspace trade-off at the bench config: the memory-lean plans, same inputs
        lean = []
        try:
            for plan, label in (("hybrid", "winograd-block, hybrid plan (top level depth-first, breadth-first below)"),
                                ("depth-first", "winograd-block, depth-first plan (P_i accumulated into C by the "
                                                "epilogue)")):
                pk.set_plan(plan)
                t = timed(lambda: pk.winograd_block_mul(A, B, C, policy), reps=2)
                lean.append({"variant": label, "ms_per_step": round(t, 3), "value": round(tf(2.0 * n ** 3, t), 4),
                             "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels))})
        finally:
            pk.set_plan()
        t = timed(lambda: pk.two_temp_winograd(A, B, C, policy), reps=2)
        lean.append({"variant": "two-temp (default plan: the paper's Table-2 schedule)", "ms_per_step": round(t, 3),
                     "value": round(tf(2.0 * n ** 3, t), 4),
                     "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS["two-temp"], n, levels))})
        a2, b2 = da.clone(), db.clone()
        t = timed(lambda: pk.in_place_winograd(pk.Matrix(a2), pk.Matrix(b2), C, policy), reps=2)
        lean.append({"variant": "in-place, literal Table-3 schedule (inputs clobbered)", "ms_per_step": round(t, 3),
                     "value": round(tf(2.0 * n ** 3, t), 4),
                     "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS["in-place"], n, levels))})
        del a2, b2
        line["memory_lean"] = lean
    if args.ozaki_slices:
        line["ozaki_leaf"] = ozaki_leg(args, pk, lib, _lib, torch, A, B, C, dc, host_a, host_b, policy, stream, local)
    if legs & {"cfg3", "cfg5", "cublas"}:
        del A, B, C
        dc = None
        torch.cuda.empty_cache()
        line["legs"] = baseline_legs(args, pk, lib, _lib, torch, stream, peak_tflops, legs)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, levels)
    print(json.dumps(line), flush=True)


def _gather_devices(torch, dist, dev, gloo):
    """Distinct physical GPUs the ranks ran on (PCI bus ids gathered over the group)."""
    props = torch.cuda.get_device_properties(dev)
    key = getattr(props, "uuid", None)
    key = str(key) if key is not None else f"{props.pci_bus_id}:{props.pci_device_id}"
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, key)
    ids = {}
    return [ids.setdefault(k, len(ids)) for k in out]


if __name__ == "__main__":
    main()
