"""Benchmark: effective FP64 TFLOP/s (2 n^3 / t) of Strassen-Winograd on B200.

Workload (BASELINE.json config 4, the north-star target): n = 16384, A and B standard
normal from np.random.default_rng(20240901) (A then B), winograd-block with
naive_cutoff(4096) -> 2 recursion levels, 49 DMMA leaf GEMMs of 4096^3. One "step" is one
full multiplication C = A B. Inputs (2 GiB each) exceed the 126 MB L2, so no L2 flush is
needed between steps.

  python bench.py [--gpus N --steps K --warmup W]          # our engine (N ranks via torchrun)
  python bench.py --impl reference [...]                   # the reference CPU path (oracle port)

value     = whole-job 2n^3 / t, inputs resident in HBM, CUDA events, max over ranks.
e2e       = the same metric through the public API with pinned HOST buffers: per step
            H2D of A and B, the product, D2H of C.
roofline  = the dominant kernel (fused DMMA leaf product): algorithmic flops per launch /
            CUDA-event launch time inside the timed region, against the FP64 tensor roofline
            measured in the same run by a DMMA-only microbenchmark (mk_fp64_peak).
cpu_baseline = the oracle (numpy restatement of the reference, bit-identical to it) on the
            host cores, bounded sample: n = 8192 with the same 2-level recursion.
N > 1     = strong scaling of one product: the 49 leaves, split into 8 row panels each, sharded
            evenly over ranks; partial C sum-reduced to rank 0 over NVLink (NCCL).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective FP64 TFLOP/s (2n^3/t) of Strassen-Winograd, n={n}"
UNIT = "TFLOP/s"


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
                   help="N > 1: leaf epilogues add into the owning rank's C row slab over peer memory "
                        "(mk_strassen_partial_slabs) instead of partial C + NCCL reduce")
    p.add_argument("--alt", default="8192,2048", help="extra cutoffs to report (comma list, '' for none)")
    p.add_argument("--ozaki-slices", type=int, default=8,
                   help="also time the same workload with INT8 tensor-core (Ozaki) leaves, 0 = skip")
    return p.parse_args()


def config(args, levels):
    c = {
        "workload": f"BASELINE cfg4: n={args.n} standard-normal FP64, {args.algo}, naive_cutoff({args.cutoff}) "
                    f"-> {levels} levels ({7 ** levels} DMMA leaf GEMMs)",
        "n": args.n, "cutoff": args.cutoff, "levels": levels, "algo": args.algo,
        "l2": "inputs 2 GiB each > 126 MB L2 (no flush needed)",
    }
    if args.gpus > 1:
        c["parallelism"] = (f"leaf row panels over {args.gpus} ranks; " +
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
def cpu_sample_seconds(n_sample, cutoff_sample, algo):
    """One oracle (reference restatement) product of the bounded sample, on the host."""
    from oracle import strassen_oracle as o

    rng = np.random.default_rng(o.SEED)
    a = rng.standard_normal((n_sample, n_sample))
    b = rng.standard_normal((n_sample, n_sample))
    kernel = algo if algo in o.TABLES else "winograd-block"
    t0 = time.perf_counter()
    o.product(kernel, a, b, o.policy("naive-cutoff", cutoff_sample))
    return time.perf_counter() - t0


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


def cpu_baseline(args, levels):
    n_s = args.n // 2
    cut_s = n_s >> levels
    with all_host_threads():
        # warm numpy/OpenBLAS once on a small case
        cpu_sample_seconds(512, 128, args.algo)
        t = cpu_sample_seconds(n_s, cut_s, args.algo)
        cores = blas_threads()
    return {
        "value": round(2.0 * n_s ** 3 / t / 1e12, 4), "unit": UNIT, "cores": cores, "kind": "port",
        "sample": f"oracle (numpy restatement of matmulkit, bit-identical) {args.algo} n={n_s} "
                  f"naive_cutoff({cut_s}) = same {levels}-level recursion at 1/8 the flops; "
                  f"OpenBLAS leaves on {cores} threads, block adds single-threaded; {t:.2f} s",
        "seconds": round(t, 3),
    }


def run_reference(args):
    levels = levels_for(args.n, args.cutoff)
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_s = args.n // 2
    cut_s = n_s >> levels
    with all_host_threads():
        cpu_sample_seconds(512, 128, args.algo)
        for _ in range(args.warmup):
            cpu_sample_seconds(n_s, cut_s, args.algo)
        ts = [cpu_sample_seconds(n_s, cut_s, args.algo) for _ in range(args.steps)]
        cores = blas_threads()
    ms = 1e3 * sum(ts) / len(ts)
    value = 2.0 * n_s ** 3 / (ms * 1e-3) / 1e12
    line = {
        "metric": METRIC.format(n=args.n), "value": round(value, 4), "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded standard normal)",
        "config": config(args, levels),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"oracle {args.algo} n={n_s} naive_cutoff({cut_s}) per step (bounded sample of "
                                   f"the n={args.n} workload, same recursion depth); host cores only"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- Ozaki leg
def ozaki_leg(args, pk, lib, _lib, torch, A, B, C, dc, host_a, host_b, policy, stream, local):
    """The same workload with every leaf product on the INT8 tensor cores (Ozaki scheme I,
    set_leaf("ozaki", S)): value / e2e like the headline, the leaf launches' int8 roofline, and
    the max difference from the DMMA (FP64 tensor-core) result of the same inputs."""
    n, S = args.n, args.ozaki_slices
    call = {"winograd-block": pk.winograd_block_mul, "strassen": pk.strassen_mul,
            "winograd-knuth": pk.winograd_knuth_mul}[args.algo]
    pk.set_leaf("dmma")
    call(A, B, C, policy)
    ref = dc.clone()
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
        # e2e through the public API with pinned host buffers
        host_c = torch.empty((n, n), dtype=torch.float64).pin_memory()
        hA, hB, hC = pk.Matrix(host_a.numpy()), pk.Matrix(host_b.numpy()), pk.Matrix(host_c.numpy())
        call(hA, hB, hC, policy)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            call(hA, hB, hC, policy)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / args.steps
        alts = []
        for cut in [int(x) for x in args.alt.split(",") if x]:  # same extra cutoffs as the DMMA leg
            pol = pk.BasePolicy.naive_cutoff(cut)
            for _ in range(2):
                call(A, B, C, pol)
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(3):
                call(A, B, C, pol)
            g1.record(stream)
            torch.cuda.synchronize()
            ams = g0.elapsed_time(g1) / 3
            alts.append({"cutoff": cut, "levels": levels_for(n, cut), "ms_per_step": round(ams, 3),
                         "value": round(2.0 * n ** 3 / (ams * 1e-3) / 1e12, 4)})
        lean = []  # the paper's memory-reduced schedules (literal to the leaves) with INT8 leaves
        if args.alt:
            pk.set_plan("breadth-first", two_temp_tail=False)
            for name, fn, mk_in in (("two-temp", pk.two_temp_winograd, False), ("in-place", pk.in_place_winograd, True)):
                a2, b2 = (dc.new_empty(dc.shape).copy_(A.arr), dc.new_empty(dc.shape).copy_(B.arr)) if mk_in else (None, None)
                X, Y = (pk.Matrix(a2), pk.Matrix(b2)) if mk_in else (A, B)
                fn(X, Y, C, policy)
                torch.cuda.synchronize()
                g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                fn(X, Y, C, policy)
                g1.record(stream)
                torch.cuda.synchronize()
                lms = g0.elapsed_time(g1)
                lean.append({"variant": name, "ms_per_step": round(lms, 3),
                             "value": round(2.0 * n ** 3 / (lms * 1e-3) / 1e12, 4),
                             "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[name], n,
                                                                           levels_for(n, args.cutoff)))})
                del a2, b2
    finally:
        pk.set_leaf("dmma")
        pk.set_plan()
    pairs = S * (S + 1) // 2
    peak = None
    src = "nominal 4500 TOPS dense INT8 (B200 datasheet)"
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        if mp.get("bf16_tflops"):
            peak = 2.0 * float(mp["bf16_tflops"])
            src = "2 x MEASURED_PEAKS.json bf16_tflops (burst; the tensor pipe's 8-bit rate is twice its 16-bit rate)"
    except Exception:
        pass
    if peak is None:
        peak = 4500.0
    achieved = pairs * kfl.value / (kms.value * 1e-3) / 1e12 if kms.value > 0 else None
    return {
        "slices": S, "digit_bits": 7 + 8 * (S - 1), "int8_products_per_leaf": pairs,
        "extra_workspace_bytes": 2 * int(lib.mk_ozaki_workspace_bytes(n >> levels_for(n, args.cutoff),
                                                                       n >> levels_for(n, args.cutoff),
                                                                       n >> levels_for(n, args.cutoff), S)),
        "value": round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 4), "unit": UNIT, "ms_per_step": round(ms, 3),
        "step_ms": {"median": round(statistics.median(step_ms), 3), "best": round(min(step_ms), 3),
                    "worst": round(max(step_ms), 3)},
        "e2e": {"value": round(2.0 * n ** 3 / (ems * 1e-3) / 1e12, 4), "unit": UNIT, "ms_per_step": round(ems, 2),
                "h2d_bytes_per_step": 2 * n * n * 8, "d2h_bytes_per_step": n * n * 8},
        "max_abs_diff_vs_dmma_result": diff, "result_max_abs": scale,
        "roofline": {"bound": "tensor", "achieved": round(achieved, 1) if achieved else None, "peak": round(peak, 1),
                     "unit": "TOPS (int8)", "frac": round(achieved / peak, 4) if achieved else None,
                     "kernel": "mk::oz::ozaki_product_kernel + digit splitting (per leaf, CUDA events)",
                     "peak_source": src},
        "clocks": clk.summary(),
        "alt_cutoffs": alts,
        "memory_lean": lean,
        "dtype": "f64 operands/results; int8 x int8 -> int32 tensor-core products (Ozaki scheme I)",
    }


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2309_00628_b200 as pk
    from paper_2309_00628_b200 import _lib, multigpu
    from paper_2309_00628_b200.device import require_engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
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

    from oracle import strassen_oracle as o  # seeded inputs identical to the oracle's (cfg4 generator)

    rng = np.random.default_rng(o.SEED)
    host_a = torch.from_numpy(rng.standard_normal((n, n))).pin_memory()
    host_b = torch.from_numpy(rng.standard_normal((n, n))).pin_memory()
    da, db = host_a.to(dev), host_b.to(dev)
    dc = torch.empty((n, n), dtype=torch.float64, device=dev)
    A, B, C = pk.Matrix(da), pk.Matrix(db), pk.Matrix(dc)
    ws = None
    ex = None
    if world > 1:
        need = int(lib.mk_partial_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels))
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
        if args.fused_reduce:
            ex = multigpu.SlabExchange(n)

    def step():
        if world == 1:
            {"winograd-block": pk.winograd_block_mul, "strassen": pk.strassen_mul,
             "winograd-knuth": pk.winograd_knuth_mul}[args.algo](A, B, C, policy)
        elif ex is not None:
            multigpu.fused_sharded_multiply(args.algo, da, db, levels, ex, out=dc if rank == 0 else None, ws=ws)
        else:
            multigpu.sharded_multiply(args.algo, da, db, levels, out=dc, ws=ws)

    def barrier():
        if world > 1:
            dist.barrier()

    torch.cuda.reset_peak_memory_stats(dev)
    mem0 = torch.cuda.memory_allocated(dev)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the clock sampler starts before the warm-up steps so that nvidia-smi's own start-up work
    # is over before the timed region; only samples taken after mark() are summarised
    with ClockSampler(local) as clk:
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        peak_mem = torch.cuda.max_memory_allocated(dev) - mem0
        launches0 = lib.mk_launch_count()
        barrier()
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
        barrier()
    kms, kcnt, kfl = ctypes.c_double(), ctypes.c_int(), ctypes.c_double()
    _lib.check(lib.mk_timing_end(ctypes.byref(kms), ctypes.byref(kcnt), ctypes.byref(kfl)), "mk_timing_end")
    launches = lib.mk_launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    bounds = [e0] + marks + [e1]
    step_ms = [bounds[i].elapsed_time(bounds[i + 1]) for i in range(args.steps)]
    if os.environ.get("MK_BENCH_VERBOSE"):
        print("step_ms", [round(x, 3) for x in step_ms], file=sys.stderr)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([launches], device=dev, dtype=torch.int64)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt.item())
    value = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
    clocks = clk.summary()

    # -------- e2e: public API with pinned host buffers (H2D A, B; product; D2H C) --------
    e2e = None
    if not args.no_e2e:
        host_c = torch.empty((n, n), dtype=torch.float64).pin_memory()
        moved = [2 * n * n * 8]  # H2D bytes of this rank per step
        hA, hB, hC = pk.Matrix(host_a.numpy()), pk.Matrix(host_b.numpy()), pk.Matrix(host_c.numpy())

        def e2e_step():
            if world == 1:
                pk.winograd_block_mul(hA, hB, hC, policy)
            else:  # each rank uploads only the operand quadrants its shard reads
                moved[0] = multigpu.upload_operands(args.algo, levels, host_a, host_b, da, db)
                if ex is not None:
                    multigpu.fused_sharded_multiply(args.algo, da, db, levels, ex, out=dc if rank == 0 else None,
                                                    ws=ws)
                else:
                    multigpu.sharded_multiply(args.algo, da, db, levels, out=dc, ws=ws)
                if rank == 0:
                    host_c.copy_(dc, non_blocking=True)
                torch.cuda.current_stream().synchronize()

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fmarks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps - 1)]
        f0.record(stream)
        for i in range(args.steps):
            e2e_step()
            if i < args.steps - 1:
                fmarks[i].record(stream)
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = f0.elapsed_time(f1) / args.steps
        fb = [f0] + fmarks + [f1]
        e2e_steps = [fb[i].elapsed_time(fb[i + 1]) for i in range(args.steps)]
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = moved[0]
        if world > 1:
            t = torch.tensor([h2d], device=dev, dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            h2d = int(t.item())
        e2e = {"value": round(2.0 * n ** 3 / (ems * 1e-3) / 1e12, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": n * n * 8,
               "step_ms": {"median": round(statistics.median(e2e_steps), 3), "best": round(min(e2e_steps), 3),
                           "worst": round(max(e2e_steps), 3)},
               "ms_per_step": round(ems, 2)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

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
        "metric": METRIC.format(n=n), "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 3), "higher_is_better": True,
        "step_ms": {"median": round(statistics.median(step_ms), 3), "best": round(min(step_ms), 3),
                    "worst": round(max(step_ms), 3)},
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded standard normal)",
        "config": config(args, levels),
        "actual_tflops": round(f_act / (ms * 1e-3) / 1e12, 4),
        "frac_of_fp64_peak_actual": round(f_act / (ms * 1e-3) / 1e12 / peak_tflops, 4),
        "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels) if world == 1
                               else lib.mk_partial_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels)),
        "peak_mem_delta_bytes": int(peak_mem),
        "roofline": roofline, "clocks": clocks, "gpu_launches": int(launches), "e2e": e2e,
    }
    if world == 1 and args.alt:
        alts = []
        for cut in [int(x) for x in args.alt.split(",") if x]:
            pol = pk.BasePolicy.naive_cutoff(cut)
            lv = levels_for(n, cut)
            for _ in range(2):
                pk.winograd_block_mul(A, B, C, pol)
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(3):
                pk.winograd_block_mul(A, B, C, pol)
            g1.record(stream)
            torch.cuda.synchronize()
            ams = g0.elapsed_time(g1) / 3
            alts.append({"cutoff": cut, "levels": lv, "ms_per_step": round(ams, 3),
                         "value": round(2.0 * n ** 3 / (ams * 1e-3) / 1e12, 4),
                         "actual_tflops": round(actual_flops(n, lv, args.algo) / (ams * 1e-3) / 1e12, 4),
                         "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, lv))})
        line["alt_cutoffs"] = alts
    if world == 1 and args.alt:
        # peak-workspace trade-off at the bench config: the memory-lean plans, same inputs
        def timed(fn, reps=2):
            fn()
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for _ in range(reps):
                fn()
            g1.record(stream)
            torch.cuda.synchronize()
            return g0.elapsed_time(g1) / reps

        lean = []
        try:
            pk.set_plan("hybrid", two_temp_tail=False)
            ms_hy = timed(lambda: pk.winograd_block_mul(A, B, C, policy))
            lean.append({"variant": "winograd-block, hybrid plan (top level depth-first, breadth-first below)",
                         "ms_per_step": round(ms_hy, 3), "value": round(2.0 * n ** 3 / (ms_hy * 1e-3) / 1e12, 4),
                         "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels))})
            pk.set_plan("depth-first", two_temp_tail=False)
            ms_dfs = timed(lambda: pk.winograd_block_mul(A, B, C, policy))
            lean.append({"variant": "winograd-block, depth-first plan (P_i accumulated into C by the epilogue)",
                         "ms_per_step": round(ms_dfs, 3), "value": round(2.0 * n ** 3 / (ms_dfs * 1e-3) / 1e12, 4),
                         "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS[args.algo], n, levels))})
            ms_tt = timed(lambda: pk.two_temp_winograd(A, B, C, policy))
            lean.append({"variant": "two-temp, literal Table-2 schedule to the leaves",
                         "ms_per_step": round(ms_tt, 3), "value": round(2.0 * n ** 3 / (ms_tt * 1e-3) / 1e12, 4),
                         "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS["two-temp"], n, levels))})
        finally:
            pk.set_plan()
        a2, b2 = da.clone(), db.clone()
        ms_ip = timed(lambda: pk.in_place_winograd(pk.Matrix(a2), pk.Matrix(b2), C, policy))
        lean.append({"variant": "in-place, literal Table-3 schedule (inputs clobbered)",
                     "ms_per_step": round(ms_ip, 3), "value": round(2.0 * n ** 3 / (ms_ip * 1e-3) / 1e12, 4),
                     "workspace_bytes": int(lib.mk_workspace_bytes(_lib.ALGO_IDS["in-place"], n, levels))})
        del a2, b2
        line["memory_lean"] = lean
    if world == 1 and args.ozaki_slices:
        line["ozaki_leaf"] = ozaki_leg(args, pk, lib, _lib, torch, A, B, C, dc, host_a, host_b, policy, stream,
                                       local)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, levels)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
