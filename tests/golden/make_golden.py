"""Generate golden vectors by running the reference package itself (matmulkit).

Run in the development container only (it imports /root/reference, which does not exist
on the GPU box):  python tests/golden/make_golden.py

Writes tests/golden/golden.json (case metadata, counters, traces, legality reports, cost
model values, SHA-256 of large results) and tests/golden/golden.npz (small results).
Operands are regenerated from the recorded seeds with numpy's PCG64, exactly as the
reference's metrics.random_matrix draws them (metrics.py:62-68).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import matmulkit as mk  # noqa: E402
from matmulkit import kernels as rk  # noqa: E402
from matmulkit import schedules as rs  # noqa: E402

SEED = 20240901


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def draw(seed: int, shape_a, shape_b, exact: bool):
    rng = np.random.default_rng(seed)
    if exact:
        return (rng.integers(-8, 9, size=shape_a, dtype=np.int64), rng.integers(-8, 9, size=shape_b, dtype=np.int64))
    return rng.uniform(-1.0, 1.0, size=shape_a), rng.uniform(-1.0, 1.0, size=shape_b)


POLICIES = {
    "scalar": mk.BasePolicy.scalar_only(),
    "unrolled2": mk.BasePolicy.unrolled_up_to(2),
    "unrolled8": mk.BasePolicy.unrolled_up_to(8),
    "cutoff12": mk.BasePolicy.naive_cutoff(12),
    "cutoff4": mk.BasePolicy.naive_cutoff(4),
}
FUNCS = {
    "strassen": mk.strassen_mul,
    "winograd-block": mk.winograd_block_mul,
    "winograd-knuth": mk.winograd_knuth_mul,
    "winograd-knuth-8call": lambda a, b, c, policy=None: mk.winograd_knuth_mul(a, b, c, policy=policy,
                                                                              recompute_first_product=True),
    "two-temp": mk.two_temp_winograd,
    "in-place": mk.in_place_winograd,
}


def main() -> None:
    meta: dict = {"seed": SEED, "reference": "matmulkit 0.1.0 (/root/reference/pkg)", "numpy": np.__version__}
    arrays: dict = {}

    # 1. square kernel cases
    cases = []
    idx = 0
    for kernel, fn in FUNCS.items():
        for pname, pol in POLICIES.items():
            for n in (1, 2, 4, 8, 16, 32, 64):
                for exact in (True, False):
                    if not exact and n > 16:
                        continue
                    if pname in ("scalar", "unrolled2") and n > 32:
                        continue
                    seed = SEED + 1000 + idx
                    a, b = draw(seed, (n, n), (n, n), exact)
                    c = mk.Matrix.zeros(n, n, np.int64 if exact else np.float64)
                    aa, bb = mk.Matrix(a.copy()), mk.Matrix(b.copy())
                    ctr = fn(aa, bb, c, policy=pol)
                    key = f"c{idx}"
                    arrays[key] = c.arr
                    cases.append({"id": idx, "kernel": kernel, "policy": pname, "n": n, "exact": exact,
                                  "seed": seed, "counter": list(ctr.snapshot()), "key": key,
                                  "a_clobbered": bool(not np.array_equal(aa.arr, a))})
                    idx += 1
    meta["square_cases"] = cases

    # 2. multiply() on rectangular shapes, every preset
    rect = []
    for j, (m, k, n) in enumerate([(1, 1, 1), (3, 5, 7), (12, 14, 10), (33, 17, 9), (16, 16, 16), (20, 9, 31)]):
        for exact in (True, False):
            seed = SEED + 5000 + 10 * j + int(exact)
            a, b = draw(seed, (m, k), (k, n), exact)
            for preset in mk.preset_names():
                spec = mk.get_variant(preset, cutoff=4)
                ctr = mk.OpCounter()
                lines: list = []
                c = mk.multiply(mk.Matrix(a), mk.Matrix(b), spec, ctr,
                                trace=lines.append if spec.kernel in ("two-temp", "in-place") else None)
                key = f"r{len(rect)}"
                arrays[key] = c.arr
                rect.append({"m": m, "k": k, "n": n, "exact": exact, "seed": seed, "preset": preset, "cutoff": 4,
                             "counter": list(ctr.snapshot()), "trace_lines": len(lines), "key": key})
    meta["rect_cases"] = rect

    # 3. BASELINE cfg1 (n=256 uniform, cutoff 32) and cfg2 (n=1024 integer-valued, cutoff 64)
    cfgs = {}
    rng = np.random.default_rng(SEED)
    a1, b1 = rng.uniform(-1.0, 1.0, (256, 256)), rng.uniform(-1.0, 1.0, (256, 256))
    naive1 = mk.multiply(mk.Matrix(a1), mk.Matrix(b1), mk.get_variant("naive")).arr
    cfgs["cfg1"] = {"n": 256, "cutoff": 32, "naive_sha": sha(naive1), "variants": {}}
    for preset in ("strassen-mod2", "winograd-mod2", "two-temp-mod", "in-place-mod"):
        ctr = mk.OpCounter()
        c = mk.multiply(mk.Matrix(a1), mk.Matrix(b1), mk.get_variant(preset, cutoff=32), ctr).arr
        cfgs["cfg1"]["variants"][preset] = {"sha": sha(c), "err_vs_naive": float(np.abs(c - naive1).max()),
                                            "counter": list(ctr.snapshot())}
    rng = np.random.default_rng(SEED)
    a2 = rng.integers(-8, 9, (1024, 1024), dtype=np.int64).astype(np.float64)
    b2 = rng.integers(-8, 9, (1024, 1024), dtype=np.int64).astype(np.float64)
    naive2 = mk.multiply(mk.Matrix(a2), mk.Matrix(b2), mk.get_variant("naive")).arr
    cfgs["cfg2"] = {"n": 1024, "cutoff": 64, "naive_sha": sha(naive2), "variants": {}}
    for preset in ("strassen-mod2", "winograd-mod2", "two-temp-mod", "in-place-mod"):
        ctr = mk.OpCounter()
        c = mk.multiply(mk.Matrix(a2), mk.Matrix(b2), mk.get_variant(preset, cutoff=64), ctr).arr
        cfgs["cfg2"]["variants"][preset] = {"sha": sha(c), "bit_exact_vs_naive": bool(np.array_equal(c, naive2)),
                                            "counter": list(ctr.snapshot())}
    meta["configs"] = cfgs

    # 4. traces, legality of every adjacent swap, cost models
    traces = {}
    for name, fn in (("two-temp", mk.two_temp_winograd), ("in-place", mk.in_place_winograd)):
        lines: list = []
        fn(mk.Matrix(np.array([[1, 2], [3, 4]])), mk.Matrix(np.array([[5, 6], [7, 8]])),
           mk.Matrix.zeros(2, 2, np.int64), trace=lines.append)
        traces[name] = lines
    meta["traces"] = traces
    legality = []
    for name, steps, clob in (("two-temp", rs.TWO_TEMP_STEPS, False), ("in-place", rs.IN_PLACE_STEPS, True)):
        for i in range(1, 22):
            rows = list(steps)
            rows[i - 1], rows[i] = rows[i], rows[i - 1]
            rows = tuple(rs.ScheduleStep(j + 1, s.symbol, s.op, s.lhs, s.rhs, s.store) for j, s in enumerate(rows))
            for flag in (False, True):
                rep = mk.validate_schedule(rows, products_clobber_operands=flag)
                legality.append({"schedule": name, "swap": i, "clobber": flag, "ok": rep.ok,
                                 "violation_index": rep.violation_index, "reason": rep.reason})
    meta["legality"] = legality
    costs = []
    pols = dict(POLICIES, cutoff32=mk.BasePolicy.naive_cutoff(32), cutoff64=mk.BasePolicy.naive_cutoff(64),
                cutoff512=mk.BasePolicy.naive_cutoff(512), cutoff1024=mk.BasePolicy.naive_cutoff(1024),
                cutoff4096=mk.BasePolicy.naive_cutoff(4096), cutoff8192=mk.BasePolicy.naive_cutoff(8192))
    for kernel in ("naive", "strassen", "winograd-knuth", "winograd-block", "two-temp", "in-place"):
        for pname, pol in pols.items():
            for e in range(0, 15):
                order = 1 << e
                p = None if kernel == "naive" else pol
                if kernel == "naive" and pname != "scalar":
                    continue
                costs.append({"kernel": kernel, "policy": pname, "order": order,
                              "ops": list(mk.predicted_ops(kernel, p, order)),
                              "buffers": list(mk.predicted_buffers(kernel, p, order))})
    meta["costs"] = costs
    meta["model_cost_8call"] = [[1 << e, list(rk.model_cost("winograd-knuth-8call", mk.BasePolicy.scalar_only(), 1 << e))]
                                for e in range(0, 10)]

    # 5. the reference CLI's `count` report (stdout, exit code) for a few presets
    import contextlib
    import io

    from matmulkit import cli as rcli

    cli_count = {}
    for preset in ("winograd-mod2", "strassen-mod", "two-temp", "in-place-mod", "winograd-knuth"):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = rcli.main(["count", "--algo", preset, "--orders", "2..256"])
        cli_count[preset] = {"rc": rc, "stdout": buf.getvalue()}
    meta["cli_count"] = cli_count
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = rcli.main(["verify", "--orders", "1..32", "--seeds", "2", "--cutoff", "4"])
    meta["cli_verify"] = {"args": ["verify", "--orders", "1..32", "--seeds", "2", "--cutoff", "4"], "rc": rc,
                          "stdout": buf.getvalue()}
    # `multiply --trace` on text files (integer entries, non-square shapes, every schedule preset)
    import tempfile

    rng = np.random.default_rng(SEED + 77)
    a = rng.integers(-8, 9, (13, 22))
    b = rng.integers(-8, 9, (22, 9))
    cli_mul = {"a": a.tolist(), "b": b.tolist(), "runs": {}}
    with tempfile.TemporaryDirectory() as td:
        fa, fb, fc = (os.path.join(td, x) for x in ("a.txt", "b.txt", "c.txt"))
        mk.write_matrix(mk.Matrix(a), fa)
        mk.write_matrix(mk.Matrix(b), fb)
        for preset in ("two-temp-mod", "in-place-mod", "winograd-mod2", "naive"):
            buf = io.StringIO()
            args = ["multiply", fa, fb, "--algo", preset, "--cutoff", "4", "-o", fc, "--trace"]
            with contextlib.redirect_stdout(buf):
                rc = rcli.main(args)
            cli_mul["runs"][preset] = {"rc": rc, "stdout": buf.getvalue(), "out": open(fc).read()}
    meta["cli_multiply"] = cli_mul
    # metrics.bench_run records (everything but the times)
    bench = []
    for preset in ("winograd-mod2", "two-temp-mod", "in-place", "naive"):
        for exact in (True, False):
            for rec in mk.bench_run(preset, [1, 2, 8, 32, 64], 2, SEED, exact=exact, cutoff=8):
                bench.append({"algo": rec.algo, "order": rec.order, "reps": rec.reps, "mults": rec.mults,
                              "adds": rec.adds, "temp_buffers": rec.temp_buffers,
                              "peak_live_elements": rec.peak_live_elements, "seed": rec.seed, "exact": exact})
    meta["bench_run"] = bench
    meta["bench_csv_header"] = mk.BenchRecord.CSV_HEADER

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print(f"{len(cases)} square cases, {len(rect)} rect cases, {len(costs)} cost rows")


if __name__ == "__main__":
    main()
