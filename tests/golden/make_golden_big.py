"""Golden pins for the full-size BASELINE configs 3, 4 and 5, produced by running the reference
package itself (matmulkit) on the seeded BASELINE inputs.

Run in the development container only (it imports /root/reference, absent on the GPU box):
    python tests/golden/make_golden_big.py          # ~5 min of CPU, ~20 GB of RAM

The full results (0.5-2 GiB each) are too large to commit, so each reference result R is pinned
by size-independent and sampled data that the GPU tests (tests/test_gpu_parity_big.py) compare
the engine's result with:

* ``sha``            SHA-256 of R (bit-level identity of a rerun here; not used on the GPU)
* ``max_abs``        max|R|
* ``err_vs_naive``   max|R - N| over the whole matrix, N = the reference's naive product
                     (np.matmul, kernels.py:258-266) of the same inputs
* rows / cols        a few full rows and columns of R (quadrant boundaries included)
* rowsum / colsum    R @ 1 and 1^T R (every element contributes)
* pts                R at 4096 fixed pseudo-random positions

for R = the reference's Winograd result and R = its naive result.

Calls:
  cfg3: winograd_block_mul(A, B, C, naive_cutoff(1024))        kernels.py:378-383 -> _dc :269-315
  cfg4: winograd_block_mul(A, B, C, naive_cutoff(8192|4096))   same
  cfg5: multiply(A, B, VariantSpec("winograd-block", naive_cutoff(512)))  hybrid.py:105-146
        (pads to 16384^2 -> 5 levels) and multiply(A, B, naive)
Inputs: oracle.strassen_oracle.operands(cfg) = A then B from np.random.default_rng(20240901),
exactly as the reference's generator draws them (metrics.py:62-68, 105-109).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import matmulkit as mk  # noqa: E402

from oracle import strassen_oracle as o  # noqa: E402  (input generator only)

PTS = 4096


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_lines(extent: int) -> list[int]:
    """Rows (or columns) to keep: both ends, quadrant boundaries of the first two levels and an
    interior line."""
    q = extent // 4
    idx = {0, q, 2 * q - 1, 2 * q, extent - 1, (extent * 5) // 7}
    return sorted(i for i in idx if 0 <= i < extent)


def points(m: int, n: int) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(7)
    return rng.integers(0, m, PTS), rng.integers(0, n, PTS)


def pin(name: str, r: np.ndarray, naive: np.ndarray, arrays: dict) -> dict:
    m, n = r.shape
    rows, cols = sample_lines(m), sample_lines(n)
    pi, pj = points(m, n)
    arrays[f"{name}_rows"] = np.ascontiguousarray(r[rows, :])
    arrays[f"{name}_cols"] = np.ascontiguousarray(r[:, cols].T)
    arrays[f"{name}_rowsum"] = r.sum(axis=1)
    arrays[f"{name}_colsum"] = r.sum(axis=0)
    arrays[f"{name}_pts"] = r[pi, pj]
    return {"sha": sha(r), "max_abs": float(np.abs(r).max()),
            "err_vs_naive": float(np.abs(r - naive).max()) if naive is not None else 0.0,
            "rows": rows, "cols": cols}


def main() -> None:
    meta: dict = {"reference": "matmulkit 0.1.0 (/root/reference/pkg)", "numpy": np.__version__,
                  "seed": o.SEED, "pts": PTS, "configs": {}}
    arrays: dict = {}
    only = set(sys.argv[1:])

    def want(c):
        return not only or c in only

    # ---- cfg3: n = 8192 uniform[-1,1), winograd-block, naive_cutoff(1024) -> 3 levels
    if want("cfg3"):
        a, b = o.operands(3)
        t0 = time.time()
        cn = mk.Matrix.zeros(8192, 8192)
        mk.naive_mul(mk.Matrix(a), mk.Matrix(b), cn)
        tn = time.time() - t0
        t0 = time.time()
        c = mk.Matrix.zeros(8192, 8192)
        ctr = mk.winograd_block_mul(mk.Matrix(a), mk.Matrix(b), c, mk.BasePolicy.naive_cutoff(1024))
        tw = time.time() - t0
        meta["configs"]["cfg3"] = {
            "call": "winograd_block_mul(A, B, C, BasePolicy.naive_cutoff(1024))", "n": 8192, "cutoff": 1024,
            "amax": float(np.abs(a).max()), "bmax": float(np.abs(b).max()),
            "winograd": pin("cfg3_wino", c.arr, cn.arr, arrays), "naive": pin("cfg3_naive", cn.arr, None, arrays),
            "counter": list(ctr.snapshot()), "seconds_here": {"winograd": round(tw, 2), "naive": round(tn, 2)}}
        print("cfg3", meta["configs"]["cfg3"]["winograd"]["err_vs_naive"], tw, tn, flush=True)
        del a, b, c, cn

    # ---- cfg4: n = 16384 standard normal, winograd-block, naive_cutoff(8192 | 4096)
    if want("cfg4"):
        a, b = o.operands(4)
        t0 = time.time()
        cn = mk.Matrix.zeros(16384, 16384)
        mk.naive_mul(mk.Matrix(a), mk.Matrix(b), cn)
        tn = time.time() - t0
        entry = {"n": 16384, "amax": float(np.abs(a).max()), "bmax": float(np.abs(b).max()),
                 "naive": pin("cfg4_naive", cn.arr, None, arrays), "cutoffs": {},
                 "seconds_here": {"naive": round(tn, 2)}}
        for cut in (8192, 4096):
            t0 = time.time()
            c = mk.Matrix.zeros(16384, 16384)
            ctr = mk.winograd_block_mul(mk.Matrix(a), mk.Matrix(b), c, mk.BasePolicy.naive_cutoff(cut))
            tw = time.time() - t0
            entry["cutoffs"][str(cut)] = {
                "call": f"winograd_block_mul(A, B, C, BasePolicy.naive_cutoff({cut}))",
                "winograd": pin(f"cfg4_c{cut}", c.arr, cn.arr, arrays), "counter": list(ctr.snapshot())}
            entry["seconds_here"][f"winograd_{cut}"] = round(tw, 2)
            print("cfg4", cut, entry["cutoffs"][str(cut)]["winograd"]["err_vs_naive"], tw, flush=True)
            del c
        meta["configs"]["cfg4"] = entry
        del a, b, cn

    # ---- cfg5: 12000x14000 . 14000x10000 uniform[-1,1), multiply(winograd-block, cutoff 512)
    if want("cfg5"):
        a, b = o.operands(5)
        t0 = time.time()
        cn = mk.multiply(mk.Matrix(a), mk.Matrix(b), mk.get_variant("naive"))
        tn = time.time() - t0
        t0 = time.time()
        ctr = mk.OpCounter()
        c = mk.multiply(mk.Matrix(a), mk.Matrix(b), mk.VariantSpec("winograd-block", mk.BasePolicy.naive_cutoff(512)),
                        ctr)
        tw = time.time() - t0
        meta["configs"]["cfg5"] = {
            "call": "multiply(A, B, VariantSpec('winograd-block', BasePolicy.naive_cutoff(512)))",
            "m": 12000, "k": 14000, "n": 10000, "cutoff": 512, "reference_padded_order": 16384,
            "amax": float(np.abs(a).max()), "bmax": float(np.abs(b).max()),
            "winograd": pin("cfg5_wino", c.arr, cn.arr, arrays), "naive": pin("cfg5_naive", cn.arr, None, arrays),
            "counter": list(ctr.snapshot()), "seconds_here": {"winograd": round(tw, 2), "naive": round(tn, 2)}}
        print("cfg5", meta["configs"]["cfg5"]["winograd"]["err_vs_naive"], tw, tn, flush=True)
        del a, b, c, cn

    path_j = os.path.join(HERE, "golden_big.json")
    path_a = os.path.join(HERE, "golden_big.npz")
    if only and os.path.exists(path_j):  # partial regeneration: merge with the existing pins
        old = json.load(open(path_j))
        old["configs"].update(meta["configs"])
        meta = old
        with np.load(path_a) as z:
            merged = {k: z[k] for k in z.files}
        merged.update(arrays)
        arrays = merged
    with open(path_j, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    np.savez(path_a, **arrays)
    print("wrote", path_j, path_a, sum(v.nbytes for v in arrays.values()) / 2 ** 20, "MiB")


if __name__ == "__main__":
    main()
