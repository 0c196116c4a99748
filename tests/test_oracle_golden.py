"""Pin the CPU oracle (oracle/strassen_oracle.py) against golden vectors produced by the
reference package itself (tests/golden/make_golden.py). CPU only."""
import hashlib
import os

import numpy as np
import pytest

from conftest import REFERENCE_SRC, draw, loop_matmul
from oracle import strassen_oracle as o

POL = {
    "scalar": o.policy("scalar"),
    "unrolled2": o.policy("unrolled", 2),
    "unrolled8": o.policy("unrolled", 8),
    "cutoff12": o.policy("naive-cutoff", 12),
    "cutoff4": o.policy("naive-cutoff", 4),
}
PRESET = {  # preset name -> (kernel, policy kind) with cutoff 4 / unroll 8 (hybrid.py:63-82)
    "naive": ("naive", None), "strassen": ("strassen", "scalar"), "winograd-knuth": ("winograd-knuth", "scalar"),
    "winograd-block": ("winograd-block", "scalar"), "strassen-mod": ("strassen", "unrolled8"),
    "winograd-mod": ("winograd-block", "unrolled8"), "strassen-mod2": ("strassen", "cutoff4"),
    "winograd-mod2": ("winograd-block", "cutoff4"), "two-temp": ("two-temp", "scalar"),
    "in-place": ("in-place", "scalar"), "two-temp-mod": ("two-temp", "cutoff4"), "in-place-mod": ("in-place", "cutoff4"),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_square_cases_bit_identical(golden):
    meta, arrays = golden
    assert len(meta["square_cases"]) > 300
    for case in meta["square_cases"]:
        n = case["n"]
        a, b = draw(case["seed"], (n, n), (n, n), case["exact"])
        got = o.product(case["kernel"], a, b, POL[case["policy"]])
        want = arrays[case["key"]]
        assert got.dtype == want.dtype
        assert np.array_equal(got, want), case
        assert list(o.cost(case["kernel"], POL[case["policy"]], n)) == case["counter"], case


def test_rect_multiply_cases_bit_identical(golden):
    meta, arrays = golden
    for case in meta["rect_cases"]:
        a, b = draw(case["seed"], (case["m"], case["k"]), (case["k"], case["n"]), case["exact"])
        kernel, pk = PRESET[case["preset"]]
        got = o.multiply(a, b, kernel, POL[pk] if pk else None)
        assert np.array_equal(got, arrays[case["key"]]), case


def test_baseline_cfg1_and_cfg2_hashes(golden):
    meta, _ = golden
    for cfg, cutoff in (("cfg1", 32), ("cfg2", 64)):
        a, b = o.operands(1 if cfg == "cfg1" else 2)
        info = meta["configs"][cfg]
        naive = o.multiply(a, b, "naive", None)
        assert sha(naive) == info["naive_sha"]
        for preset, v in info["variants"].items():
            kernel = PRESET[preset][0]
            got = o.multiply(a, b, kernel, o.policy("naive-cutoff", cutoff))
            assert sha(got) == v["sha"], (cfg, preset)
            if cfg == "cfg2":
                assert v["bit_exact_vs_naive"] and np.array_equal(got, naive)


def test_cost_models_match_reference(golden):
    meta, _ = golden
    pols = dict(POL)
    for t in (32, 64, 512, 1024, 4096, 8192):
        pols[f"cutoff{t}"] = o.policy("naive-cutoff", t)
    for row in meta["costs"]:
        order = row["order"]
        if row["kernel"] == "naive":
            assert row["ops"] == [order ** 3, order * order * (order - 1)]
            continue
        m, a, bufs, peak = o.cost(row["kernel"], pols[row["policy"]], order)
        assert [m, a] == row["ops"] and [bufs, peak] == row["buffers"], row


def test_known_answers():
    a = np.array([[1, 2], [3, 4]], dtype=np.int64)
    b = np.array([[5, 6], [7, 8]], dtype=np.int64)
    for kernel in ("strassen", "winograd-block", "winograd-knuth", "winograd-knuth-8call", "two-temp", "in-place"):
        assert o.product(kernel, a, b, o.policy("scalar")).tolist() == [[19, 22], [43, 50]]
    assert o.cost("strassen", o.policy("scalar"), 2)[:2] == (7, 18)
    assert o.cost("winograd-block", o.policy("scalar"), 2)[:2] == (7, 15)
    assert o.cost("winograd-knuth-8call", o.policy("scalar"), 2)[0] == 8


def test_oracle_against_independent_triple_loop(rng):
    for n in (1, 2, 4, 8):
        a = rng.integers(-8, 9, (n, n), dtype=np.int64)
        b = rng.integers(-8, 9, (n, n), dtype=np.int64)
        want = loop_matmul(a, b)
        for kernel in ("strassen", "winograd-block", "winograd-knuth", "two-temp", "in-place"):
            assert np.array_equal(o.product(kernel, a, b, o.policy("scalar")), want)


def test_tolerance_formula():
    # c * n^log2(12) * u * |A| |B|; at n = 8192 with unit operands the bound is ~0.0118
    assert abs(o.tolerance(8192, 1.0, 1.0) - 8192 ** np.log2(12) * 2.0 ** -53) < 1e-15
    assert 0.011 < o.tolerance(8192, 1.0, 1.0) < 0.0125


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference package not mounted")
def test_oracle_matches_live_reference_random():
    import sys

    sys.path.insert(0, REFERENCE_SRC)
    import matmulkit as mk

    r = np.random.default_rng(7)
    for kernel, fn in (("strassen", mk.strassen_mul), ("winograd-block", mk.winograd_block_mul),
                       ("two-temp", mk.two_temp_winograd), ("in-place", mk.in_place_winograd)):
        for n in (16, 64):
            a, b = r.uniform(-1, 1, (n, n)), r.uniform(-1, 1, (n, n))
            c = mk.Matrix.zeros(n, n)
            fn(mk.Matrix(a.copy()), mk.Matrix(b.copy()), c, policy=mk.BasePolicy.naive_cutoff(8))
            assert np.array_equal(o.product(kernel, a, b, o.policy("naive-cutoff", 8)), c.arr)


def test_big_config_pins_are_consistent():
    """tests/golden/golden_big.* (the reference's own cfg3/cfg4/cfg5 outputs, pinned by rows,
    columns, sums and points): shapes agree with the configs and the input generator reproduces
    the recorded operand maxima."""
    import json

    from conftest import GOLDEN_DIR

    meta = json.load(open(os.path.join(GOLDEN_DIR, "golden_big.json")))
    arr = np.load(os.path.join(GOLDEN_DIR, "golden_big.npz"))
    shapes = {"cfg3_wino": (8192, 8192), "cfg3_naive": (8192, 8192), "cfg4_naive": (16384, 16384),
              "cfg4_c8192": (16384, 16384), "cfg4_c4096": (16384, 16384), "cfg5_wino": (12000, 10000),
              "cfg5_naive": (12000, 10000)}
    for key, (m, n) in shapes.items():
        assert arr[f"{key}_rowsum"].shape == (m,) and arr[f"{key}_colsum"].shape == (n,)
        assert arr[f"{key}_rows"].shape[1] == n and arr[f"{key}_cols"].shape[1] == m
        assert arr[f"{key}_pts"].shape == (meta["pts"],)
    c3 = meta["configs"]["cfg3"]
    a, b = o.operands(3)
    assert float(np.abs(a).max()) == c3["amax"] and float(np.abs(b).max()) == c3["bmax"]
    # the reference's own Winograd error vs its naive product, as recorded in SURVEY/BASELINE
    assert c3["winograd"]["err_vs_naive"] < 1e-11
    assert meta["configs"]["cfg4"]["cutoffs"]["4096"]["winograd"]["err_vs_naive"] < 1e-11
    assert meta["configs"]["cfg5"]["winograd"]["err_vs_naive"] < 1e-10


def test_oracle_reproduces_reference_cfg3_full_size():
    """The oracle run at full cfg3 (n = 8192, winograd-block, naive_cutoff(1024): 343 leaves) is
    bit-identical to the reference's own output (SHA-256 recorded by make_golden_big.py)."""
    import json

    from conftest import GOLDEN_DIR

    meta = json.load(open(os.path.join(GOLDEN_DIR, "golden_big.json")))
    a, b = o.operands(3)
    c = o.product("winograd-block", a, b, o.policy("naive-cutoff", 1024))
    assert hashlib.sha256(np.ascontiguousarray(c).tobytes()).hexdigest() == meta["configs"]["cfg3"]["winograd"]["sha"]
