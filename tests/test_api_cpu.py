"""Host-side behaviour of the drop-in API (no GPU needed): tables, counters, cost models,
schedule legality, trace rendering, presets and the validation / error conventions that
run before any engine call. Modeled on the reference's own tests."""
import numpy as np
import pytest

import paper_2309_00628_b200 as pk
from paper_2309_00628_b200 import tables
from paper_2309_00628_b200.kernels import KERNEL_DEFS, model_cost
from paper_2309_00628_b200.schedules import IN_PLACE, TWO_TEMP, schedule_model_cost
from conftest import has_gpu

POL = {
    "scalar": pk.BasePolicy.scalar_only(),
    "unrolled2": pk.BasePolicy.unrolled_up_to(2),
    "unrolled8": pk.BasePolicy.unrolled_up_to(8),
    "cutoff12": pk.BasePolicy.naive_cutoff(12),
    "cutoff4": pk.BasePolicy.naive_cutoff(4),
}
for _t in (32, 64, 512, 1024, 4096, 8192):
    POL[f"cutoff{_t}"] = pk.BasePolicy.naive_cutoff(_t)


def test_public_names_match_reference_surface():
    ref_all = {
        "AliasError", "BasePolicy", "BenchRecord", "DimensionError", "IN_PLACE_STEPS", "LegalityReport", "Matrix",
        "MatrixView", "OpCounter", "ScheduleError", "ScheduleStep", "TWO_TEMP_STEPS", "VariantSpec", "bench_run",
        "block_add", "cutoff_naive_preferred", "get_variant", "in_place_winograd", "max_abs_diff", "multiply",
        "naive_mul", "pad_to_pow2", "predicted_buffers", "predicted_ops", "preset_names", "quadrants",
        "random_matrix", "read_matrix", "strassen_mul", "two_temp_winograd", "unpad", "unrolled_base",
        "validate_schedule", "variant_catalog", "winograd_block_mul", "winograd_knuth_mul", "write_matrix",
    }
    assert ref_all <= set(pk.__all__)
    for name in ref_all:
        assert hasattr(pk, name), name


def test_step_table_shapes():
    assert (KERNEL_DEFS["strassen"].adds_per_level, KERNEL_DEFS["strassen"].muls_per_level) == (18, 7)
    assert (KERNEL_DEFS["winograd-block"].adds_per_level, KERNEL_DEFS["winograd-block"].muls_per_level) == (15, 7)
    assert KERNEL_DEFS["winograd-knuth"].muls_per_level == 7
    assert KERNEL_DEFS["winograd-knuth-8call"].muls_per_level == 8
    assert [len(KERNEL_DEFS[k].temp_names) for k in ("strassen", "winograd-block", "winograd-knuth")] == [17, 18, 18]


def test_coefficients_reproduce_the_product_symbolically():
    # (sum_q a[p][q] A_q)(sum_q b[p][q] B_q) combined by c must equal the 2x2 block product
    for steps in (tables.STRASSEN_STEPS, tables.WINOGRAD_BLOCK_STEPS, tables.WINOGRAD_KNUTH_STEPS,
                  tables.WINOGRAD_KNUTH_8CALL_STEPS):
        a, b, c = tables.coefficients(steps)
        r = np.random.default_rng(0)
        A = [r.integers(-5, 6, (3, 3)) for _ in range(4)]
        B = [r.integers(-5, 6, (3, 3)) for _ in range(4)]
        P = [sum(a[p][q] * A[q] for q in range(4)) @ sum(b[p][q] * B[q] for q in range(4)) for p in range(len(a))]
        C = [sum(c[q][p] * P[p] for p in range(len(a))) for q in range(4)]
        want = [A[0] @ B[0] + A[1] @ B[2], A[0] @ B[1] + A[1] @ B[3], A[2] @ B[0] + A[3] @ B[2], A[2] @ B[1] + A[3] @ B[3]]
        for x, y in zip(C, want):
            assert np.array_equal(x, y)


def test_cost_models_match_golden(golden):
    meta, _ = golden
    for row in meta["costs"]:
        order = row["order"]
        pol = None if row["kernel"] == "naive" else POL[row["policy"]]
        assert list(pk.predicted_ops(row["kernel"], pol, order)) == row["ops"], row
        assert list(pk.predicted_buffers(row["kernel"], pol, order)) == row["buffers"], row
    for order, want in meta["model_cost_8call"]:
        assert list(model_cost("winograd-knuth-8call", pk.BasePolicy.scalar_only(), order)) == want


def test_closed_form_counts():
    for k in range(7):
        n = 2 ** k
        assert model_cost("strassen", POL["scalar"], n)[:2] == (7 ** k, 6 * (7 ** k - 4 ** k))
        assert model_cost("winograd-block", POL["scalar"], n)[:2] == (7 ** k, 5 * (7 ** k - 4 ** k))
    assert model_cost("strassen", POL["cutoff12"], 32)[0] == 25088
    for k in range(1, 8):
        n = 2 ** k
        bufs, peak = schedule_model_cost(TWO_TEMP, POL["scalar"], n)[2:]
        assert bufs == 2 * (7 ** k - 1) // 6 and peak <= 2 * n * n / 3
        assert schedule_model_cost(IN_PLACE, POL["scalar"], n)[2:] == (0, 0)


def test_validate_schedule_matches_golden_legality(golden):
    meta, _ = golden
    steps = {"two-temp": pk.TWO_TEMP_STEPS, "in-place": pk.IN_PLACE_STEPS}
    for row in meta["legality"]:
        rows = list(steps[row["schedule"]])
        i = row["swap"]
        rows[i - 1], rows[i] = rows[i], rows[i - 1]
        rows = tuple(pk.ScheduleStep(j + 1, s.symbol, s.op, s.lhs, s.rhs, s.store) for j, s in enumerate(rows))
        rep = pk.validate_schedule(rows, products_clobber_operands=row["clobber"])
        assert (rep.ok, rep.violation_index, rep.reason) == (row["ok"], row["violation_index"], row["reason"]), row


def test_builtin_schedules_legal_and_malformed_rejected():
    assert pk.validate_schedule(pk.TWO_TEMP_STEPS).ok
    assert pk.validate_schedule(pk.IN_PLACE_STEPS, products_clobber_operands=True).ok
    with pytest.raises(pk.ScheduleError):
        pk.validate_schedule(pk.TWO_TEMP_STEPS[:21])
    no_product = tuple(pk.ScheduleStep(s.index, s.symbol, "+" if s.op == "*" else s.op, s.lhs, s.rhs, s.store)
                       for s in pk.TWO_TEMP_STEPS)
    with pytest.raises(pk.ScheduleError):
        pk.validate_schedule(no_product)


def test_trace_rendering_matches_golden(golden):
    meta, _ = golden
    assert [s.render() for s in pk.IN_PLACE_STEPS] == meta["traces"]["in-place"]
    assert [s.render() for s in pk.TWO_TEMP_STEPS] == meta["traces"]["two-temp"]
    assert pk.IN_PLACE_STEPS[6].render() == "step 7: P1 = A11*B11 -> C11"


def test_presets_and_policies():
    assert len(pk.preset_names()) == 12
    assert pk.get_variant("winograd-mod2", cutoff=64).base == pk.BasePolicy.naive_cutoff(64)
    with pytest.raises(KeyError):
        pk.get_variant("nope")
    with pytest.raises(ValueError):
        pk.BasePolicy.unrolled_up_to(3)
    with pytest.raises(ValueError):
        pk.BasePolicy.naive_cutoff(0)
    with pytest.raises(ValueError):
        pk.BasePolicy("mystery")
    with pytest.raises(ValueError):
        pk.VariantSpec("naive", pk.BasePolicy.scalar_only(), pad=False)
    with pytest.raises(ValueError):
        pk.VariantSpec("strassen", None)
    assert pk.cutoff_naive_preferred(12, 12, 12) and not pk.cutoff_naive_preferred(13, 13, 13)


def test_errors_raised_before_any_engine_call():
    sq = pk.Matrix(np.zeros((4, 4)))
    for fn in (pk.strassen_mul, pk.winograd_block_mul, pk.winograd_knuth_mul, pk.two_temp_winograd,
               pk.in_place_winograd):
        with pytest.raises(pk.DimensionError):
            fn(pk.Matrix(np.zeros((6, 6))), pk.Matrix(np.zeros((6, 6))), pk.Matrix(np.zeros((6, 6))))
        with pytest.raises(pk.DimensionError):
            fn(pk.Matrix(np.zeros((4, 2))), sq, sq)
        with pytest.raises(pk.AliasError):
            fn(sq, sq, sq)
    with pytest.raises(TypeError):
        pk.naive_mul(np.zeros((2, 2)), sq, sq)
    with pytest.raises(pk.DimensionError):
        pk.naive_mul(pk.Matrix(np.zeros((2, 3))), pk.Matrix(np.zeros((2, 2))), pk.Matrix(np.zeros((2, 2))))
    a = pk.Matrix(np.zeros((4, 4)))
    with pytest.raises(pk.AliasError):
        pk.in_place_winograd(a, a, pk.Matrix(np.zeros((4, 4))))
    with pytest.raises(pk.DimensionError):
        pk.unrolled_base(pk.Matrix(np.zeros((16, 16))), pk.Matrix(np.zeros((16, 16))), pk.Matrix(np.zeros((16, 16))), 16)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    a = pk.Matrix(np.eye(4))
    with pytest.raises(pk.EngineUnavailable):
        pk.winograd_block_mul(a, pk.Matrix(np.eye(4)), pk.Matrix(np.zeros((4, 4))))
    with pytest.raises(pk.EngineUnavailable):
        pk.naive_mul(a, pk.Matrix(np.eye(4)), pk.Matrix(np.zeros((4, 4))))


def test_core_views_quadrants_padding_text(tmp_path):
    m = pk.Matrix(np.arange(16).reshape(4, 4))
    q = pk.quadrants(m)
    assert [v.arr.tolist() for v in q][3] == [[10, 11], [14, 15]]
    v = pk.MatrixView(m, 1, 2, 2, 2)
    v[0, 0] = 99
    assert m[1, 2] == 99
    p = pk.pad_to_pow2(pk.Matrix(np.ones((3, 5))))
    assert (p.rows, p.cols) == (8, 8) and p.arr.sum() == 15
    assert pk.unpad(p, 3, 5).arr.shape == (3, 5)
    path = tmp_path / "m.txt"
    pk.write_matrix(pk.Matrix(np.array([[1.5, -2.0], [1e-17, 3.0]])), str(path))
    back = pk.read_matrix(str(path))
    assert back.arr.dtype == np.float64 and back.arr[1, 0] == 1e-17
    with pytest.raises(ValueError):
        pk.read_matrix(__import__("io").StringIO("2 2\n1 2 3"))
    assert pk.max_abs_diff(pk.Matrix(np.ones((2, 2))), pk.Matrix(np.zeros((2, 2)))) == 1.0


def test_set_plan_validates_and_round_trips():
    """set_plan (B200 addition): bad names raise ValueError; the options reach the engine's
    planner (workspace sizes change) and can be restored. Host-only: no GPU needed."""
    import ctypes

    from paper_2309_00628_b200 import _lib

    import os

    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    with pytest.raises(ValueError):
        pk.set_plan("sideways")
    lib = _lib.load()
    v = ctypes.c_int(-1)
    try:
        pk.set_plan("depth-first", two_temp_tail=False)
        assert lib.mk_get_option(_lib.MK_OPT_PLAN, ctypes.byref(v)) == 0 and v.value == 1
        assert lib.mk_get_option(_lib.MK_OPT_LITERAL_TAIL, ctypes.byref(v)) == 0 and v.value == 0
        lean = lib.mk_workspace_bytes(_lib.ALGO_IDS["winograd-block"], 4096, 3)
    finally:
        pk.set_plan()
    assert lib.mk_get_option(_lib.MK_OPT_PLAN, ctypes.byref(v)) == 0 and v.value == 0
    assert lib.mk_workspace_bytes(_lib.ALGO_IDS["winograd-block"], 4096, 3) > lean
    assert lib.mk_get_option(99, ctypes.byref(v)) == _lib.MK_ERR_ARG


def test_set_leaf_validates_and_round_trips():
    """set_leaf (B200 addition): the INT8 tensor-core (Ozaki) leaf takes 4..8 slices; bad kinds and
    slice counts raise ValueError; the option reaches the engine (and its overlapped host path
    picks a product order for the faster leaves); the DMMA leaf is the default. Host-only."""
    import ctypes

    from paper_2309_00628_b200 import _lib

    lib = _lib.load()
    assert pk.get_leaf() == ("dmma", 0)
    with pytest.raises(ValueError):
        pk.set_leaf("int8")
    with pytest.raises(ValueError):
        pk.set_leaf("ozaki", 3)
    assert lib.mk_set_option(_lib.MK_OPT_LEAF_SLICES, 9) == _lib.MK_ERR_ARG
    order, up = (ctypes.c_int * 8)(), (ctypes.c_int * 8)()
    assert lib.mk_overlap_order(_lib.ALGO_IDS["winograd-block"], order, up) == 7
    dmma_order = list(order)[:7]
    try:
        pk.set_leaf("ozaki", 6)
        assert pk.get_leaf() == ("ozaki", 6)
        lib.mk_overlap_order(_lib.ALGO_IDS["winograd-block"], order, up)
        assert sorted(list(order)[:7]) == list(range(7)) and list(order)[:7] != dmma_order
        assert list(order)[0] == 0  # P1 = A11 B11 first: the fewest quadrants before any product
        v = ctypes.c_int(-1)
        assert lib.mk_get_option(_lib.MK_OPT_LEAF_MIN_LOG2, ctypes.byref(v)) == 0 and v.value == 29
        pk.set_leaf("ozaki", 8, min_work=4096 ** 3)
        assert lib.mk_get_option(_lib.MK_OPT_LEAF_MIN_LOG2, ctypes.byref(v)) == 0 and v.value == 36
        pk.set_leaf("ozaki", 8, min_work=0)
        assert lib.mk_get_option(_lib.MK_OPT_LEAF_MIN_LOG2, ctypes.byref(v)) == 0 and v.value == 0
        assert lib.mk_set_option(_lib.MK_OPT_LEAF_MIN_LOG2, 63) == _lib.MK_ERR_ARG
    finally:
        pk.set_leaf("dmma")
    assert pk.get_leaf() == ("dmma", 0)


def test_ozaki_workspace_and_chunking_bounds():
    """mk_ozaki_workspace_bytes: digit planes of both operands padded to whole tiles; K longer than
    the exact int32 accumulation allows is processed in chunks, so the workspace stops growing."""
    from paper_2309_00628_b200 import _lib

    lib = _lib.load()
    assert lib.mk_ozaki_workspace_bytes(1024, 1024, 1024, 3) == 0
    w8 = lib.mk_ozaki_workspace_bytes(4096, 4096, 4096, 8)
    assert w8 >= 8 * (4096 + 4096) * 4096
    assert lib.mk_ozaki_workspace_bytes(4096, 4096, 4096, 4) < w8
    # K = 4096 fits one chunk at 8 slices; 3 x 4096 runs as three chunks of 4096 (same workspace)
    assert lib.mk_ozaki_workspace_bytes(4096, 4096, 3 * 4096, 8) == w8


def test_baseline_operands_match_the_oracle_generators():
    """bench.py's GPU legs draw their inputs from the package (metrics.baseline_operands); the
    parity tests draw theirs from the oracle. Same seed, same draws, same bytes."""
    from oracle import strassen_oracle as o
    from paper_2309_00628_b200.metrics import BASELINE_SEED, ParameterError, baseline_operands

    assert BASELINE_SEED == o.SEED
    for cfg, scale in ((1, 1), (2, 4), (3, 32), (4, 64), (5, 20)):
        a, b = baseline_operands(cfg, scale=scale)
        ra, rb = o.operands(cfg, scale=scale)
        assert a.dtype == np.float64 and np.array_equal(a, ra) and np.array_equal(b, rb)
    with pytest.raises(ParameterError):
        baseline_operands(6)
