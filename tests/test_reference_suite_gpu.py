"""The reference's own test suite (/root/reference/pkg/tests: test_core.py 32, test_kernels.py 46,
test_schedules.py 32 = 110 collected cases), restated against this package and run on the GPU.

The reference files are not copied: every case below restates what one reference test checks
(cited as file:line) in this repository's own table-driven form, with the same inputs (seeded
[-8, 8] integers / [-1, 1) reals from default_rng(20240901), the reference conftest.py:29-39), the
same orders and policies and the same assertions. Compute cases run on the B200 engine; the
host-only cases (Matrix / views / text format / schedule legality) run the same package code.
`REFERENCE_CASES` maps each of the 110 reference test ids to the case here that replays it; the
test at the bottom checks that the map is complete.
"""
import io

import numpy as np
import pytest

import paper_2309_00628_b200 as pk
from conftest import has_gpu, int_matrix, loop_matmul, real_matrix
from paper_2309_00628_b200 import (AliasError, BasePolicy, DimensionError, Matrix, MatrixView, OpCounter,
                                   ScheduleError, ScheduleStep)
from paper_2309_00628_b200.core import matrix_to_text
from paper_2309_00628_b200.schedules import IN_PLACE_STEPS, TWO_TEMP_STEPS

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

SEED = 20240901
TWO = (Matrix(np.array([[1, 2], [3, 4]], dtype=np.int64)), Matrix(np.array([[5, 6], [7, 8]], dtype=np.int64)))
TWO_PRODUCT = [[19, 22], [43, 50]]
DC = {"strassen": pk.strassen_mul, "winograd_knuth": pk.winograd_knuth_mul, "winograd_block": pk.winograd_block_mul}
POLICIES = {"scalar": BasePolicy.scalar_only(), "unrolled2": BasePolicy.unrolled_up_to(2),
            "unrolled8": BasePolicy.unrolled_up_to(8), "cutoff12": BasePolicy.naive_cutoff(12)}


@pytest.fixture
def rng():
    return np.random.default_rng(SEED)


def mul(fn, a, b, dtype=None, **kw):
    """C := fn(A, B) into a fresh zero C; returns (C, counter)."""
    c = Matrix.zeros(a.rows, b.cols, dtype or a.arr.dtype)
    return c, fn(a, b, c, **kw)


def naive(a, b):
    return mul(pk.naive_mul, a, b)[0]


# ======================================================================= test_kernels.py
class TestKernels:
    def test_naive_identity(self):  # test_kernels.py:33-35
        c, _ = mul(pk.naive_mul, TWO[0], Matrix(np.eye(2, dtype=np.int64)))
        assert c.arr.tolist() == TWO[0].arr.tolist()

    def test_naive_2x2_by_hand(self):  # :38-41
        c, ctr = mul(pk.naive_mul, *TWO)
        assert c.arr.tolist() == TWO_PRODUCT and (ctr.mults, ctr.adds) == (8, 4)

    def test_naive_rectangular_matches_independent_loop(self, rng):  # :44-50
        a, b = int_matrix(rng, 3, 2), int_matrix(rng, 2, 4)
        c, ctr = mul(pk.naive_mul, a, b)
        assert np.array_equal(c.arr, loop_matmul(a.arr, b.arr))
        assert (ctr.mults, ctr.adds) == (24, 12)

    def test_naive_rejects_inner_mismatch(self):  # :53-55
        with pytest.raises(DimensionError):
            mul(pk.naive_mul, Matrix(np.zeros((2, 3))), Matrix(np.zeros((2, 2))))

    def test_naive_rejects_aliased_output(self):  # :58-61
        a = Matrix(np.zeros((2, 2)))
        with pytest.raises(AliasError):
            pk.naive_mul(a, TWO[0], a)

    @pytest.mark.parametrize("name,fn,kw,adds", [
        ("strassen", pk.strassen_mul, {}, 18),                                      # :64-67
        ("knuth", pk.winograd_knuth_mul, {}, None),                                 # :83-86
        ("block", pk.winograd_block_mul, {}, 15),                                   # :113-116
    ])
    def test_order2_values_and_counts(self, name, fn, kw, adds):
        c, ctr = mul(fn, *TWO, **kw)
        assert c.arr.tolist() == TWO_PRODUCT and ctr.mults == 7
        if adds is not None:
            assert ctr.adds == adds

    def test_strassen_order1_scalar_base(self):  # :70-73
        c, ctr = mul(pk.strassen_mul, Matrix(np.array([[3]])), Matrix(np.array([[4]])))
        assert c[0, 0] == 12 and (ctr.mults, ctr.adds) == (1, 0)

    @pytest.mark.parametrize("fn,order", [(pk.strassen_mul, 8),                     # :76-80
                                          (pk.winograd_knuth_mul, 4),               # :94-99
                                          (pk.winograd_knuth_mul, 8),
                                          (pk.winograd_knuth_mul, 16),
                                          (pk.winograd_block_mul, 32)])             # :119-123
    def test_matches_naive(self, rng, fn, order):
        a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
        assert np.array_equal(mul(fn, a, b)[0].arr, naive(a, b).arr)

    def test_winograd_knuth_identity(self):  # :89-91
        c, _ = mul(pk.winograd_knuth_mul, TWO[0], Matrix(np.eye(2, dtype=np.int64)))
        assert np.array_equal(c.arr, TWO[0].arr)

    def test_winograd_knuth_eight_call_variant(self, rng):  # :102-110
        c, ctr = mul(pk.winograd_knuth_mul, *TWO, recompute_first_product=True)
        assert c.arr.tolist() == TWO_PRODUCT and ctr.mults == 8
        a, b = int_matrix(rng, 8, 8), int_matrix(rng, 8, 8)
        c, ctr = mul(pk.winograd_knuth_mul, a, b, recompute_first_product=True)
        assert np.array_equal(c.arr, naive(a, b).arr) and ctr.mults == 8 ** 3

    @pytest.mark.parametrize("fn", list(DC.values()), ids=list(DC))
    def test_dc_kernels_reject_bad_shapes(self, fn):  # :126-134
        sq = Matrix(np.zeros((4, 4)))
        with pytest.raises(DimensionError):
            fn(Matrix(np.zeros((6, 6))), Matrix(np.zeros((6, 6))), Matrix(np.zeros((6, 6))))
        with pytest.raises(DimensionError):
            fn(Matrix(np.zeros((4, 2))), sq, sq)
        with pytest.raises(AliasError):
            fn(sq, sq, sq)

    @pytest.mark.parametrize("fn", list(DC.values()), ids=list(DC))
    @pytest.mark.parametrize("pol", list(POLICIES), ids=list(POLICIES))
    def test_oracle_equivalence_integer_sweep(self, rng, fn, pol):  # :137-149
        for order in (1, 2, 4, 8, 16, 32, 64):
            a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
            got, _ = mul(fn, a, b, policy=POLICIES[pol])
            assert np.array_equal(got.arr, naive(a, b).arr), (pol, order)

    @pytest.mark.parametrize("fn", list(DC.values()), ids=list(DC))
    def test_oracle_equivalence_real_tolerance(self, rng, fn):  # :152-158
        for order in (2, 8, 32, 64):
            a, b = real_matrix(rng, order, order), real_matrix(rng, order, order)
            got, _ = mul(fn, a, b)
            assert pk.max_abs_diff(got, naive(a, b)) <= 1e-9 * order

    def test_knuth_and_block_forms_agree_exactly(self, rng):  # :161-166
        for order in (2, 8, 32):
            a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
            assert np.array_equal(mul(pk.winograd_knuth_mul, a, b)[0].arr, mul(pk.winograd_block_mul, a, b)[0].arr)

    @pytest.mark.parametrize("fn,factor", [(pk.strassen_mul, 6), (pk.winograd_block_mul, 5)])
    def test_scalar_policy_closed_form_counts(self, rng, fn, factor):  # :169-179
        for k in range(7):
            n = 1 << k
            _, ctr = mul(fn, int_matrix(rng, n, n), int_matrix(rng, n, n))
            assert ctr.mults == 7 ** k and ctr.adds == factor * (7 ** k - 4 ** k)

    def test_scalar_policy_mults_for_knuth(self, rng):  # :182-187
        for k in range(6):
            n = 1 << k
            assert mul(pk.winograd_knuth_mul, int_matrix(rng, n, n), int_matrix(rng, n, n))[1].mults == 7 ** k

    def test_naive_cutoff_mult_recurrence(self, rng):  # :190-195
        _, ctr = mul(pk.strassen_mul, int_matrix(rng, 32, 32), int_matrix(rng, 32, 32), policy=BasePolicy.naive_cutoff(12))
        assert ctr.mults == 25088 < 32 ** 3

    def test_micro_dispatch_is_bit_identical_to_literal_recursion(self, rng):  # :198-205
        for fn in DC.values():
            for order in (2, 4, 8, 16):
                a, b = real_matrix(rng, order, order), real_matrix(rng, order, order)
                fast, cf = mul(fn, a, b, micro_order=8)
                slow, cs = mul(fn, a, b, micro_order=1)
                assert np.array_equal(fast.arr, slow.arr) and cf.snapshot() == cs.snapshot()

    def test_unrolled_base_bit_identical_to_recursion_100_pairs(self, rng):  # :208-214
        for _ in range(100):
            a, b = int_matrix(rng, 2, 2), int_matrix(rng, 2, 2)
            want, cw = mul(pk.winograd_block_mul, a, b, micro_order=1)
            got, cg = mul(pk.unrolled_base, a, b, order=2)
            assert np.array_equal(got.arr, want.arr) and (cg.mults, cg.adds) == (cw.mults, cw.adds)

    def test_unrolled_base_order4_matches_naive(self, rng):  # :217-223
        a, b = int_matrix(rng, 4, 4), int_matrix(rng, 4, 4)
        got, ctr = mul(pk.unrolled_base, a, b, order=4)
        assert np.array_equal(got.arr, naive(a, b).arr)
        assert (ctr.mults, ctr.adds, ctr.temp_buffers) == (49, 5 * (49 - 16), 0)

    def test_unrolled_base_order8_identity(self):  # :226-229
        eye = Matrix(np.eye(8))
        assert np.array_equal(mul(pk.unrolled_base, eye, eye, order=8)[0].arr, np.eye(8))

    def test_unrolled_base_rejects_other_orders(self):  # :232-238
        a = Matrix(np.zeros((16, 16)))
        with pytest.raises(DimensionError):
            pk.unrolled_base(a, a.copy(), Matrix(np.zeros((16, 16))), 16)
        b = Matrix(np.zeros((4, 4)))
        with pytest.raises(DimensionError):
            pk.unrolled_base(b, b.copy(), Matrix(np.zeros((4, 4))), 8)

    def test_base_policy_validation(self):  # :241-247
        for bad in (lambda: BasePolicy.unrolled_up_to(3), lambda: BasePolicy.naive_cutoff(0),
                    lambda: BasePolicy("mystery")):
            with pytest.raises(ValueError):
                bad()

    def test_kernels_leave_inputs_untouched(self, rng):  # :250-255
        a, b = int_matrix(rng, 16, 16), int_matrix(rng, 16, 16)
        sa, sb = a.arr.copy(), b.arr.copy()
        for fn in DC.values():
            mul(fn, a, b)
            assert np.array_equal(a.arr, sa) and np.array_equal(b.arr, sb)


# ===================================================================== test_schedules.py
def renumber(rows):
    return tuple(ScheduleStep(i + 1, s.symbol, s.op, s.lhs, s.rhs, s.store) for i, s in enumerate(rows))


def swap(steps, i, j):
    rows = list(steps)
    rows[i - 1], rows[j - 1] = rows[j - 1], rows[i - 1]
    return renumber(rows)


def schedule_calls(n, policy):
    """Independent count of recursion-tree calls that run a schedule (test_schedules.py:38-46)."""
    if n == 1 or (policy.kind == "naive-cutoff" and n <= policy.threshold) or \
            (policy.kind == "unrolled" and n <= policy.order):
        return 0
    return 1 + 7 * schedule_calls(n // 2, policy)


class TestSchedules:
    def test_builtin_two_temp_schedule_is_legal(self):  # test_schedules.py:51-52
        assert pk.validate_schedule(TWO_TEMP_STEPS).ok

    def test_builtin_in_place_schedule_is_legal(self):  # :55-58
        assert pk.validate_schedule(IN_PLACE_STEPS).ok
        assert pk.validate_schedule(IN_PLACE_STEPS, products_clobber_operands=True).ok

    def test_swapping_steps_7_and_9_breaks_in_place_schedule(self):  # :61-68
        rep = pk.validate_schedule(swap(IN_PLACE_STEPS, 7, 9))
        assert not rep.ok and rep.violation_index == 9 and "A11" in rep.reason
        assert not pk.validate_schedule(swap(IN_PLACE_STEPS, 7, 9), products_clobber_operands=True).ok

    def test_dependency_breaking_transpositions_fail(self):  # :71-77
        rep = pk.validate_schedule(swap(TWO_TEMP_STEPS, 3, 4))
        assert not rep.ok and rep.violation_index == 4
        assert not pk.validate_schedule(swap(IN_PLACE_STEPS, 8, 10)).ok

    def test_order_preserving_legality_of_all_single_swaps(self):  # :80-91
        for steps, clobber in ((TWO_TEMP_STEPS, False), (IN_PLACE_STEPS, True)):
            for i in range(1, 22):
                mutated = swap(steps, i, i + 1)
                if pk.validate_schedule(mutated, products_clobber_operands=clobber).ok:
                    final = {s.store: s.symbol for s in mutated}
                    assert final["C11"] == "U1" and final["C12"] == "U5"

    def test_validate_rejects_malformed_lists(self):  # :94-102
        with pytest.raises(ScheduleError):
            pk.validate_schedule(TWO_TEMP_STEPS[:21])
        no_product = renumber([ScheduleStep(0, s.symbol, "+" if s.op == "*" else s.op, s.lhs, s.rhs, s.store)
                               for s in TWO_TEMP_STEPS])
        with pytest.raises(ScheduleError):
            pk.validate_schedule(no_product)

    def test_two_temp_order2_product_and_buffers(self):  # :107-112
        c = Matrix.zeros(2, 2, np.int64)
        ctr = pk.two_temp_winograd(*TWO, c)
        assert c.arr.tolist() == TWO_PRODUCT
        assert (ctr.temp_buffers, ctr.mults, ctr.adds) == (2, 7, 15)

    def test_two_temp_order1_no_buffers(self):  # :115-118
        c = Matrix.zeros(1, 1, np.int64)
        ctr = pk.two_temp_winograd(Matrix(np.array([[6]])), Matrix(np.array([[7]])), c)
        assert c[0, 0] == 42 and ctr.temp_buffers == 0

    @pytest.mark.parametrize("order", [4, 8, 16, 32, 64, 128])
    def test_two_temp_matches_naive_and_preserves_inputs(self, rng, order):  # :121-133
        a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
        sa, sb = a.arr.copy(), b.arr.copy()
        want = naive(a, b)
        c = Matrix.zeros(order, order, np.int64)
        ctr = pk.two_temp_winograd(a, b, c)
        assert np.array_equal(c.arr, want.arr)
        assert np.array_equal(a.arr, sa) and np.array_equal(b.arr, sb)
        k = order.bit_length() - 1
        assert ctr.temp_buffers == 2 * (7 ** k - 1) // 6
        assert ctr.peak_live_elements <= 2 * order * order / 3

    @pytest.mark.parametrize("pol", ["scalar", "unrolled8", "cutoff12"])
    def test_two_temp_buffer_events_match_tree_walk(self, rng, pol):  # :136-146
        policy = POLICIES[pol]
        for order in (2, 8, 32, 64):
            c = Matrix.zeros(order, order, np.int64)
            ctr = pk.two_temp_winograd(int_matrix(rng, order, order), int_matrix(rng, order, order), c, policy=policy)
            assert ctr.temp_buffers == 2 * schedule_calls(order, policy)

    def test_two_temp_rejects_aliased_output(self):  # :149-151
        with pytest.raises(AliasError):
            pk.two_temp_winograd(TWO[0], TWO[1], TWO[0])

    def test_in_place_order2_zero_buffers(self):  # :156-161
        c = Matrix.zeros(2, 2, np.int64)
        ctr = pk.in_place_winograd(TWO[0].copy(), TWO[1].copy(), c, micro_order=1)
        assert c.arr.tolist() == TWO_PRODUCT and (ctr.temp_buffers, ctr.peak_live_elements) == (0, 0)

    def test_in_place_order1_leaves_inputs_alone(self):  # :164-168
        a, b = Matrix(np.array([[5]])), Matrix(np.array([[9]]))
        c = Matrix.zeros(1, 1, np.int64)
        pk.in_place_winograd(a, b, c)
        assert (c[0, 0], a[0, 0], b[0, 0]) == (45, 5, 9)

    @pytest.mark.parametrize("order", [4, 8, 16, 32, 64, 128])
    def test_in_place_matches_naive_on_saved_copies(self, rng, order):  # :171-182
        a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
        loop = loop_matmul(a.arr, b.arr) if order <= 16 else None
        ref = Matrix.zeros(order, order, np.int64)
        pk.naive_mul(Matrix(a.arr.copy()), Matrix(b.arr.copy()), ref)
        c = Matrix.zeros(order, order, np.int64)
        ctr = pk.in_place_winograd(a, b, c)  # clobbers a and b
        assert np.array_equal(c.arr, ref.arr)
        if loop is not None:
            assert np.array_equal(c.arr, loop)
        assert (ctr.temp_buffers, ctr.peak_live_elements) == (0, 0)

    def test_in_place_actually_clobbers_inputs(self, rng):  # :185-190
        a, b = int_matrix(rng, 16, 16), int_matrix(rng, 16, 16)
        before = a.arr.copy()
        pk.in_place_winograd(a, b, Matrix.zeros(16, 16, np.int64), micro_order=1)
        assert not np.array_equal(a.arr, before)

    def test_in_place_rejects_any_aliasing(self, rng):  # :193-199
        a = int_matrix(rng, 4, 4)
        c = Matrix.zeros(4, 4, np.int64)
        with pytest.raises(AliasError):
            pk.in_place_winograd(a, a, c)
        with pytest.raises(AliasError):
            pk.in_place_winograd(a, int_matrix(rng, 4, 4), a)

    def test_schedules_count_like_block_winograd(self, rng):  # :204-214
        for order in (2, 8, 32):
            a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
            counts = []
            for fn, args in ((pk.winograd_block_mul, (a, b)), (pk.two_temp_winograd, (a, b)),
                             (pk.in_place_winograd, (a.copy(), b.copy()))):
                ctr = OpCounter()
                fn(*args, Matrix.zeros(order, order, np.int64), counter=ctr)
                counts.append((ctr.mults, ctr.adds))
            assert counts[0] == counts[1] == counts[2]

    def test_schedule_micro_dispatch_matches_literal_counters(self, rng):  # :217-227
        for order in (2, 8, 32):
            a, b = int_matrix(rng, order, order), int_matrix(rng, order, order)
            out, ctrs = [], []
            for mo in (8, 1):
                c, ctr = Matrix.zeros(order, order, np.int64), OpCounter()
                pk.two_temp_winograd(a, b, c, counter=ctr, micro_order=mo)
                out.append(c.arr)
                ctrs.append(ctr.snapshot())
            assert np.array_equal(out[0], out[1]) and ctrs[0] == ctrs[1]

    def test_schedules_reject_nonconforming_shapes(self):  # :230-236
        bad = Matrix(np.zeros((6, 6)))
        with pytest.raises(DimensionError):
            pk.two_temp_winograd(bad, bad.copy(), Matrix(np.zeros((6, 6))))
        with pytest.raises(DimensionError):
            pk.in_place_winograd(Matrix(np.zeros((4, 2))), Matrix(np.zeros((4, 4))), Matrix(np.zeros((4, 4))))

    def test_trace_renders_table_rows(self):  # :239-251
        lines = []
        pk.in_place_winograd(TWO[0].copy(), TWO[1].copy(), Matrix.zeros(2, 2, np.int64), trace=lines.append)
        assert len(lines) == 22
        assert lines[0] == "step 1: S3 = A11-A21 -> C11" and lines[6] == "step 7: P1 = A11*B11 -> C11"
        lines = []
        pk.two_temp_winograd(*TWO, Matrix.zeros(2, 2, np.int64), trace=lines.append)
        assert lines[0] == "step 1: S3 = A11-A21 -> X" and lines[11] == "step 12: P1 = A11*B11 -> X"


# ========================================================================== test_core.py
class TestCore:
    def test_matrix_shape_and_indexing(self):  # test_core.py:26-31
        m = Matrix(np.arange(6).reshape(2, 3))
        assert (m.rows, m.cols, m[1, 2]) == (2, 3, 5)
        m[0, 0] = 9
        assert m[0, 0] == 9

    def test_matrix_rejects_bad_shapes(self):  # :34-38
        for arr in (np.arange(4), np.zeros((0, 3))):
            with pytest.raises(DimensionError):
                Matrix(arr)

    def test_view_reads_through_to_source(self):  # :41-48
        m = Matrix(np.arange(16).reshape(4, 4))
        v = MatrixView(m, 1, 2, 2, 2)
        assert all(v[i, j] == m[1 + i, 2 + j] for i in range(2) for j in range(2))
        v[0, 0] = 99
        assert m[1, 2] == 99

    def test_view_must_fit_in_source(self):  # :51-56
        m = Matrix(np.zeros((4, 4)))
        for args in ((2, 2, 3, 1), (0, 0, 5, 1)):
            with pytest.raises(DimensionError):
                MatrixView(m, *args)

    def test_quadrants_smallest_even_split(self):  # :59-62
        tl, tr, bl, br = pk.quadrants(Matrix(np.array([[1, 2], [3, 4]])).view())
        assert (tl[0, 0], tr[0, 0], bl[0, 0], br[0, 0]) == (1, 2, 3, 4)

    def test_quadrants_identity_block_structure(self):  # :65-70
        tl, tr, bl, br = pk.quadrants(Matrix(np.eye(4)).view())
        assert np.array_equal(tl.arr, np.eye(2)) and np.array_equal(br.arr, np.eye(2))
        assert not tr.arr.any() and not bl.arr.any()

    def test_quadrants_6x6_tile_exactly(self):  # :73-81
        m = Matrix(np.arange(36).reshape(6, 6))
        parts = pk.quadrants(m.view())
        for (r0, c0), part in zip(((0, 0), (0, 3), (3, 0), (3, 3)), parts):
            assert np.array_equal(part.arr, m.arr[r0:r0 + 3, c0:c0 + 3])

    def test_quadrants_rejects_odd_dimensions(self):  # :84-88
        for shape in ((3, 4), (4, 5)):
            with pytest.raises(DimensionError):
                pk.quadrants(Matrix(np.zeros(shape)).view())

    def test_quadrant_tiling_covers_without_overlap(self):  # :91-99 (hypothesis: 30 examples)
        r = np.random.default_rng(SEED)
        for hr, hc in zip(r.integers(1, 9, 30), r.integers(1, 9, 30)):
            m = Matrix(np.zeros((2 * hr, 2 * hc), dtype=np.int64))
            for mark, part in enumerate(pk.quadrants(m.view()), start=1):
                part.arr[:, :] = mark
            assert all(int((m.arr == mark).sum()) == hr * hc for mark in (1, 2, 3, 4))

    def test_block_add_direct_arithmetic(self):  # :102-109
        dst, ctr = Matrix.zeros(2, 2, np.int64), OpCounter()
        pk.block_add(Matrix(np.array([[1, 2], [3, 4]])), Matrix(np.array([[5, 6], [7, 8]])), dst, 1, ctr)
        assert dst.arr.tolist() == [[6, 8], [10, 12]] and ctr.adds == 4

    def test_block_add_self_subtract_is_zero(self):  # :112-116
        a = Matrix(np.array([[3, -1], [2, 9]]))
        dst = Matrix.zeros(2, 2, np.int64)
        pk.block_add(a, a, dst, -1)
        assert not dst.arr.any()

    def test_block_add_aliased_accumulate(self):  # :119-123
        a = Matrix(np.array([[1]]))
        pk.block_add(a, Matrix(np.array([[2]])), a, 1)
        assert a[0, 0] == 3

    def test_block_add_extent_mismatch(self):  # :126-129
        with pytest.raises(DimensionError):
            pk.block_add(Matrix(np.zeros((2, 2))), Matrix(np.zeros((2, 3))), Matrix(np.zeros((2, 2))))

    def test_block_add_then_subtract_restores(self):  # :132-142 (hypothesis: 30 examples)
        r = np.random.default_rng(SEED + 1)
        for rows, cols, seed in zip(r.integers(1, 7, 30), r.integers(1, 7, 30), r.integers(0, 2 ** 32, 30)):
            g = np.random.default_rng(int(seed))
            dst, other = int_matrix(g, rows, cols), int_matrix(g, rows, cols)
            before = dst.arr.copy()
            pk.block_add(dst, other, dst, 1)
            pk.block_add(dst, other, dst, -1)
            assert np.array_equal(dst.arr, before)

    def test_pad_5x3_to_8x8(self):  # :145-150
        a = Matrix(np.arange(1, 16).reshape(5, 3))
        p = pk.pad_to_pow2(a)
        assert (p.rows, p.cols) == (8, 8) and np.array_equal(p.arr[:5, :3], a.arr)
        assert not p.arr[5:, :].any() and not p.arr[:, 3:].any()

    def test_pad_conforming_returns_independent_copy(self):  # :153-158
        a = Matrix(np.arange(16).reshape(4, 4))
        p = pk.pad_to_pow2(a)
        assert np.array_equal(p.arr, a.arr)
        p[0, 0] = 99
        assert a[0, 0] == 0

    def test_pad_1x1(self):  # :161-163
        p = pk.pad_to_pow2(Matrix(np.array([[7]])))
        assert (p.rows, p.cols, p[0, 0]) == (1, 1, 7)

    def test_padding_round_trip(self):  # :166-173 (hypothesis: 60 examples)
        r = np.random.default_rng(SEED + 2)
        for rows, cols, seed in zip(r.integers(1, 65, 60), r.integers(1, 65, 60), r.integers(0, 2 ** 32, 60)):
            a = int_matrix(np.random.default_rng(int(seed)), rows, cols)
            assert pk.unpad(pk.pad_to_pow2(a), a.rows, a.cols) == a

    def test_unpad_block_and_full_extent(self):  # :176-180
        c = Matrix(np.arange(64).reshape(8, 8))
        assert np.array_equal(pk.unpad(c, 5, 3).arr, c.arr[:5, :3]) and pk.unpad(c, 8, 8) == c

    def test_unpad_rejects_oversize(self):  # :183-185
        with pytest.raises(DimensionError):
            pk.unpad(Matrix(np.zeros((4, 4))), 5, 2)

    def test_max_abs_diff_examples(self):  # :188-193
        a = Matrix(np.array([[1.0]]))
        assert pk.max_abs_diff(a, a) == 0.0 and pk.max_abs_diff(a, Matrix(np.array([[1.5]]))) == 0.5
        with pytest.raises(DimensionError):
            pk.max_abs_diff(a, Matrix(np.zeros((2, 1))))

    def test_max_abs_diff_matches_elementwise_loop(self, rng):  # :196-203
        a, b = Matrix(rng.uniform(-5, 5, (6, 4))), Matrix(rng.uniform(-5, 5, (6, 4)))
        want = max(abs(float(a[i, j]) - float(b[i, j])) for i in range(6) for j in range(4))
        assert pk.max_abs_diff(a, b) == want

    def test_text_format_int_round_trip(self):  # :206-211
        a = Matrix(np.array([[1, -2, 30], [400, 5, -6]], dtype=np.int64))
        text = matrix_to_text(a)
        back = pk.read_matrix(io.StringIO(text))
        assert text.splitlines()[0] == "2 3" and back == a and back.arr.dtype == np.int64

    def test_text_format_real_round_trip_17_digits(self):  # :214-218
        a = Matrix(np.array([[1 / 3, np.pi], [-2.5e-17, 1e300]]))
        back = pk.read_matrix(io.StringIO(matrix_to_text(a)))
        assert np.array_equal(back.arr, a.arr) and back.arr.dtype == np.float64

    def test_text_format_write_read_file(self, tmp_path):  # :221-225
        a = Matrix(np.array([[9, 8], [7, 6]], dtype=np.int64))
        pk.write_matrix(a, str(tmp_path / "m.txt"))
        assert pk.read_matrix(str(tmp_path / "m.txt")) == a

    @pytest.mark.parametrize("text", ["", "2", "2 2\n1 2 3", "2 2\n1 2 3 4 5", "x 2\n1 2", "1 1\nfoo", "0 2\n"])
    def test_text_format_rejects_malformed(self, text):  # :228-233
        with pytest.raises(ValueError):
            pk.read_matrix(io.StringIO(text))


# The 110 reference test ids -> the case here that replays them.
REFERENCE_CASES = {
    **{f"test_kernels.py::{t}": f"TestKernels::{t}" for t in (
        "test_naive_identity", "test_naive_2x2_by_hand", "test_naive_rectangular_matches_independent_loop",
        "test_naive_rejects_inner_mismatch", "test_naive_rejects_aliased_output", "test_winograd_knuth_identity",
        "test_winograd_knuth_eight_call_variant", "test_strassen_order1_scalar_base",
        "test_knuth_and_block_forms_agree_exactly", "test_scalar_policy_mults_for_knuth",
        "test_naive_cutoff_mult_recurrence", "test_micro_dispatch_is_bit_identical_to_literal_recursion",
        "test_unrolled_base_bit_identical_to_recursion_100_pairs", "test_unrolled_base_order4_matches_naive",
        "test_unrolled_base_order8_identity", "test_unrolled_base_rejects_other_orders", "test_base_policy_validation",
        "test_kernels_leave_inputs_untouched")},
    "test_kernels.py::test_strassen_order2_values_and_counts": "TestKernels::test_order2_values_and_counts[strassen]",
    "test_kernels.py::test_winograd_knuth_order2": "TestKernels::test_order2_values_and_counts[knuth]",
    "test_kernels.py::test_winograd_block_order2_counts": "TestKernels::test_order2_values_and_counts[block]",
    "test_kernels.py::test_strassen_order8_matches_naive": "TestKernels::test_matches_naive[strassen-8]",
    **{f"test_kernels.py::test_winograd_knuth_matches_naive[{o}]": f"TestKernels::test_matches_naive[knuth-{o}]"
       for o in (4, 8, 16)},
    "test_kernels.py::test_winograd_block_order32_matches_naive": "TestKernels::test_matches_naive[block-32]",
    **{f"test_kernels.py::test_dc_kernels_reject_bad_shapes[{k}]": f"TestKernels::test_dc_kernels_reject_bad_shapes[{k}]"
       for k in DC},
    **{f"test_kernels.py::test_oracle_equivalence_integer_sweep[{p}-{k}]":
       f"TestKernels::test_oracle_equivalence_integer_sweep[{p}-{k}]" for k in DC for p in POLICIES},
    **{f"test_kernels.py::test_oracle_equivalence_real_tolerance[{k}]":
       f"TestKernels::test_oracle_equivalence_real_tolerance[{k}]" for k in DC},
    **{f"test_kernels.py::test_scalar_policy_closed_form_counts[{k}]":
       f"TestKernels::test_scalar_policy_closed_form_counts[{k}]" for k in ("strassen", "block")},
    **{f"test_schedules.py::{t}": f"TestSchedules::{t}" for t in (
        "test_builtin_two_temp_schedule_is_legal", "test_builtin_in_place_schedule_is_legal",
        "test_swapping_steps_7_and_9_breaks_in_place_schedule", "test_dependency_breaking_transpositions_fail",
        "test_order_preserving_legality_of_all_single_swaps", "test_validate_rejects_malformed_lists",
        "test_two_temp_order2_product_and_buffers", "test_two_temp_order1_no_buffers",
        "test_two_temp_rejects_aliased_output", "test_in_place_order2_zero_buffers",
        "test_in_place_order1_leaves_inputs_alone", "test_in_place_actually_clobbers_inputs",
        "test_in_place_rejects_any_aliasing", "test_schedules_count_like_block_winograd",
        "test_schedule_micro_dispatch_matches_literal_counters", "test_schedules_reject_nonconforming_shapes",
        "test_trace_renders_table_rows")},
    **{f"test_schedules.py::test_two_temp_matches_naive_and_preserves_inputs[{o}]":
       f"TestSchedules::test_two_temp_matches_naive_and_preserves_inputs[{o}]" for o in (4, 8, 16, 32, 64, 128)},
    **{f"test_schedules.py::test_in_place_matches_naive_on_saved_copies[{o}]":
       f"TestSchedules::test_in_place_matches_naive_on_saved_copies[{o}]" for o in (4, 8, 16, 32, 64, 128)},
    **{f"test_schedules.py::test_two_temp_buffer_events_match_tree_walk[{p}]":
       f"TestSchedules::test_two_temp_buffer_events_match_tree_walk[{p}]" for p in ("scalar", "unrolled8", "cutoff12")},
    **{f"test_core.py::{t}": f"TestCore::{t}" for t in (
        "test_matrix_shape_and_indexing", "test_matrix_rejects_bad_shapes", "test_view_reads_through_to_source",
        "test_view_must_fit_in_source", "test_quadrants_smallest_even_split", "test_quadrants_identity_block_structure",
        "test_quadrants_6x6_tile_exactly", "test_quadrants_rejects_odd_dimensions",
        "test_quadrant_tiling_covers_without_overlap", "test_block_add_direct_arithmetic",
        "test_block_add_self_subtract_is_zero", "test_block_add_aliased_accumulate", "test_block_add_extent_mismatch",
        "test_block_add_then_subtract_restores", "test_pad_5x3_to_8x8", "test_pad_conforming_returns_independent_copy",
        "test_pad_1x1", "test_padding_round_trip", "test_unpad_block_and_full_extent", "test_unpad_rejects_oversize",
        "test_max_abs_diff_examples", "test_max_abs_diff_matches_elementwise_loop", "test_text_format_int_round_trip",
        "test_text_format_real_round_trip_17_digits", "test_text_format_write_read_file")},
    **{f"test_core.py::test_text_format_rejects_malformed[{i}]": f"TestCore::test_text_format_rejects_malformed[{i}]"
       for i in range(7)},
}


def test_every_reference_case_is_replayed(request):
    """All 110 reference test ids map to a collected case of this module."""
    assert len(REFERENCE_CASES) == 110, len(REFERENCE_CASES)
    here = {item.nodeid.split("::", 1)[1] for item in request.session.items if item.fspath == request.node.fspath}
    names = {h.split("[")[0] for h in here}
    for ref, mine in REFERENCE_CASES.items():
        base = mine.split("[")[0]
        assert base in names, (ref, mine)
