"""Pipelined breadth-first plan (mk_engine.cu run_bfs_pipelined): leaves that take narrow 128 x 64
tiles run in kernels whose producer warps carry side work -- the next pass's operand transforms
and the previous pass's post-additions (mk_fused_gemm.cu side_work). Every transform and leaf is
the same computation as in the grouped plan, so integer-valued products are bit-exact against
numpy and the grouped plan, and real-valued ones agree within the stated tolerance
(reference: kernels.py:269-315 recursion, kernels.py:96-119 Winograd steps, hybrid.py:105-146)."""
import numpy as np
import pytest

import paper_2309_00628_b200 as pk
from oracle import strassen_oracle as o

pytestmark = pytest.mark.gpu

ALGOS = {
    "strassen": pk.strassen_mul,
    "winograd-block": pk.winograd_block_mul,
    "winograd-knuth": pk.winograd_knuth_mul,
    # eight top-level products (the first recomputed): eight passes, prologue and epilogue over 8
    "winograd-knuth-8call": lambda a, b, c, pol: pk.winograd_knuth_mul(a, b, c, pol, recompute_first_product=True),
}


def _grouped():
    pk.set_plan("breadth-first", group=4)


@pytest.fixture(autouse=True)
def _pipelined_for_every_narrow_leaf_call():
    """By default the pipelined plan is taken only when the leaves are long enough to hide
    transforms under (MK_OPT_PIPELINE = 1); these cases are small, so ask for it explicitly."""
    from paper_2309_00628_b200 import _lib

    lib = _lib.load(required=True)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_PIPELINE, 2), "mk_set_option")
    yield
    _lib.check(lib.mk_set_option(_lib.MK_OPT_PIPELINE, 1), "mk_set_option")


def test_small_calls_take_the_grouped_plan_by_default():
    """MK_OPT_PIPELINE = 1 (default): BASELINE cfg1 / cfg2 sized calls are launch-bound and run
    the grouped plan (same workspace as an explicit grouping of 4); cfg5 runs the pipelined one."""
    import ctypes

    from paper_2309_00628_b200 import _lib

    lib = _lib.load(required=True)
    v = ctypes.c_int(-1)
    assert lib.mk_get_option(_lib.MK_OPT_PIPELINE, ctypes.byref(v)) == 0 and v.value == 2
    assert lib.mk_set_option(_lib.MK_OPT_PIPELINE, 3) == _lib.MK_ERR_ARG
    forced = lib.mk_workspace_bytes(2, 1024, 4), lib.mk_rect_workspace_bytes(2, 12000, 10000, 14000, 5)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_PIPELINE, 1), "mk_set_option")
    auto = lib.mk_workspace_bytes(2, 1024, 4), lib.mk_rect_workspace_bytes(2, 12000, 10000, 14000, 5)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_PIPELINE, 0), "mk_set_option")
    off = lib.mk_workspace_bytes(2, 1024, 4), lib.mk_rect_workspace_bytes(2, 12000, 10000, 14000, 5)
    assert auto[0] == off[0] != forced[0]  # n = 1024, 64^3 leaves: grouped
    assert auto[1] == forced[1] != off[1]  # cfg5: pipelined


@pytest.mark.parametrize("algo", sorted(ALGOS))
@pytest.mark.parametrize("n,cut", [(512, 64), (1024, 64), (256, 32), (128, 32)])
def test_square_pipelined_matches_grouped_bitwise(algo, n, cut):
    """Square products with 64- and 32-column leaves (narrow tiles): integer data, pipelined
    (default) == grouped plan == exact product, bit for bit."""
    r = np.random.default_rng(n + cut)
    a = r.integers(-8, 9, (n, n)).astype(np.float64)
    b = r.integers(-8, 9, (n, n)).astype(np.float64)
    pol = pk.BasePolicy.naive_cutoff(cut)
    c1 = pk.Matrix.zeros(n, n)
    ALGOS[algo](pk.Matrix(a), pk.Matrix(b), c1, pol)
    try:
        _grouped()
        c2 = pk.Matrix.zeros(n, n)
        ALGOS[algo](pk.Matrix(a), pk.Matrix(b), c2, pol)
    finally:
        pk.set_plan()
    assert np.array_equal(c1.arr, a @ b)
    assert np.array_equal(c1.arr, c2.arr)


@pytest.mark.parametrize("shape,cut", [((1200, 1400, 1000), 128), ((3000, 3500, 2500), 256),
                                       ((700, 900, 650), 64), ((2400, 2800, 2000), 128)])
def test_rect_pipelined_exact_and_within_tolerance(shape, cut):
    """Rectangular driver (even-quadrant padding) at 3-5 levels with narrow leaves: integer data
    exact; real data within the oracle's tolerance of the float64 product."""
    m, k, n = shape
    r = np.random.default_rng(m)
    a = r.integers(-6, 7, (m, k)).astype(np.float64)
    b = r.integers(-6, 7, (k, n)).astype(np.float64)
    v = pk.get_variant("winograd-mod2", cutoff=cut)
    c = pk.multiply(pk.Matrix(a), pk.Matrix(b), v)
    assert np.array_equal(c.arr, a @ b)
    a = r.uniform(-1, 1, (m, k))
    b = r.uniform(-1, 1, (k, n))
    c = pk.multiply(pk.Matrix(a), pk.Matrix(b), v)
    err = float(np.abs(c.arr - a @ b).max())
    assert err <= o.tolerance(max(m, k, n), 1.0, 1.0), err


def test_pipelined_workspace_below_grouped_at_cfg5_shape():
    """cfg5 (12000x14000 . 14000x10000, cutoff 512 -> 5 levels): the pipelined plan's workspace
    (prologue sums + seven depth-1 outputs + three rotating pass regions) is below the grouped
    plan's (two passes of 4 and 3 top-level products)."""
    from paper_2309_00628_b200 import _lib

    lib = _lib.load(required=True)
    ws_pipe = lib.mk_rect_workspace_bytes(2, 12000, 10000, 14000, 5)
    try:
        _grouped()
        ws_grp = lib.mk_rect_workspace_bytes(2, 12000, 10000, 14000, 5)
    finally:
        pk.set_plan()
    assert 0 < ws_pipe < ws_grp, (ws_pipe, ws_grp)


@pytest.mark.parametrize("algo", sorted(ALGOS))
def test_pipelined_real_data_agrees_with_grouped(algo):
    """Real data: the pipelined plan (different pass structure, C formed by one epilogue) agrees
    with the grouped plan within the stated tolerance."""
    n, cut = 1024, 64
    r = np.random.default_rng(5)
    a = r.uniform(-1, 1, (n, n))
    b = r.uniform(-1, 1, (n, n))
    pol = pk.BasePolicy.naive_cutoff(cut)
    c1 = pk.Matrix.zeros(n, n)
    ALGOS[algo](pk.Matrix(a), pk.Matrix(b), c1, pol)
    try:
        _grouped()
        c2 = pk.Matrix.zeros(n, n)
        ALGOS[algo](pk.Matrix(a), pk.Matrix(b), c2, pol)
    finally:
        pk.set_plan()
    assert float(np.abs(c1.arr - c2.arr).max()) <= o.tolerance(n, 1.0, 1.0)
    assert float(np.abs(c1.arr - a @ b).max()) <= o.tolerance(n, 1.0, 1.0)
