"""Overlapped host path (mk_strassen_host, 2 levels): the top-level products between the first few
and the last run as one grouped breadth-first pass once every upload has landed
(mk_engine.cu host_group_range / fused_overlapped). Same products, same leaves; only the order in
which C's partial sums are added changes, so integer data stay bit-exact against numpy with the
pass forced to start after 1..4 products, off, and in auto mode -- from pinned and from pageable
(staged) host arrays, whose uploads alternate between two copy streams. Reference: the
recursion kernels.py:269-315 with the step tables kernels.py:66-160."""
import numpy as np
import pytest
import torch

import paper_2309_00628_b200 as pk
from paper_2309_00628_b200 import _lib

pytestmark = pytest.mark.gpu

ALGOS = {
    "strassen": pk.strassen_mul,
    "winograd-block": pk.winograd_block_mul,
    "winograd-knuth": pk.winograd_knuth_mul,
    "winograd-knuth-8call": lambda a, b, c, pol: pk.winograd_knuth_mul(a, b, c, pol, recompute_first_product=True),
}


def _set(v):
    lib = _lib.load(required=True)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_HOST_GROUP, v), "mk_set_option")


@pytest.mark.parametrize("algo", sorted(ALGOS))
@pytest.mark.parametrize("pinned", [True, False])
def test_grouped_middle_pass_exact_on_integers(algo, pinned):
    n = 2048
    r = np.random.default_rng(77)
    a = r.integers(-8, 9, (n, n)).astype(np.float64)
    b = r.integers(-8, 9, (n, n)).astype(np.float64)
    want = a @ b
    if pinned:
        ha, hb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
        hc = torch.empty((n, n), dtype=torch.float64).pin_memory()
        A, B, C = ha.numpy(), hb.numpy(), hc.numpy()
    else:
        A, B, C = a, b, np.empty((n, n))
    pol = pk.BasePolicy.naive_cutoff(512)
    try:
        for setting in (1, 2, 3, 4, 0, -1):
            _set(setting)
            C[:] = np.nan
            ALGOS[algo](pk.Matrix(A), pk.Matrix(B), pk.Matrix(C), pol)
            assert pk.last_stats().path == "overlapped-host"
            assert np.array_equal(C, want), (algo, pinned, setting)
    finally:
        _set(-1)


def test_grouped_middle_pass_on_reals_and_option_range():
    import ctypes

    lib = _lib.load(required=True)
    assert lib.mk_set_option(_lib.MK_OPT_HOST_GROUP, 7) == _lib.MK_ERR_ARG
    assert lib.mk_set_option(_lib.MK_OPT_HOST_GROUP, -2) == _lib.MK_ERR_ARG
    v = ctypes.c_int(5)
    assert lib.mk_get_option(_lib.MK_OPT_HOST_GROUP, ctypes.byref(v)) == 0 and v.value == -1
    n = 2048
    r = np.random.default_rng(5)
    a, b = r.standard_normal((n, n)), r.standard_normal((n, n))
    want = a @ b
    pol = pk.BasePolicy.naive_cutoff(512)
    outs = []
    try:
        for setting in (3, 0):
            _set(setting)
            c = np.empty((n, n))
            pk.winograd_block_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c), pol)
            assert pk.last_stats().path == "overlapped-host"
            outs.append(c)
    finally:
        _set(-1)
    tol = float(n) ** np.log2(12.0) * 2.0 ** -53 * np.abs(a).max() * np.abs(b).max()  # the stated bound, c = 1
    for c in outs:
        assert np.max(np.abs(c - want)) <= tol
    assert np.max(np.abs(outs[0] - outs[1])) < 1e-10
