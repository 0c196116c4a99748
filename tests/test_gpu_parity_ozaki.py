"""The whole GPU parity suite again with INT8 tensor-core leaves (Ozaki scheme I, 8 slices).

Every test of test_gpu_parity.py is re-collected here and runs with
``set_leaf("ozaki", 8)``: integer data must stay bit-exact, real data must meet the same stated
bound and the same secondary gates (no larger than the reference CPU's own error on cfg3/cfg4).
Below them, direct tests of the C-ABI entry point ``mk_ozaki_dgemm``.
"""
import ctypes

import numpy as np
import pytest

import paper_2309_00628_b200 as pk
from conftest import has_gpu
from paper_2309_00628_b200 import _lib
from test_gpu_parity import *  # noqa: F401,F403  (re-collect every parity test under Ozaki leaves)

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(autouse=True)
def ozaki_leaves():
    pk.set_leaf("ozaki", 8, min_work=0)  # every leaf, however small, on the INT8 kernels
    assert pk.get_leaf() == ("ozaki", 8)
    yield
    pk.set_leaf("dmma")


def _dgemm(a, b, slices, ws_bytes=None):
    import torch

    m, k = a.shape
    n = b.shape[1]
    lib = _lib.load()
    c = torch.full((m, n), 7.0, dtype=torch.float64, device="cuda")
    need = lib.mk_ozaki_workspace_bytes(m, n, k, slices)
    ws = torch.empty(max(need, 256) + 256, dtype=torch.uint8, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = lib.mk_ozaki_dgemm(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0), m, n, k,
                            slices, ws.data_ptr(), need if ws_bytes is None else ws_bytes, st)
    torch.cuda.synchronize()
    return rc, c


@pytest.mark.parametrize("shape", [(1, 1, 1), (128, 64, 32), (300, 200, 260), (129, 65, 33), (64, 64, 1),
                                   (257, 130, 9000)])
@pytest.mark.parametrize("slices", [4, 8])
def test_ozaki_dgemm_integer_exact(shape, slices):
    """Integer data in the reference fixtures' range is exact at any slice count (the digits hold
    it), including ragged tiles and K above the int32 chunk limit (9000 > 4402: two K chunks)."""
    import torch

    m, n, k = shape
    r = np.random.default_rng(20240901 + m + n + k)
    a = torch.from_numpy(r.integers(-8, 9, (m, k)).astype(np.float64)).cuda()
    b = torch.from_numpy(r.integers(-8, 9, (k, n)).astype(np.float64)).cuda()
    rc, c = _dgemm(a, b, slices)
    assert rc == 0, _lib.load().mk_last_error()
    assert torch.equal(c, a @ b)


def test_ozaki_dgemm_accuracy_at_least_dmma():
    """8 slices (63 digit bits) against an extended-precision product: no larger error than the
    FP64 tensor-core (DMMA) product of the same operands."""
    import torch

    r = np.random.default_rng(20240901)
    an, bn = r.standard_normal((384, 512)), r.standard_normal((512, 320))
    exact = np.matmul(an.astype(np.longdouble), bn.astype(np.longdouble))
    a, b = torch.from_numpy(an).cuda(), torch.from_numpy(bn).cuda()
    rc, c = _dgemm(a, b, 8)
    assert rc == 0
    c_dmma = torch.empty_like(c)
    pk.set_leaf("dmma")
    pk.naive_mul(pk.Matrix(a), pk.Matrix(b), pk.Matrix(c_dmma))
    err_oz = float(np.abs(c.cpu().numpy().astype(np.longdouble) - exact).max())
    err_dmma = float(np.abs(c_dmma.cpu().numpy().astype(np.longdouble) - exact).max())
    assert err_oz <= err_dmma, (err_oz, err_dmma)


def test_ozaki_dgemm_nonfinite_rows_and_columns_are_nan():
    import torch

    r = np.random.default_rng(1)
    a = torch.from_numpy(r.uniform(-1, 1, (130, 70))).cuda()
    b = torch.from_numpy(r.uniform(-1, 1, (70, 90))).cuda()
    a[5, 3] = float("inf")
    b[7, 11] = float("nan")
    rc, c = _dgemm(a, b, 8)
    assert rc == 0
    ref = a @ b
    bad = torch.zeros_like(c, dtype=torch.bool)
    bad[5, :] = True
    bad[:, 11] = True
    assert torch.isnan(c[bad]).all()
    assert torch.allclose(c[~bad], ref[~bad], rtol=0, atol=1e-13)


def test_ozaki_dgemm_errors():
    import torch

    a = torch.zeros((64, 64), dtype=torch.float64, device="cuda")
    rc, _ = _dgemm(a, a, 3)
    assert rc == 5  # MK_ERR_ARG
    rc, _ = _dgemm(a, a, 8, ws_bytes=16)
    assert rc == 4  # MK_ERR_WORKSPACE
    with pytest.raises(ValueError):
        pk.set_leaf("ozaki", 9)
    with pytest.raises(ValueError):
        pk.set_leaf("int8")


def test_ozaki_dgemm_extreme_exponents():
    """Rows / columns whose maxima span the double range (down to subnormal scale, up to 1e300):
    every product stays within 8 ulps of its own magnitude scale (no overflow of the digit scale,
    no underflow of the recombination), like the FP64 product of the same data."""
    import torch

    r = np.random.default_rng(7)
    m, k, n = 130, 96, 70
    a = r.uniform(-1, 1, (m, k))
    b = r.uniform(-1, 1, (k, n))
    row_scale = np.array([1e-300, 1e-200, 1e-100, 1.0, 1e100, 1e150] * 22)[:m]
    col_scale = np.array([1e-150, 1e-20, 1.0, 1e20, 1e140] * 14)[:n]
    a *= row_scale[:, None]
    b *= col_scale[None, :]
    a[3, :] = 0.0  # a zero row
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    rc, c = _dgemm(at, bt, 8)
    assert rc == 0
    ref = np.matmul(a.astype(np.longdouble), b.astype(np.longdouble))
    bound = (np.abs(a).max(1)[:, None].astype(np.longdouble) * np.abs(b).max(0)[None, :].astype(np.longdouble)
             * k * 2.0 ** -50 + k * np.longdouble(2.0) ** -1074)  # + FP64 subnormal rounding
    err = np.abs(c.cpu().numpy().astype(np.longdouble) - ref)
    assert np.all(err <= bound), float((err / np.maximum(bound, 1e-300)).max())
    assert np.all(c[3].cpu().numpy() == 0.0)


def test_integer_guard_with_fewer_slices():
    """naive_mul on int64 n = 2048 with |a| ~ 2^35 and |b| < 2^6 passes the FP64 guard,
    but INT8 leaves with 4 slices would truncate a's low bits: it must raise, not return a wrong
    integer result; with 8 slices the same product is exact."""
    n = 2048
    r = np.random.default_rng(5)
    a = r.integers(2 ** 34, 2 ** 35, (n, n), dtype=np.int64) * r.choice([-1, 1], (n, n))
    b = r.integers(-63, 64, (n, n), dtype=np.int64)
    c = pk.Matrix.zeros(n, n, np.int64)
    try:
        pk.set_leaf("ozaki", 4, min_work=0)
        with pytest.raises(pk.ExactnessError):
            pk.naive_mul(pk.Matrix(a), pk.Matrix(b), c)
        pk.set_leaf("ozaki", 8, min_work=0)
        pk.naive_mul(pk.Matrix(a[:512, :512].copy()), pk.Matrix(b[:512, :512].copy()),
                     c2 := pk.Matrix.zeros(512, 512, np.int64))
        want = (a[:512, :512].astype(object) @ b[:512, :512].astype(object)).astype(np.int64)
        assert np.array_equal(c2.arr, want)
    finally:
        pk.set_leaf("ozaki", 8, min_work=0)
