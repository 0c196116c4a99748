"""Stream-K tail of the persistent DMMA kernel: launches whose tiles leave the last wave partial
split the k-iterations of the tail over every SM and the last-arriving segment of each tile adds
the others' partial sums in k order. Integer data must stay bit-exact for every split pattern:
tiles split over 2-3 CTAs, CTAs with empty shares (launches smaller than one wave), ragged M/N/K
edges, the data-parallel + stream-K mix of larger launches, and batched leaf launches."""
import numpy as np
import pytest

import paper_2309_00628_b200 as pk
from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.mark.parametrize("m,n,k", [(128, 128, 4096), (64, 512, 512), (256, 384, 1000), (1024, 1024, 1024),
                                   (2048, 2048, 2048), (3000, 2500, 1234), (130, 6000, 700), (5000, 130, 2000),
                                   (8 * 128, 19 * 128, 3 * 16 + 5), (1536, 1664, 4096)])
def test_streamk_dgemm_exact(m, n, k):
    r = np.random.default_rng(m * 7 + n * 3 + k)
    a = r.integers(-8, 9, (m, k)).astype(np.float64)
    b = r.integers(-8, 9, (k, n)).astype(np.float64)
    c = pk.Matrix.zeros(m, n)
    for _ in range(2):  # second call reuses the stream's flags (reset by the previous launch)
        pk.naive_mul(pk.Matrix(a), pk.Matrix(b), c)
        assert np.array_equal(c.arr, a @ b)


def test_streamk_deterministic_on_reals():
    """The split and the summation order are fixed: repeated runs are bit-identical."""
    r = np.random.default_rng(9)
    a, b = r.uniform(-1, 1, (1000, 3000)), r.uniform(-1, 1, (3000, 900))
    outs = []
    for _ in range(3):
        c = pk.Matrix.zeros(1000, 900)
        pk.naive_mul(pk.Matrix(a), pk.Matrix(b), c)
        outs.append(c.arr.copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    assert float(np.abs(outs[0] - a @ b).max()) < 1e-11


@pytest.mark.parametrize("fn", ["in_place_winograd", "two_temp_winograd", "winograd_block_mul"])
def test_streamk_leaf_launches_exact(fn):
    """Literal schedules launch 1024^2 leaves one at a time (all stream-K); the breadth-first plan's
    batched launches get a stream-K tail."""
    n = 4096
    r = np.random.default_rng(4)
    a = r.integers(-8, 9, (n, n)).astype(np.float64)
    b = r.integers(-8, 9, (n, n)).astype(np.float64)
    c = pk.Matrix.zeros(n, n)
    getattr(pk, fn)(pk.Matrix(a.copy()), pk.Matrix(b.copy()), c, pk.BasePolicy.naive_cutoff(512))
    assert np.array_equal(c.arr, a @ b)
