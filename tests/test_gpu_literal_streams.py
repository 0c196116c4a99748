"""Side streams of the literal schedules (mk_engine.cu LitStreams / lit_wait): block additions of
Table 2 / Table 3 (reference schedules.py:62-112) that the next product does not depend on are
issued on side streams, ordered against the products by block-level hazard tracking. The steps,
their operands and their order per block are unchanged, so results -- and, for the in-place
schedule, the clobbered operands -- must be bit-identical to the one-stream execution, on real
data, at every depth, call after call (a missed hazard shows up as a differing or varying bit)."""
import ctypes

import numpy as np
import pytest
import torch

import paper_2309_00628_b200 as pk
from paper_2309_00628_b200 import _lib

pytestmark = pytest.mark.gpu


def _set_streams(on: bool):
    lib = _lib.load(required=True)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_LITERAL_STREAMS, 1 if on else 0), "mk_set_option")


def _run(fn, a, b, pol):
    """One call on device copies; returns (C, A after, B after)."""
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dc = torch.full_like(da, float("nan"))
    fn(pk.Matrix(da), pk.Matrix(db), pk.Matrix(dc), pol)
    torch.cuda.synchronize()
    return dc.cpu().numpy(), da.cpu().numpy(), db.cpu().numpy()


def test_option_round_trip():
    lib = _lib.load(required=True)
    v = ctypes.c_int(-1)
    assert lib.mk_get_option(_lib.MK_OPT_LITERAL_STREAMS, ctypes.byref(v)) == 0 and v.value == 1
    try:
        _set_streams(False)
        assert lib.mk_get_option(_lib.MK_OPT_LITERAL_STREAMS, ctypes.byref(v)) == 0 and v.value == 0
    finally:
        _set_streams(True)
    assert lib.mk_get_option(_lib.MK_OPT_LITERAL_STREAMS, ctypes.byref(v)) == 0 and v.value == 1


@pytest.mark.parametrize("name", ["in-place", "two-temp"])
@pytest.mark.parametrize("n,cut", [(256, 128), (512, 128), (512, 64), (1024, 128), (2048, 256), (2048, 1024), (256, 32)])
def test_side_streams_bit_identical_to_one_stream(name, n, cut):
    fn = pk.in_place_winograd if name == "in-place" else pk.two_temp_winograd
    r = np.random.default_rng(n * 7 + cut)
    a, b = r.standard_normal((n, n)), r.standard_normal((n, n))
    pol = pk.BasePolicy.naive_cutoff(cut)
    try:
        _set_streams(False)
        ref = _run(fn, a, b, pol)
    finally:
        _set_streams(True)
    for rep in range(3):
        got = _run(fn, a, b, pol)
        for x, y, what in zip(got, ref, ("C", "A after the call", "B after the call")):
            assert np.array_equal(x, y, equal_nan=True), (name, n, cut, rep, what)
    if name == "two-temp":  # operands untouched (schedules.py:332-341)
        assert np.array_equal(ref[1], a) and np.array_equal(ref[2], b)
    assert np.max(np.abs(ref[0] - a @ b)) < 1e-9 * n


@pytest.mark.parametrize("name", ["in-place", "two-temp"])
def test_side_streams_exact_on_integers_and_on_a_user_stream(name):
    """Integer data, 4 levels, issued on a non-default torch stream with work queued before and
    after on that stream: the fork / join around the side streams orders both."""
    fn = pk.in_place_winograd if name == "in-place" else pk.two_temp_winograd
    n = 1024
    r = np.random.default_rng(11)
    a = r.integers(-8, 9, (n, n)).astype(np.float64)
    b = r.integers(-8, 9, (n, n)).astype(np.float64)
    want = a @ b
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        da = torch.from_numpy(a).cuda(non_blocking=True) * 1.0  # produced on the same stream
        db = torch.from_numpy(b).cuda(non_blocking=True) * 1.0
        dc = torch.zeros_like(da)
        for _ in range(4):
            xa, xb = da.clone(), db.clone()
            fn(pk.Matrix(xa), pk.Matrix(xb), pk.Matrix(dc), pk.BasePolicy.naive_cutoff(64))
            out = dc * 1.0  # consumed on the same stream, no synchronisation in between
            dc.zero_()
    s.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)


def test_side_streams_from_two_host_threads():
    """Each host thread owns its side streams and event rings (thread-local LitStreams): two
    threads running the schedules at once, each on its own torch stream, both stay exact."""
    import threading

    n = 512
    r = np.random.default_rng(3)
    a = r.integers(-8, 9, (n, n)).astype(np.float64)
    b = r.integers(-8, 9, (n, n)).astype(np.float64)
    want = a @ b
    errors = []

    def work(fn, reps):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(reps):
                    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
                    dc = torch.zeros_like(da)
                    fn(pk.Matrix(da), pk.Matrix(db), pk.Matrix(dc), pk.BasePolicy.naive_cutoff(64))
                    s.synchronize()
                    if not np.array_equal(dc.cpu().numpy(), want):
                        errors.append(fn.__name__)
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(pk.in_place_winograd, 6)),
          threading.Thread(target=work, args=(pk.two_temp_winograd, 6))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def _set_pdl(on: bool):
    lib = _lib.load(required=True)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_PDL, 1 if on else 0), "mk_set_option")


@pytest.mark.parametrize("name", ["in-place", "two-temp", "winograd-block"])
@pytest.mark.parametrize("n,cut", [(256, 32), (1024, 128), (2048, 256), (2048, 1024)])
def test_programmatic_dependent_launches_bit_identical(name, n, cut):
    """MK_OPT_PDL (default on): sub-wave leaf launches and small additions become resident before
    their predecessor in the stream has finished and wait in griddepcontrol.wait. Same kernels in
    the same order: C -- and the in-place schedule's clobbered A and B -- must equal the plain
    stream-ordered run bit for bit on real data, call after call (a kernel touching global memory
    ahead of its wait would show up as a differing or varying bit)."""
    fn = {"in-place": pk.in_place_winograd, "two-temp": pk.two_temp_winograd,
          "winograd-block": pk.winograd_block_mul}[name]
    lib = _lib.load(required=True)
    v = ctypes.c_int(-1)
    assert lib.mk_get_option(_lib.MK_OPT_PDL, ctypes.byref(v)) == 0 and v.value == 1
    r = np.random.default_rng(n * 13 + cut)
    a, b = r.standard_normal((n, n)), r.standard_normal((n, n))
    pol = pk.BasePolicy.naive_cutoff(cut)
    try:
        _set_pdl(False)
        assert lib.mk_get_option(_lib.MK_OPT_PDL, ctypes.byref(v)) == 0 and v.value == 0
        ref = _run(fn, a, b, pol)
    finally:
        _set_pdl(True)
    for rep in range(3):
        got = _run(fn, a, b, pol)
        for x, y, what in zip(got, ref, ("C", "A after the call", "B after the call")):
            assert np.array_equal(x, y, equal_nan=True), (name, n, cut, rep, what)
    assert np.max(np.abs(ref[0] - a @ b)) < 1e-9 * n
