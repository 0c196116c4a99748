"""Device staging and engine calls.

Every compute entry point of the package funnels through here: operands are resolved to
(pointer, leading dimension) pairs of FP64 data in HBM, the C ABI is called on the current
torch CUDA stream, and results are written back to wherever the caller's output lives.

* Device operands (CUDA tensors, or views of them) that are FP64, unit-stride and 16-byte
  aligned are passed zero-copy.
* Host operands are copied host->device once per call (from pinned memory when the numpy
  array is a view of pinned storage), results device->host once.
* Integer operands are converted on the device (``mk_i64_to_f64``) after an exactness
  guard: max|a| * max|b| * n * 64**levels < 2**53 bounds every operand sum, leaf dot
  product and post-addition partial sum of an L-level Strassen/Winograd schedule (per
  level: operand sums grow <= 4x per side, destinations receive <= 4 contributions, the
  leaf order halves), so FP64 results are exact and convert back losslessly. There is no
  CPU fallback: a failing guard raises ExactnessError.
"""
from __future__ import annotations

import contextlib
import ctypes
import threading

import numpy as np

from . import _lib
from .core import AliasError, MatrixView, views_overlap
from .counters import EngineStats

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

_tls = threading.local()


def last_stats() -> EngineStats:
    st = getattr(_tls, "stats", None)
    if st is None:
        st = _tls.stats = EngineStats()
    return st


def _new_stats(**kw) -> EngineStats:
    _tls.stats = EngineStats(**kw)
    return _tls.stats


def require_engine():
    """The loaded library; raises EngineUnavailable without a CUDA device or the .so."""
    if torch is None or not torch.cuda.is_available():
        raise _lib.EngineUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return _lib.load(required=True)


def set_plan(plan: str = "breadth-first", two_temp_tail: bool = False, group: int = 0) -> None:
    """Process-wide engine plan (B200 addition; the reference has no counterpart).

    ``plan``: "breadth-first" (default for >= 2 levels: batched leaf launches, fastest),
    "hybrid" (top level depth-first, each top-level product breadth-first below it) or
    "depth-first" (workspace-minimal: operand sums only, each P_i accumulated straight into C by
    the leaf epilogue). ``group`` (breadth-first): top-level products per pass -- 0 = auto (4:
    two passes, about half the single-pass workspace), 7 = one pass (largest workspace), 1 = one
    top-level subtree at a time. ``two_temp_tail``: two_temp_winograd runs the literal Table-2
    schedule down to the leaves (default: the paper's two-temporary bound) or, if True, its last two
    levels breadth-first (faster at >= 3 levels, more scratch). Results are unchanged on integer
    data; float results differ only in summation order. Modeled OpCounter values never change.
    """
    kinds = {"breadth-first": 0, "depth-first": 1, "hybrid": 2}
    if plan not in kinds:
        raise ValueError(f"plan must be one of {sorted(kinds)}, got {plan!r}")
    if not 0 <= int(group) <= 8:
        raise ValueError(f"group must be in [0, 8], got {group!r}")
    lib = _lib.load(required=True)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_PLAN, kinds[plan]), "mk_set_option")
    _lib.check(lib.mk_set_option(_lib.MK_OPT_LITERAL_TAIL, 1 if two_temp_tail else 0), "mk_set_option")
    _lib.check(lib.mk_set_option(_lib.MK_OPT_BFS_GROUP, int(group)), "mk_set_option")


def set_leaf(kind: str = "dmma", slices: int = 8, min_work: int = 2 ** 29) -> None:
    """Process-wide leaf arithmetic (B200 addition; the reference's leaf is np.matmul, kernels.py:261).

    ``"dmma"`` (default): every leaf product on the FP64 tensor cores (mma.sync f64 -> DMMA).
    ``"ozaki"``: on the INT8 tensor cores (tcgen05.mma kind::i8, Ozaki scheme I): each operand
    row / column is split into ``slices`` (4..8) signed 7-bit digits under a power-of-two scale,
    the digit-pair products are exact int32 sums in tensor memory and are recombined in FP64.
    With 8 slices the leaf error is at or below the DMMA leaf's (63 digit bits vs 53) and integer
    data is exact whenever the FP64 guard passes; with fewer slices integer operands must also fit
    the digits (ozaki_exactness_guard: ExactnessError otherwise, never a silently truncated result). Fewer slices trade accuracy for speed. Modeled OpCounter values
    never change. ``min_work``: only leaf products with m*n*k >= min_work (rounded up to a power
    of two; default 2^29, about 812^3) use the INT8 kernels -- smaller leaves are launch- and
    wave-bound there and stay on DMMA (0: every leaf). Non-finite operand entries cannot be written
    as digits: an inf or NaN in a leaf operand's row (column) makes that whole row (column) of the
    leaf product NaN, where the FP64 product would give inf for some entries.
    """
    if kind not in ("dmma", "ozaki"):
        raise ValueError(f"leaf must be 'dmma' or 'ozaki', got {kind!r}")
    if kind == "ozaki" and not (4 <= int(slices) <= 8):
        raise ValueError(f"slices must be in [4, 8], got {slices!r}")
    if min_work < 0:
        raise ValueError("min_work must be >= 0")
    lib = _lib.load(required=True)
    _lib.check(lib.mk_set_option(_lib.MK_OPT_LEAF_SLICES, int(slices) if kind == "ozaki" else 0), "mk_set_option")
    log2 = 0 if min_work <= 1 else min(62, int(min_work - 1).bit_length())
    _lib.check(lib.mk_set_option(_lib.MK_OPT_LEAF_MIN_LOG2, log2), "mk_set_option")


def get_leaf() -> tuple:
    """(kind, slices) of the current leaf arithmetic (see set_leaf)."""
    lib = _lib.load(required=True)
    v = ctypes.c_int(0)
    _lib.check(lib.mk_get_option(_lib.MK_OPT_LEAF_SLICES, ctypes.byref(v)), "mk_get_option")
    return ("ozaki", v.value) if v.value else ("dmma", 0)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _vp(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


_INT_KINDS = ("i", "u", "b")


def _is_int(dt) -> bool:
    return np.dtype(dt).kind in _INT_KINDS


def _round_ld(cols: int) -> int:
    return (cols + 3) // 4 * 4


class Operand:
    """An FP64 device operand: `t` is a (rows x cols) CUDA view with stride (ld, 1)."""

    __slots__ = ("t", "rows", "cols", "keep")

    def __init__(self, t, rows, cols, keep=None):
        self.t, self.rows, self.cols, self.keep = t, rows, cols, keep

    @property
    def ptr(self) -> ctypes.c_void_p:
        return _vp(self.t)

    @property
    def ld(self) -> int:
        return int(self.t.stride(0))


def _fresh(rows: int, cols: int):
    """A new FP64 device block with a 32-byte aligned leading dimension."""
    buf = torch.empty((rows, _round_ld(cols)), dtype=torch.float64, device="cuda")
    return buf[:, :cols]


def _zero_copy_ok(t) -> bool:
    return (t.dtype == torch.float64 and t.stride(1) == 1 and t.stride(0) % 2 == 0
            and t.data_ptr() % 16 == 0 and t.stride(0) >= t.shape[1])


_SUPPORTED_KINDS = ("f", "i", "u", "b")


def check_dtype(*views) -> None:
    """The engine computes in FP64: real floating point and integer (exactness-guarded) operands
    only. Complex or object data raise TypeError (no silent truncation, no CPU fallback)."""
    for v in views:
        kind = np.dtype(v.dtype).kind
        if kind not in _SUPPORTED_KINDS:
            raise TypeError(f"unsupported operand dtype {v.dtype} for the FP64 engine (real or integer data only)")


def stage_in(view: MatrixView, *, copy: bool = False, stats: EngineStats | None = None) -> Operand:
    """Resolve a (host or device) view to an FP64 device operand."""
    check_dtype(view)
    rows, cols = view.rows, view.cols
    if view.on_device:
        t = view.arr
        if not copy and _zero_copy_ok(t):
            return Operand(t, rows, cols)
        out = _fresh(rows, cols)
        if t.dtype == torch.float64:
            out.copy_(t)
        elif t.dtype.is_floating_point:
            out.copy_(t.to(torch.float64))
        else:
            _convert_int_dev(t, out)
        return Operand(out, rows, cols)
    # host -> device
    src = torch.from_numpy(view.arr)  # strided host window; pinned if its storage is
    if stats is not None:
        stats.h2d_bytes += src.numel() * src.element_size()
    if _staged_ok(view.arr):  # large 8-byte rows: the engine's staged copy (bounce slots)
        lib = require_engine()
        if src.dtype == torch.float64:
            out = _fresh(rows, cols)
            _lib.check(lib.mk_copy_to_device(_vp(out), out.stride(0), ctypes.c_void_p(view.arr.ctypes.data),
                                             view.arr.strides[0] // 8, rows, cols, _stream()), "mk_copy_to_device")
            return Operand(out, rows, cols)
        dev = torch.empty((rows, cols), dtype=torch.int64, device="cuda")
        _lib.check(lib.mk_copy_to_device(_vp(dev), dev.stride(0), ctypes.c_void_p(view.arr.ctypes.data),
                                         view.arr.strides[0] // 8, rows, cols, _stream()), "mk_copy_to_device")
        out = _fresh(rows, cols)
        _convert_int_dev(dev, out)
        return Operand(out, rows, cols, keep=dev)
    if src.dtype == torch.float64:
        out = _fresh(rows, cols)
        out.copy_(src, non_blocking=src.is_pinned())
        return Operand(out, rows, cols)
    if src.dtype.is_floating_point:
        out = _fresh(rows, cols)
        out.copy_(src.to("cuda", non_blocking=src.is_pinned()).to(torch.float64))
        return Operand(out, rows, cols)
    dev = src.to("cuda", non_blocking=src.is_pinned())
    out = _fresh(rows, cols)
    _convert_int_dev(dev, out)
    return Operand(out, rows, cols, keep=dev)


_STAGED_MIN_BYTES = 8 << 20


def _staged_ok(arr) -> bool:
    """Large host blocks of 8-byte elements with unit column stride go through the engine's
    staged copies (mk_copy_to_device / mk_copy_to_host)."""
    return (arr.dtype.itemsize == 8 and arr.dtype.kind in "fi" and arr.ndim == 2 and arr.strides[1] == 8
            and arr.strides[0] % 8 == 0 and arr.strides[0] >= 8 * arr.shape[1] and arr.nbytes >= _STAGED_MIN_BYTES)


def _convert_int_dev(t, out) -> None:
    lib = require_engine()
    if t.dtype != torch.int64:
        t = t.to(torch.int64)
    if t.stride(1) != 1:
        t = t.contiguous()
    _lib.check(lib.mk_i64_to_f64(_vp(t), t.stride(0), _vp(out), out.stride(0), t.shape[0], t.shape[1], _stream()),
               "mk_i64_to_f64")


def absmax(view: MatrixView) -> float:
    """max |x| of a view, computed on the device."""
    lib = require_engine()
    t = view.arr if view.on_device else torch.from_numpy(np.ascontiguousarray(view.arr)).to("cuda")
    if t.stride(1) != 1:
        t = t.contiguous()
    out = ctypes.c_double(0.0)
    if t.dtype.is_floating_point:
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        rc = lib.mk_absmax_f64(_vp(t), t.stride(0), t.shape[0], t.shape[1], ctypes.byref(out), _stream())
    else:
        if t.dtype != torch.int64:
            t = t.to(torch.int64)
        rc = lib.mk_absmax_i64(_vp(t), t.stride(0), t.shape[0], t.shape[1], ctypes.byref(out), _stream())
    _lib.check(rc, "mk_absmax")
    return float(out.value)


def exactness_guard(a: MatrixView, b: MatrixView, inner: int, levels: int) -> None:
    """Raise ExactnessError unless an integer product is exactly representable (see module doc)."""
    ma, mb = absmax(a), absmax(b)
    bound = ma * mb * max(inner, 1) * (64.0 ** levels)
    if not bound < 2.0 ** 53:
        raise _lib.ExactnessError(
            f"integer operands too large for an exact FP64 engine run: max|a|*max|b|*n*64^L = {bound:.3e} >= 2^53"
        )
    kind, slices = get_leaf()
    if kind == "ozaki":
        ozaki_exactness_guard(ma, mb, levels, slices)


def ozaki_exactness_guard(ma: float, mb: float, levels: int, slices: int) -> None:
    """INT8 (Ozaki) leaves with S slices write a leaf operand row (column) scaled by 2^-e
    (|x| < 2^e) as a signed leading digit of weight 2^(e-7) and S-1 unsigned 8-bit digits
    below it, and drop the digit pairs s + t >= S. For integer data digit s is nonzero only if
    s <= ceil((e - 7) / 8) (lower digits cover weights below 2^0), so the product is exact iff
    ceil((e - 7)/8) + ceil((f - 7)/8) <= S - 1 (which also keeps every bit inside the S digits).
    Leaf operand sums grow by <= 4x per level and side: e and f are bounded from max|a| 4^L and
    max|b| 4^L. At S = 8 the FP64 bound above already implies the condition."""

    def exp2_above(x: float) -> int:  # smallest e with x < 2^e
        e = 0
        while x >= 2.0 ** e:
            e += 1
        return e

    def top_digit(e: int) -> int:
        return max(0, -(-(e - 7) // 8))

    e, f = exp2_above(ma * 4.0 ** levels), exp2_above(mb * 4.0 ** levels)
    if top_digit(e) + top_digit(f) > slices - 1:
        raise _lib.ExactnessError(
            f"integer operands too large for exact INT8 (Ozaki) leaves with {slices} slices: leaf operand "
            f"scales 2^{e}, 2^{f} put nonzero digits at {top_digit(e)} + {top_digit(f)} > {slices - 1} "
            f"(dropped digit pairs); use set_leaf('ozaki', 8) or set_leaf('dmma')")


class Output:
    """Where the engine writes C, and how the result reaches the caller's view."""

    def __init__(self, view: MatrixView, dtype, stats: EngineStats | None = None):
        self.view, self.dtype, self.stats = view, np.dtype(dtype), stats
        t = view.arr if view.on_device else None
        if t is not None and self.dtype == np.float64 and _zero_copy_ok(t) and t.stride(0) % 4 == 0 \
                and t.data_ptr() % 32 == 0:
            self.op = Operand(t, view.rows, view.cols)
            self.direct = True
        else:
            self.op = Operand(_fresh(view.rows, view.cols), view.rows, view.cols)
            self.direct = False

    def finish(self) -> None:
        if self.direct:
            return
        res = self.op.t
        if _is_int(self.dtype):
            lib = require_engine()
            ires = torch.empty((res.shape[0], res.shape[1]), dtype=torch.int64, device="cuda")
            _lib.check(lib.mk_f64_to_i64(_vp(res), res.stride(0), _vp(ires), ires.stride(0), res.shape[0],
                                         res.shape[1], _stream()), "mk_f64_to_i64")
            res = ires
        if self.view.on_device:
            self.view.arr.copy_(res)
            return
        host = self.view.arr
        if self.stats is not None:
            self.stats.d2h_bytes += res.shape[0] * res.shape[1] * res.element_size()
        if not host.flags.writeable:
            raise ValueError("output view is read-only")
        want = getattr(torch, self.dtype.name)
        src = res if res.dtype == want else res.to(want)
        if _staged_ok(host) and src.stride(1) == 1:
            lib = require_engine()
            _lib.check(lib.mk_copy_to_host(ctypes.c_void_p(host.ctypes.data), host.strides[0] // 8, _vp(src),
                                           src.stride(0), src.shape[0], src.shape[1], _stream()), "mk_copy_to_host")
            return
        torch.from_numpy(host).copy_(src)


def check_disjoint(a: MatrixView, b: MatrixView, c: MatrixView) -> None:
    """Output must not overlap an input (reference kernels.py:330-332)."""
    if views_overlap(c, a) or views_overlap(c, b):
        raise AliasError("output view must not alias an input view")


# Engine workspaces are kept per (device, stream, thread) and reused by later calls of that thread on
# that stream (work on one stream is ordered, so reuse is safe even while earlier calls still run): a 15.5 GB
# breadth-first workspace is neither re-requested from the allocator nor re-checked against free
# device memory on every call (either occasionally stalled the host for tens of ms).
_ws_cache: dict = {}
_ws_lock = threading.Lock()


def _ws_key():
    # per calling thread too: two threads enqueueing on one stream interleave their launches
    return (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream, threading.get_ident())


def workspace(nbytes: int):
    nbytes = max(int(nbytes), 16)
    key = _ws_key()
    with _ws_lock:
        t = _ws_cache.get(key)
        if t is not None and t.numel() >= nbytes:
            return t
        _ws_cache.pop(key, None)  # a smaller one goes back to torch's stream-ordered cache first
    t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    with _ws_lock:
        _ws_cache[key] = t
    return t


def release_workspaces() -> None:
    """Drop the cached engine workspaces (their memory returns to torch's caching allocator)."""
    with _ws_lock:
        _ws_cache.clear()



_WS_MARGIN = 256 << 20
_WS_QUERY_MIN = 1 << 30  # workspaces below 1 GiB are allocated without asking the driver first


def _fits(nbytes: int) -> bool:
    """Whether a workspace of nbytes can be allocated now (this stream's cached workspace, else free
    device memory plus what torch's caching allocator holds unused)."""
    with _ws_lock:
        t = _ws_cache.get(_ws_key())
    if t is not None and t.numel() >= nbytes:
        return True
    free, _ = torch.cuda.mem_get_info()
    slack = torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    return nbytes + _WS_MARGIN <= free + slack


@contextlib.contextmanager
def _memory_aware_plan(size_of, levels: int = 3):
    """Yield the workspace size for this call. When the configured plan's workspace does not fit
    in device memory, the call runs with leaner options instead -- the hybrid plan first for
    deep recursions (breadth-first speed at ~1/7 of the memory), else the depth-first plan and the
    literal two-temp schedule (same results on integer data). The leaner options are set as
    calling-thread overrides (mk_set_thread_option) for both the sizing and the launch inside the
    ``with`` block, then removed: other threads' options are never touched, and another thread's
    set_plan() cannot change this call's plan between its sizing and its launch."""
    need = int(size_of())
    if need < _WS_QUERY_MIN or _fits(need):  # small workspaces: skip the (~0.7 ms) memory query
        yield need
        return
    lib = _lib.load(required=True)
    try:
        _lib.check(lib.mk_set_thread_option(_lib.MK_OPT_LITERAL_TAIL, 0), "mk_set_thread_option")
        need = -1
        if levels >= 3:  # at <= 2 levels depth-first is as fast and smaller
            _lib.check(lib.mk_set_thread_option(_lib.MK_OPT_PLAN, 2), "mk_set_thread_option")  # hybrid
            need = int(size_of())
        if need < 0 or not _fits(need):
            _lib.check(lib.mk_set_thread_option(_lib.MK_OPT_PLAN, 1), "mk_set_thread_option")  # depth-first
            need = int(size_of())
        yield need
    finally:
        lib.mk_set_thread_option(_lib.MK_OPT_PLAN, -1)
        lib.mk_set_thread_option(_lib.MK_OPT_LITERAL_TAIL, -1)


# ---------------------------------------------------------------------------------
# Engine calls
# ---------------------------------------------------------------------------------

def device_gemm(a: MatrixView, b: MatrixView, c: MatrixView, dtype) -> None:
    """C = A B on the DMMA kernel (mk_dgemm); replaces _naive_arrays kernels.py:258-266."""
    lib = require_engine()
    check_dtype(a, b, c)
    st = _new_stats(algo="naive")
    if _is_int(dtype):
        exactness_guard(a, b, a.cols, 0)
    A, B = stage_in(a, stats=st), stage_in(b, stats=st)
    out = Output(c, dtype, st)
    C = out.op
    rc = lib.mk_dgemm(A.ptr, A.ld, B.ptr, B.ld, C.ptr, C.ld, a.rows, b.cols, a.cols, _stream())
    _lib.check(rc, "mk_dgemm")
    out.finish()


def levels_for(n: int, policy, algo: str) -> int:
    """Engine recursion depth for the reference's base policy (mk_levels_for_policy)."""
    lib = require_engine()
    kind = {"scalar": 0, "unrolled": 1, "naive-cutoff": 2}[policy.kind]
    param = policy.order if policy.kind == "unrolled" else policy.threshold
    lv = ctypes.c_int(0)
    _lib.check(lib.mk_levels_for_policy(n, kind, param, _lib.ALGO_IDS[algo], ctypes.byref(lv)),
               "mk_levels_for_policy")
    return int(lv.value)


_PIPE_ALGOS = ("strassen", "winograd-block", "winograd-knuth", "winograd-knuth-8call")
_copy_streams: dict = {}  # device index -> copy stream of the overlapped host path


def _copy_stream():
    dev = torch.cuda.current_device()
    if dev not in _copy_streams:
        _copy_streams[dev] = torch.cuda.Stream(device=dev)
    return _copy_streams[dev]


def _overlap_applies(a: MatrixView, b: MatrixView, c: MatrixView, levels: int, algo: str, dtype) -> bool:
    """Whether the overlapped host path applies: FP64 host operands and result with unit column
    stride (pinned memory is copied by DMA directly; pageable arrays go through the engine's
    pinned bounce slots), large enough for transfers to matter, one of the fused algorithms.
    MK_PIPELINE=0 disables it."""
    import os

    if os.environ.get("MK_PIPELINE", "1") == "0" or algo not in _PIPE_ALGOS or levels < 1:
        return False
    if a.on_device or b.on_device or c.on_device or np.dtype(dtype) != np.float64:
        return False
    if not (a.dtype == b.dtype == c.dtype == np.float64) or not c.arr.flags.writeable or a.rows < 2048:
        return False
    return all(v.arr.strides[1] == 8 and v.arr.strides[0] % 8 == 0 for v in (a, b, c))


def _overlapped_host_product(algo: str, a: MatrixView, b: MatrixView, c: MatrixView, levels: int,
                             st: EngineStats) -> None:
    """C = A B for host operands through mk_strassen_host: operand blocks go up on copy
    streams in the order the compute first needs them, each top-level product (or child)
    starts as soon as the blocks it reads have landed, each C block comes back as soon as its
    last contributor is done. Pageable arrays are staged through pinned bounce slots by the
    engine's host thread pool."""
    lib = require_engine()
    n = a.rows
    ld = _round_ld(n)
    dA = torch.empty((n, ld), dtype=torch.float64, device="cuda")
    dB = torch.empty((n, ld), dtype=torch.float64, device="cuda")
    dC = torch.empty((n, ld), dtype=torch.float64, device="cuda")
    aid = _lib.ALGO_IDS[algo]
    with _memory_aware_plan(lambda: lib.mk_host_workspace_bytes(aid, n, levels), levels) as ws_bytes:
        ws = workspace(ws_bytes)
        st.workspace_bytes = ws_bytes
        st.path = "overlapped-host"
        rc = _call_host(lib, aid, a, b, c, n, levels, dA, dB, dC, ld, ws, ws_bytes)
    _lib.check(rc, f"mk_strassen_host({algo})")
    st.h2d_bytes += 2 * n * n * 8
    st.d2h_bytes += n * n * 8


def _call_host(lib, aid, a, b, c, n, levels, dA, dB, dC, ld, ws, ws_bytes):
    return lib.mk_strassen_host(aid, ctypes.c_void_p(a.arr.ctypes.data), a.arr.strides[0] // 8,
                                ctypes.c_void_p(b.arr.ctypes.data), b.arr.strides[0] // 8,
                                ctypes.c_void_p(c.arr.ctypes.data), c.arr.strides[0] // 8, n, levels, _vp(dA), _vp(dB),
                                _vp(dC), ld, _vp(ws), ws_bytes, _stream(), ctypes.c_void_p(_copy_stream().cuda_stream))


def device_square(algo: str, a: MatrixView, b: MatrixView, c: MatrixView, levels: int, dtype,
                  clobber_inputs: bool = False) -> None:
    """Square power-of-two product through mk_strassen.

    With ``clobber_inputs`` (the in-place schedule, schedules.py:344-353) the engine works in
    device copies of A and B whose final (clobbered) contents are written back to the caller's
    views, so host callers observe the same "inputs destroyed" contract as the reference.
    """
    lib = require_engine()
    check_dtype(a, b, c)
    st = _new_stats(algo=algo, levels=levels)
    n = a.rows
    if _is_int(dtype):
        exactness_guard(a, b, n, levels)
    if not clobber_inputs and _overlap_applies(a, b, c, levels, algo, dtype):
        _overlapped_host_product(algo, a, b, c, levels, st)
        return
    A = stage_in(a, copy=clobber_inputs and a.on_device and not _zero_copy_ok(a.arr), stats=st)
    B = stage_in(b, copy=clobber_inputs and b.on_device and not _zero_copy_ok(b.arr), stats=st)
    out = Output(c, dtype, st)
    C = out.op
    aid = _lib.ALGO_IDS[algo]
    with _memory_aware_plan(lambda: lib.mk_workspace_bytes(aid, n, levels), levels) as ws_bytes:
        st.workspace_bytes = ws_bytes
        ws = workspace(ws_bytes)
        rc = lib.mk_strassen(aid, A.ptr, A.ld, B.ptr, B.ld, C.ptr, C.ld, n, levels, _vp(ws), ws_bytes, _stream())
    _lib.check(rc, f"mk_strassen({algo})")
    out.finish()
    if clobber_inputs:
        for src, op in ((a, A), (b, B)):
            if op.t is src.arr:
                continue  # engine already worked in the caller's storage
            _write_back(src, op.t)


def _write_back(view: MatrixView, t) -> None:
    """Copy engine-side (clobbered) FP64 contents back into the caller's view."""
    dt = np.dtype(view.dtype)
    if _is_int(dt):
        vals = torch.round(t).to(torch.int64)
    else:
        vals = t.to(getattr(torch, dt.name))
    if view.on_device:
        view.arr.copy_(vals)
    else:
        if not view.arr.flags.writeable:
            return
        torch.from_numpy(view.arr).copy_(vals.cpu())


def device_rect(algo: str, a: MatrixView, b: MatrixView, c: MatrixView, levels: int, dtype) -> None:
    """Rectangular product with even-quadrant padding (mk_multiply_rect)."""
    lib = require_engine()
    check_dtype(a, b, c)
    st = _new_stats(algo=algo, levels=levels)
    m, k, n = a.rows, a.cols, b.cols
    if _is_int(dtype):
        exactness_guard(a, b, k, levels)
    A, B = stage_in(a, stats=st), stage_in(b, stats=st)
    out = Output(c, dtype, st)
    C = out.op
    aid = _lib.ALGO_IDS[algo]
    with _memory_aware_plan(lambda: lib.mk_rect_workspace_bytes(aid, m, n, k, levels), levels) as ws_bytes:
        st.workspace_bytes = ws_bytes
        ws = workspace(ws_bytes)
        rc = lib.mk_multiply_rect(aid, A.ptr, A.ld, B.ptr, B.ld, C.ptr, C.ld, m, n, k, levels, _vp(ws), ws_bytes,
                                  _stream())
    _lib.check(rc, f"mk_multiply_rect({algo})")
    out.finish()


def device_block_combine(dst: MatrixView, terms) -> None:
    """dst = sum sign_i * view_i on the device (mk_block_combine)."""
    lib = require_engine()
    dtype = np.result_type(*[v.dtype for v, _ in terms], dst.dtype)
    ops = [stage_in(v) for v, _ in terms]
    out = Output(dst, dst.dtype if dst.dtype == dtype else dtype)
    C = out.op
    n = len(ops)
    ptrs = (ctypes.c_void_p * n)(*[o.t.data_ptr() for o in ops])
    lds = (ctypes.c_int64 * n)(*[o.ld for o in ops])
    sg = (ctypes.c_double * n)(*[float(s) for _, s in terms])
    rc = lib.mk_block_combine(C.ptr, C.ld, ptrs, lds, sg, n, dst.rows, dst.cols, _stream())
    _lib.check(rc, "mk_block_combine")
    out.finish()
