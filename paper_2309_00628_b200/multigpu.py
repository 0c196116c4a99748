"""Multi-GPU Strassen-Winograd: the 7^L leaf products of one multiplication spread over the
GPUs of one node, partial C blocks sum-reduced over NVLink.

Decomposition. An L-level product is a sum of 7^L leaf contributions (Kronecker powers of
the one-level coefficients); each leaf's output rows are independent, so the shard unit is a
leaf row panel (``PANELS`` per leaf). Rank r of W computes a contiguous range of units in
level-major order (``shard_range``): every rank gets the same amount of work, and leaves sharing
an outer-level operand sum land on the same rank, where that sum is materialised once. Each rank accumulates its leaves
into a zero-initialised partial C with the fused multi-destination epilogue
(``mk_strassen_partial``); the partials are then summed with one collective
(``torch.distributed.reduce``, NCCL on GPUs, gloo in the CPU tests). That reduce is the
path's only exchange step: operands are replicated (inputs resident on every GPU, as
BASELINE.json's multi-GPU config states) and nothing else crosses GPUs.

Load balance: with whole leaves 49 over 8 GPUs would cap efficiency at 49/56; in row-panel
units (49 x 8 = 392) the split is exact.

Fused alternative (``fused_sharded_multiply``): C is split into W row slabs, slab r owned by
rank r; every rank maps all slabs (its own local, the others through CUDA IPC handles exchanged
with the process group -- NVLink peer memory on a multi-GPU node) and its leaf epilogue adds each
contribution straight into the owning rank's slab (``mk_strassen_partial_slabs``, REDG.ADD.F64):
the compute and the reduce-scatter are one kernel, there is no partial-C buffer and no reduce
collective. Rank 0 then pulls the other slabs over peer memory if it needs the whole C.
"""
from __future__ import annotations

import ctypes

from . import _lib, tables

PANELS = 8  # row panels per leaf (shard granularity)

_STEPS = {
    "strassen": tables.STRASSEN_STEPS,
    "winograd-block": tables.WINOGRAD_BLOCK_STEPS,
    "winograd-knuth": tables.WINOGRAD_KNUTH_STEPS,
    "winograd-knuth-8call": tables.WINOGRAD_KNUTH_8CALL_STEPS,
}


def operand_quadrants(algo: str, levels: int, first: int, count: int, panels: int = PANELS):
    """Top-level quadrants of A and B (0..3 = 11, 12, 21, 22) that shard units
    [first, first+count) read: the units of one top-level product read only the quadrants in
    its operand sums, so a rank needs only those uploaded (the rest of its A/B buffers is never
    touched)."""
    if levels < 1 or count <= 0:
        return (set(range(4)), set(range(4))) if count > 0 else (set(), set())
    a, b, _ = tables.coefficients(_STEPS[algo])
    per_parent = len(a) ** (levels - 1) * panels
    qa, qb = set(), set()
    for p in range(first // per_parent, (first + count - 1) // per_parent + 1):
        qa |= {q for q in range(4) if a[p][q]}
        qb |= {q for q in range(4) if b[p][q]}
    return qa, qb


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [first, first+count) of ``total`` leaf products for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def leaf_count(algo: str, levels: int) -> int:
    lib = _lib.load()
    n = lib.mk_product_count(_lib.ALGO_IDS[algo], levels)
    if n < 0:
        raise ValueError(f"{algo} has no leaf-product form")
    return n


def _check_operand(t, name: str) -> None:
    """The ABI reads row-major FP64 with unit column stride: anything else would be read as wrong
    data without an error, so refuse it here."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64, got {t.dtype}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{name} must be a 2-D view with unit column stride, got strides {tuple(t.stride())}")


def _workspace(need: int, ws, device, stream):
    """A workspace of >= need bytes for kernels queued on ``stream``: a caller-provided one, or a
    fresh one whose memory the caching allocator keeps reserved until ``stream`` has finished
    with it (record_stream), since it is freed on return while the kernels may still run."""
    import torch

    if ws is not None and ws.numel() >= need:
        return ws
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=device)
    if stream is not None:
        ws.record_stream(stream)
    return ws


def partial_product(algo: str, a, b, c_partial, levels: int, first: int, count: int, stream=None, ws=None,
                    panels: int = PANELS) -> int:
    """c_partial += shard units [first, first+count) of A B (all CUDA FP64, square order n).

    ``c_partial`` must be zero-initialised (or hold earlier partial sums). Returns the
    workspace bytes used.
    """
    import torch

    lib = _lib.load()
    for t, nm in ((a, "a"), (b, "b"), (c_partial, "c_partial")):
        _check_operand(t, nm)
    n = a.shape[0]
    aid = _lib.ALGO_IDS[algo]
    need = int(lib.mk_partial_workspace_bytes(aid, n, levels))
    ws = _workspace(need, ws, a.device, stream)
    st = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    rc = lib.mk_strassen_partial(aid, ctypes.c_void_p(a.data_ptr()), a.stride(0), ctypes.c_void_p(b.data_ptr()),
                                 b.stride(0), ctypes.c_void_p(c_partial.data_ptr()), c_partial.stride(0), n, levels,
                                 first, count, panels, ctypes.c_void_p(ws.data_ptr()), need, st)
    _lib.check(rc, "mk_strassen_partial")
    return need


def assemble(partial, dst_rank: int = 0, group=None):
    """Sum the ranks' partial C blocks onto ``dst_rank`` (the path's single exchange step)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if partial.is_cuda and dist.get_backend(group) == "gloo":  # plumbing checks on one GPU
            host = partial.cpu()
            dist.reduce(host, dst=dst_rank, op=dist.ReduceOp.SUM, group=group)
            partial.copy_(host)
        else:
            dist.reduce(partial, dst=dst_rank, op=dist.ReduceOp.SUM, group=group)
    return partial


def my_shard(algo: str, levels: int, group=None) -> tuple[int, int]:
    """This rank's [first, first+count) shard units."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return shard_range(leaf_count(algo, levels) * PANELS, world, rank)


def upload_operands(algo: str, levels: int, host_a, host_b, dev_a, dev_b, group=None, stream=None) -> int:
    """Copy to this rank's device buffers only the operand quadrants its shard reads (pinned or
    pageable host tensors/arrays of order n; the engine's staged copies). Returns the bytes."""
    import numpy as np
    import torch

    lib = _lib.load()
    first, count = my_shard(algo, levels, group)
    qa, qb = operand_quadrants(algo, levels, first, count)
    n = dev_a.shape[0]
    h = n // 2 if levels >= 1 else n
    st = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    moved = 0
    for quads, src, dst in ((qa, host_a, dev_a), (qb, host_b, dev_b)):
        arr = src.numpy() if isinstance(src, torch.Tensor) else np.asarray(src)
        for q in sorted(quads) if levels >= 1 else [0]:
            r0, c0 = (q >> 1) * h, (q & 1) * h
            hp = arr.ctypes.data + (r0 * arr.strides[0] + c0 * 8)
            dp = dst.data_ptr() + (r0 * dst.stride(0) + c0) * 8
            _lib.check(lib.mk_copy_to_device(ctypes.c_void_p(dp), dst.stride(0), ctypes.c_void_p(hp),
                                             arr.strides[0] // 8, h, h, st), "mk_copy_to_device")
            moved += h * h * 8
    return moved


def sharded_multiply(algo: str, a, b, levels: int, group=None, out=None, ws=None):
    """C = A B with this rank's share of the leaves plus the reduce; C is valid on rank 0.

    a, b: replicated CUDA FP64 operands (square, power-of-two order). Returns ``out``.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    total = leaf_count(algo, levels) * PANELS
    first, count = shard_range(total, world, rank)
    if out is None:
        out = torch.zeros_like(a)
    else:
        out.zero_()
    if count:
        partial_product(algo, a, b, out, levels, first, count, ws=ws)
    return assemble(out, 0, group)


# ------------------------------------------------------------------------------------------
# fused reduce-scatter: leaf epilogues write into the owning rank's C row slab (peer memory)
# ------------------------------------------------------------------------------------------
def slab_rows(n: int, world: int) -> int:
    """Rows of C each rank owns in the fused path (C = W row slabs of n / W rows)."""
    if world < 1 or n % world:
        raise ValueError(f"the order {n} must split into {world} equal row slabs")
    return n // world


def slab_owner(row: int, n: int, world: int) -> tuple[int, int]:
    """(owning rank, row inside its slab) of C row ``row`` -- the routing the epilogue applies."""
    sr = slab_rows(n, world)
    return row // sr, row % sr


def enable_peer_access(peer_device: int) -> None:
    """Let the current device address ``peer_device``'s memory (NVLink P2P); no-op for itself."""
    lib = _lib.load()
    _lib.check(lib.mk_enable_peer_access(int(peer_device)), "mk_enable_peer_access")


class SlabExchange:
    """Every rank's C row slab mapped into this process: its own as a local tensor, the peers'
    through CUDA IPC handles gathered over the process group (torch's CUDA tensor reductions).
    Keep the object alive on every rank until all ranks are done with the slabs."""

    def __init__(self, n: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.n = n
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.slab = torch.zeros((slab_rows(n, self.world), n), dtype=torch.float64, device=dev)
        if self.world == 1:
            self.slabs = [self.slab]
            return
        rebuild, args = reduce_tensor(self.slab)
        gathered = [None] * self.world
        dist.all_gather_object(gathered, args, group=group)
        self.slabs = []
        for r in range(self.world):
            if r == self.rank:
                self.slabs.append(self.slab)
                continue
            peer = rebuild(*gathered[r])
            if peer.device != dev:
                enable_peer_access(peer.device.index)
            self.slabs.append(peer)


def partial_product_slabs(algo: str, a, b, slabs, levels: int, first: int, count: int, stream=None, ws=None,
                          panels: int = PANELS) -> int:
    """Add shard units [first, first+count) of A B into the row slabs ``slabs`` (W tensors of
    n / W x n with one common row stride; local or peer-mapped), each row into its owner's slab."""
    import torch

    lib = _lib.load()
    for t, nm in ((a, "a"), (b, "b"), *((sl, f"slabs[{i}]") for i, sl in enumerate(slabs))):
        _check_operand(t, nm)
    n = a.shape[0]
    aid = _lib.ALGO_IDS[algo]
    need = int(lib.mk_partial_workspace_bytes(aid, n, levels))
    ws = _workspace(need, ws, a.device, stream)
    ld = slabs[0].stride(0)
    if any(s.stride(0) != ld or s.shape != slabs[0].shape for s in slabs):
        raise ValueError("slabs must share shape and row stride")
    ptrs = (ctypes.c_void_p * len(slabs))(*[s.data_ptr() for s in slabs])
    st = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    rc = lib.mk_strassen_partial_slabs(aid, ctypes.c_void_p(a.data_ptr()), a.stride(0), ctypes.c_void_p(b.data_ptr()),
                                       b.stride(0), ptrs, len(slabs), slabs[0].shape[0], ld, n, levels, first, count,
                                       panels, ctypes.c_void_p(ws.data_ptr()), need, st)
    _lib.check(rc, "mk_strassen_partial_slabs")
    return need


def fused_sharded_multiply(algo: str, a, b, levels: int, exchange: SlabExchange, out=None, ws=None):
    """C = A B with the fused reduce-scatter: this rank's leaves are added straight into the owning
    ranks' row slabs (one kernel does the product and the exchange); on return every rank's
    ``exchange.slab`` holds its rows of C, and ``out`` (rank 0 only, optional) the whole C, pulled
    from the peers' slabs. Host barriers only -- no kernel waits on another rank."""
    import torch
    import torch.distributed as dist

    world, rank, group = exchange.world, exchange.rank, exchange.group
    total = leaf_count(algo, levels) * PANELS
    first, count = shard_range(total, world, rank)
    exchange.slab.zero_()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group)  # every slab is zero before any rank adds into it
    if count:
        partial_product_slabs(algo, a, b, exchange.slabs, levels, first, count, ws=ws)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(group)  # every contribution has landed
    if out is not None and rank == 0:
        sr = exchange.slab.shape[0]
        for r, s in enumerate(exchange.slabs):
            out[r * sr:(r + 1) * sr].copy_(s)
        torch.cuda.synchronize()
    if world > 1:
        # rank 0 may still be reading the peers' slabs: no rank may return (and zero its slab in
        # the next call) before the pull is over
        dist.barrier(group)
    return exchange.slab


# ------------------------------------------------------------------------------------------
# rectangular products (BASELINE cfg5 on N GPUs): the padded rectangular recursion, sharded the
# same way (leaf row panels), partials summed by one reduce
# ------------------------------------------------------------------------------------------
def rect_partial_product(algo: str, a, b, out, levels: int, first: int, count: int, ws=None,
                         panels: int = PANELS) -> int:
    """out (m x n) := shard units [first, first+count) of A B (CUDA FP64, any m, k, n)."""
    import torch

    lib = _lib.load()
    for t, nm in ((a, "a"), (b, "b"), (out, "out")):
        _check_operand(t, nm)
    m, k = a.shape
    n = b.shape[1]
    aid = _lib.ALGO_IDS[algo]
    need = int(lib.mk_rect_partial_workspace_bytes(aid, m, n, k, levels, panels))
    ws = _workspace(need, ws, a.device, None)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = lib.mk_multiply_rect_partial(aid, ctypes.c_void_p(a.data_ptr()), a.stride(0), ctypes.c_void_p(b.data_ptr()),
                                      b.stride(0), ctypes.c_void_p(out.data_ptr()), out.stride(0), m, n, k, levels,
                                      first, count, panels, ctypes.c_void_p(ws.data_ptr()), need, st)
    _lib.check(rc, "mk_multiply_rect_partial")
    return need


def sharded_multiply_rect(algo: str, a, b, levels: int, group=None, out=None, ws=None):
    """C = A B (rectangular) with this rank's share of the leaves plus the reduce; C on rank 0."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    first, count = shard_range(leaf_count(algo, levels) * PANELS, world, rank)
    if out is None:
        out = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float64, device=a.device)
    rect_partial_product(algo, a, b, out, levels, first, count, ws=ws)
    return assemble(out, 0, group)


# ------------------------------------------------------------------------------------------
# one process driving several GPUs (the C ABI's mk_multi_gpu_winograd): no process group
# ------------------------------------------------------------------------------------------
def single_process_multiply(algo: str, a, b, levels: int, devices=None, out=None):
    """C = A B over the GPUs ``devices`` (default: every visible GPU) from ONE process: A, B and C
    live on devices[0]; every other device receives over NVLink only the operand quadrants its
    leaf row panels read, computes its partial C, and device 0 adds the partials in rank order
    (mk_multi_gpu_winograd). A device may be listed more than once (ranks sharing one GPU)."""
    import torch

    lib = _lib.load()
    for t, nm in ((a, "a"), (b, "b")):
        _check_operand(t, nm)
    n = a.shape[0]
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [int(d) for d in devices]
    if a.device.index != devices[0] or b.device.index != devices[0]:
        raise ValueError("a and b must live on devices[0]")
    if out is None:
        out = torch.empty((n, n), dtype=torch.float64, device=a.device)
    _check_operand(out, "out")
    aid = _lib.ALGO_IDS[algo]
    g = len(devices)
    wss, streams = [], []
    for r, d in enumerate(devices):
        need = int(lib.mk_multi_gpu_workspace_bytes(aid, n, levels, r, g))
        if need == 0 and r > 0:
            raise ValueError(f"unsupported multi-GPU shape: n={n}, levels={levels}")
        wss.append(torch.empty(max(need, 16), dtype=torch.uint8, device=torch.device("cuda", d)))
        streams.append(torch.cuda.current_stream(d) if r == 0 else torch.cuda.Stream(device=d))
    dev_arr = (ctypes.c_int * g)(*devices)
    ws_arr = (ctypes.c_void_p * g)(*[w.data_ptr() for w in wss])
    sz_arr = (ctypes.c_size_t * g)(*[w.numel() for w in wss])
    st_arr = (ctypes.c_void_p * g)(*[s.cuda_stream for s in streams])
    rc = lib.mk_multi_gpu_winograd(aid, g, dev_arr, ctypes.c_void_p(a.data_ptr()), a.stride(0),
                                   ctypes.c_void_p(b.data_ptr()), b.stride(0), ctypes.c_void_p(out.data_ptr()),
                                   out.stride(0), n, levels, ws_arr, sz_arr, st_arr)
    _lib.check(rc, "mk_multi_gpu_winograd")
    for w, s in zip(wss[1:], streams[1:]):
        w.record_stream(s)  # freed on return while the peers' kernels may still run
    return out
