"""Multi-rank logic of the sharded product on CPU (gloo, world size 2): shard ranges,
leaf-product decomposition, and the sum-reduce assembly through paper_2309_00628_b200.multigpu."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_00628_b200.multigpu import assemble, operand_quadrants, shard_range
from oracle import strassen_oracle as o


def test_shard_ranges_cover_every_leaf_once():
    for total in (1, 7, 8, 49, 343):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                first, count = shard_range(total, world, r)
                seen.extend(range(first, first + count))
            assert seen == list(range(total))
            counts = [shard_range(total, world, r)[1] for r in range(world)]
            assert max(counts) - min(counts) <= 1


@pytest.mark.parametrize("kernel", ["strassen", "winograd-block", "winograd-knuth", "winograd-knuth-8call"])
@pytest.mark.parametrize("levels", [1, 2])
def test_leaf_decomposition_sums_to_the_product(kernel, levels):
    r = np.random.default_rng(5)
    n = 16
    a, b = r.integers(-8, 9, (n, n)), r.integers(-8, 9, (n, n))
    for panels in (1, 4):
        total = len(o.one_level_coefficients(kernel)[0]) ** levels * panels
        acc = np.zeros((n, n), dtype=np.int64)
        for w in range(3):
            first, count = shard_range(total, 3, w)
            acc += o.leaf_partial(kernel, a, b, levels, first, count, panels)
        assert np.array_equal(acc, a @ b), panels


@pytest.mark.parametrize("kernel", ["strassen", "winograd-block", "winograd-knuth", "winograd-knuth-8call"])
@pytest.mark.parametrize("levels", [1, 2])
def test_operand_quadrants_cover_what_a_shard_reads(kernel, levels):
    """A shard's partial (oracle leaf decomposition) depends only on the quadrants
    operand_quadrants names: NaN elsewhere in A and B never reaches it."""
    r = np.random.default_rng(8)
    n, h = 16, 8
    a, b = r.integers(-8, 9, (n, n)).astype(np.float64), r.integers(-8, 9, (n, n)).astype(np.float64)
    panels = 2
    total = len(o.one_level_coefficients(kernel)[0]) ** levels * panels
    for world in (2, 4, 8):
        for w in range(world):
            first, count = shard_range(total, world, w)
            if not count:
                continue
            qa, qb = operand_quadrants(kernel, levels, first, count, panels)
            ra, rb = np.full_like(a, np.nan), np.full_like(b, np.nan)
            for q in qa:
                ra[(q >> 1) * h:(q >> 1) * h + h, (q & 1) * h:(q & 1) * h + h] = a[(q >> 1) * h:(q >> 1) * h + h, (q & 1) * h:(q & 1) * h + h]
            for q in qb:
                rb[(q >> 1) * h:(q >> 1) * h + h, (q & 1) * h:(q & 1) * h + h] = b[(q >> 1) * h:(q >> 1) * h + h, (q & 1) * h:(q & 1) * h + h]
            want = o.leaf_partial(kernel, a, b, levels, first, count, panels)
            got = o.leaf_partial(kernel, ra, rb, levels, first, count, panels)
            assert np.array_equal(got, want), (kernel, levels, world, w)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kernel, levels, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = np.random.default_rng(9)
        n = 32
        a, b = r.integers(-8, 9, (n, n)), r.integers(-8, 9, (n, n))
        panels = 8
        total = len(o.one_level_coefficients(kernel)[0]) ** levels * panels
        first, count = shard_range(total, world, rank)
        part = torch.from_numpy(o.leaf_partial(kernel, a, b, levels, first, count, panels))
        out = assemble(part, dst_rank=0)
        if rank == 0:
            q.put(bool(np.array_equal(out.numpy(), a @ b)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("levels", [1, 2])
def test_two_rank_gloo_assembly(levels):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "winograd-block", levels, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


def test_slab_routing_covers_every_row_once():
    """Fused path: C = W row slabs; every row has exactly one owner and slot."""
    from paper_2309_00628_b200.multigpu import slab_owner, slab_rows

    for n, world in ((16, 1), (16, 2), (64, 4), (64, 8), (16384, 8)):
        sr = slab_rows(n, world)
        seen = {slab_owner(r, n, world) for r in range(n)}
        assert len(seen) == n and all(0 <= o_ < world and 0 <= i < sr for o_, i in seen)
    with pytest.raises(ValueError):
        slab_rows(10, 4)


def _fused_worker(rank, world, port, kernel, levels, q):
    """Host-side model of the fused reduce-scatter: each rank routes its partial's rows to the
    owning rank (the epilogue's slab addressing), owners sum what they receive, rank 0 gathers."""
    from paper_2309_00628_b200.multigpu import slab_owner, slab_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = np.random.default_rng(11)
        n = 32
        a, b = r.integers(-8, 9, (n, n)), r.integers(-8, 9, (n, n))
        panels = 8
        total = len(o.one_level_coefficients(kernel)[0]) ** levels * panels
        first, count = shard_range(total, world, rank)
        part = o.leaf_partial(kernel, a, b, levels, first, count, panels)
        sr = slab_rows(n, world)
        outgoing = [np.zeros((sr, n), dtype=np.int64) for _ in range(world)]
        for row in range(n):
            owner, local = slab_owner(row, n, world)
            outgoing[owner][local] += part[row]
        incoming = [torch.zeros((sr, n), dtype=torch.int64) for _ in range(world)]
        # gloo has no all_to_all: one scatter per source rank models the peer writes
        for src in range(world):
            recv = torch.zeros((sr, n), dtype=torch.int64)
            dist.scatter(recv, [torch.from_numpy(x) for x in outgoing] if rank == src else None, src=src)
            incoming[src] = recv
        slab = sum(incoming)
        gathered = [torch.zeros((sr, n), dtype=torch.int64) for _ in range(world)] if rank == 0 else None
        dist.gather(slab, gathered, dst=0)
        if rank == 0:
            q.put(bool(np.array_equal(torch.cat(gathered).numpy(), a @ b)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("levels", [1, 2])
def test_two_rank_gloo_fused_slab_routing(levels):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, "winograd-block", levels, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True
