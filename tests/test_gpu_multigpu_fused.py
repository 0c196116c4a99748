"""Fused multi-GPU reduce-scatter (mk_strassen_partial_slabs) on the B200.

* one process: the W ranks' shards run in turn, each routing its leaf contributions into the W
  row slabs (local buffers) -- the slabs together must be the product (bit-exact on integers);
* two processes on the same GPU (gloo for the host barriers): each maps the other's slab through
  a CUDA IPC handle and its leaf epilogue adds straight into it -- the cross-process peer-memory
  path of a multi-GPU node, minus NVLink. The processes only meet at host barriers; no kernel
  waits on another process's kernel.
"""
import os
import socket

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(params=["dmma", "ozaki"])
def leaf(request):
    import paper_2309_00628_b200 as pk

    pk.set_leaf(request.param, 8, min_work=0) if request.param == "ozaki" else pk.set_leaf("dmma")
    yield request.param
    pk.set_leaf("dmma")


@pytest.mark.parametrize("algo", ["strassen", "winograd-block", "winograd-knuth"])
@pytest.mark.parametrize("levels", [1, 2])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_partials_assemble_the_product(algo, levels, world, leaf):
    """Both leaf kernels route rows to owner slabs (DMMA: REDG.ADD epilogue; INT8 Ozaki: atomic
    adds from the persistent kernel's write-back)."""
    import torch

    from paper_2309_00628_b200 import multigpu as mg

    n = 1024
    r = np.random.default_rng(world * 10 + levels)
    a = torch.from_numpy(r.integers(-8, 9, (n, n)).astype(np.float64)).cuda()
    b = torch.from_numpy(r.integers(-8, 9, (n, n)).astype(np.float64)).cuda()
    sr = mg.slab_rows(n, world)
    panels = 8
    slabs = [torch.zeros((sr, n), dtype=torch.float64, device="cuda") for _ in range(world)]
    total = mg.leaf_count(algo, levels) * panels
    for rank in range(world):
        first, count = mg.shard_range(total, world, rank)
        if count:
            mg.partial_product_slabs(algo, a, b, slabs, levels, first, count, panels=panels)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(slabs), a @ b)


def test_slab_path_rejects_bad_layouts():
    import torch

    from paper_2309_00628_b200 import _lib
    from paper_2309_00628_b200 import multigpu as mg

    n = 256
    a = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    slabs = [torch.zeros((n // 2, n), dtype=torch.float64, device="cuda") for _ in range(2)]
    with pytest.raises(Exception):
        mg.partial_product_slabs("winograd-block", a, a, slabs, 3, 0, 1)  # levels > 2: post-adds outside the epilogue
    with pytest.raises(Exception):
        mg.partial_product_slabs("winograd-block", a, a, slabs[:1], 1, 0, 1)  # slabs do not tile C
    assert _lib.load().mk_enable_peer_access(torch.cuda.current_device()) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, levels, exact, result_path, leaf="dmma"):
    import torch
    import torch.distributed as dist

    import paper_2309_00628_b200 as pk
    from paper_2309_00628_b200 import multigpu as mg

    if leaf == "ozaki":
        pk.set_leaf("ozaki", 8, min_work=0)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 2048
        r = np.random.default_rng(20240901)
        if exact:
            an = r.integers(-8, 9, (n, n)).astype(np.float64)
            bn = r.integers(-8, 9, (n, n)).astype(np.float64)
        else:
            an, bn = r.uniform(-1, 1, (n, n)), r.uniform(-1, 1, (n, n))
        a, b = torch.from_numpy(an).cuda(), torch.from_numpy(bn).cuda()
        ex = mg.SlabExchange(n)
        assert ex.slabs[rank].data_ptr() == ex.slab.data_ptr()
        out = torch.empty((n, n), dtype=torch.float64, device="cuda") if rank == 0 else None
        ref = a @ b
        bad = []
        # back-to-back calls with different operands, `out` checked after every call: the slabs
        # are re-zeroed and reused, and a peer that raced ahead into its next call (zeroing its
        # slab while rank 0 still pulls it) would leave zeroed or stale rows in `out`
        for it in range(4):
            s = float(it + 1)
            mg.fused_sharded_multiply("winograd-block", a * s, b, levels, ex, out=out)
            if rank == 0:
                want = ref * s
                ok = bool(torch.equal(out, want)) if exact else float((out - want).abs().max()) < 1e-11 * s
                if not ok:
                    bad.append(f"call {it}: mismatch {float((out - want).abs().max())}")
        if rank == 0:
            with open(result_path, "w") as f:
                f.write("ok" if not bad else "; ".join(bad))
        dist.barrier()  # peers keep their slabs alive until rank 0 has read them
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("levels,exact,leaf", [(1, True, "dmma"), (2, True, "dmma"), (2, False, "dmma"),
                                               (2, True, "ozaki"), (2, False, "ozaki")])
def test_two_process_ipc_fused_reduce_scatter(levels, exact, leaf, tmp_path):
    import torch.multiprocessing as mp

    result = str(tmp_path / "result.txt")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, levels, exact, result, leaf)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert open(result).read() == "ok"


@pytest.mark.parametrize("shape,levels,world", [((300, 500, 200), 2, 3), ((12000 // 8, 14000 // 8, 10000 // 8), 3, 8),
                                                ((129, 77, 65), 1, 2)])
def test_rect_partials_sum_to_the_product(shape, levels, world):
    """BASELINE cfg5 on N GPUs: the ranks' rectangular partials (leaf row panels of the padded
    recursion) sum to the product -- bit-exact on integer data (ranks run in turn on one GPU)."""
    import torch

    from paper_2309_00628_b200 import multigpu as mg

    m, k, n = shape
    r = np.random.default_rng(m + k + n)
    a = torch.from_numpy(r.integers(-8, 9, (m, k)).astype(np.float64)).cuda()
    b = torch.from_numpy(r.integers(-8, 9, (k, n)).astype(np.float64)).cuda()
    total = torch.zeros((m, n), dtype=torch.float64, device="cuda")
    part = torch.empty_like(total)
    units = mg.leaf_count("winograd-block", levels) * mg.PANELS
    for rank in range(world):
        first, count = mg.shard_range(units, world, rank)
        mg.rect_partial_product("winograd-block", a, b, part, levels, first, count)
        total += part
    torch.cuda.synchronize()
    assert torch.equal(total, a @ b)


@pytest.mark.parametrize("world", [2, 8])
def test_square_partials_three_levels(world):
    """Square shards at 3 levels (leaf fan-out 64 > 16: products materialised in slots, some of
    their leaves on other ranks): the partials still sum to the product exactly."""
    import torch

    from paper_2309_00628_b200 import multigpu as mg

    n = 1024
    r = np.random.default_rng(world)
    a = torch.from_numpy(r.integers(-8, 9, (n, n)).astype(np.float64)).cuda()
    b = torch.from_numpy(r.integers(-8, 9, (n, n)).astype(np.float64)).cuda()
    total = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    units = mg.leaf_count("winograd-block", 3) * mg.PANELS
    for rank in range(world):
        first, count = mg.shard_range(units, world, rank)
        part = torch.zeros_like(total)
        mg.partial_product("winograd-block", a, b, part, 3, first, count)
        total += part
    torch.cuda.synchronize()
    assert torch.equal(total, a @ b)


@pytest.mark.parametrize("ranks,levels,algo", [(2, 1, "winograd-block"), (3, 2, "winograd-block"), (4, 2, "strassen"),
                                               (8, 2, "winograd-knuth")])
def test_single_process_multi_gpu_abi(ranks, levels, algo):
    """mk_multi_gpu_winograd (one process, several devices): here every rank is device 0, which
    runs the same code path -- quadrant peer copies into each rank's workspace, the rank's leaf row
    panels into its partial C, device 0 summing the partials in rank order -- on one GPU. Integer
    data is exact; reals match the single-GPU product to rounding."""
    import torch

    from paper_2309_00628_b200 import multigpu as mg

    n = 2048
    r = np.random.default_rng(ranks + 10 * levels)
    a = torch.from_numpy(r.integers(-8, 9, (n, n)).astype(np.float64)).cuda()
    b = torch.from_numpy(r.integers(-8, 9, (n, n)).astype(np.float64)).cuda()
    c = mg.single_process_multiply(algo, a, b, levels, devices=[0] * ranks)
    torch.cuda.synchronize()
    assert torch.equal(c, a @ b)
    ar, br = torch.rand_like(a), torch.rand_like(b)
    cr = mg.single_process_multiply(algo, ar, br, levels, devices=[0] * ranks)
    torch.cuda.synchronize()
    assert float((cr - ar @ br).abs().max()) < 1e-10
