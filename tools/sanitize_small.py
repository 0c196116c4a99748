"""Small workload touching every kernel / plan, for compute-sanitizer runs."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import quick_gpu as q
torch.manual_seed(0)
dev = "cuda"
for (m, n, k) in [(130, 3, 17), (256, 256, 256), (64, 200, 40)]:
    a = torch.randint(-8, 9, (m, k + (k % 2)), device=dev).double()[:, :k]
    b = torch.randint(-8, 9, (k, n + (n % 2)), device=dev).double()[:, :n]
    c = torch.empty((m, n), dtype=torch.float64, device=dev)
    q.dgemm(a, b, c)
    torch.cuda.synchronize()
    assert torch.equal(c, a @ b)
n = 512
a = torch.randint(-8, 9, (n, n), device=dev).double()
b = torch.randint(-8, 9, (n, n), device=dev).double()
ref = a @ b
for fuse in (0, 1):
    q.lib.mk_set_option(1, fuse)
    for algo in range(1, 7):
        for L in (1, 2, 3):
            c = torch.empty_like(a)
            q.strassen(algo, a.clone(), b.clone(), c, L)
            torch.cuda.synchronize()
            assert torch.equal(c, ref), (fuse, algo, L)
q.lib.mk_set_option(1, 0)
# rectangular with padding and in place
for (m, k, nn, L) in [(300, 517, 129, 2), (256, 256, 512, 2)]:
    a = torch.randint(-8, 9, (m, k), device=dev).double()
    b = torch.randint(-8, 9, (k, nn), device=dev).double()
    c = torch.empty((m, nn), dtype=torch.float64, device=dev)
    ws_b = q.lib.mk_rect_workspace_bytes(2, q.I64(m), q.I64(nn), q.I64(k), L)
    ws = torch.empty(max(ws_b, 8), dtype=torch.uint8, device=dev)
    rc = q.lib.mk_multiply_rect(2, q.VP(a.data_ptr()), q.I64(k), q.VP(b.data_ptr()), q.I64(nn), q.VP(c.data_ptr()), q.I64(nn),
                                q.I64(m), q.I64(nn), q.I64(k), L, q.VP(ws.data_ptr()), ctypes.c_size_t(ws_b), q.stream())
    assert rc == 0, q.lib.mk_last_error()
    torch.cuda.synchronize()
    assert torch.equal(c, a @ b)
print("sanitize workload ok")
# host paths: overlapped (pinned and pageable) and staged copies, n = 2048 (L = 1, 2, 3)
import numpy as np
import paper_2309_00628_b200 as pk
r = np.random.default_rng(3)
n = 2048
ah = r.integers(-8, 9, (n, n)).astype(np.float64)
bh = r.integers(-8, 9, (n, n)).astype(np.float64)
want = ah @ bh
for cut in (1024, 512, 256):
    ch = np.zeros((n, n))
    pk.winograd_block_mul(pk.Matrix(ah), pk.Matrix(bh), pk.Matrix(ch), pk.BasePolicy.naive_cutoff(cut))
    assert np.array_equal(ch, want) and pk.last_stats().path == "overlapped-host", cut
cr = pk.multiply(pk.Matrix(ah[:1500, :1700]), pk.Matrix(bh[:1700, :1300]), pk.get_variant("winograd-mod2", cutoff=256))
assert np.array_equal(cr.arr, ah[:1500, :1700] @ bh[:1700, :1300])
print("sanitize_small ok")
