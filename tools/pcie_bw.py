import torch, time
x = torch.empty(2 * 2**30 // 8, dtype=torch.float64).pin_memory(); x.fill_(1.0)
d = torch.empty_like(x, device="cuda")
for _ in range(2): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): d.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize()
h2d = 5 * x.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
e0.record()
for _ in range(5): x.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
d2h = 5 * x.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(f"h2d {h2d:.1f} GB/s  d2h {d2h:.1f} GB/s")
