import torch, time
x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory(); y = torch.empty_like(x, device="cuda")
for name, f in [("h2d", lambda: y.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(y, non_blocking=True))]:
    for _ in range(3): f()
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); [f() for _ in range(10)]; b.record(); torch.cuda.synchronize()
    print(name, 10 * x.numel() / (a.elapsed_time(b) * 1e-3) / 1e9, "GB/s")
