import torch
x = torch.empty(2 * 1024**3, dtype=torch.float64, device="cuda").normal_()  # 16 GB
y = torch.empty(1, dtype=torch.float64, device="cuda")
for f in ("sum", "amax"):
    fn = getattr(torch, f)
    fn(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); fn(x); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f, "read GB/s", x.numel() * 8 / (best * 1e-3) / 1e9)
z = torch.empty_like(x)
z.copy_(x); torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0.record(); z.copy_(x); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
print("copy GB/s (r+w)", 2 * x.numel() * 8 / (best * 1e-3) / 1e9)
