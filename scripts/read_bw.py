"""Reference read bandwidths on this GPU: torch copy (r+w), torch sum (read), for context."""
import torch
x = torch.randn(1 << 30, device="cuda", dtype=torch.bfloat16)   # 2 GiB
y = torch.empty_like(x)
for name, fn, byts in [("copy r+w", lambda: y.copy_(x), 2 * x.numel() * 2),
                       ("sum (read)", lambda: x.sum(dtype=torch.float32), x.numel() * 2),
                       ("amax (read)", lambda: x.amax(), x.numel() * 2)]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"{name}: best {byts / min(ts) / 1e6:.0f} GB/s  median {byts / sorted(ts)[5] / 1e6:.0f} GB/s")
