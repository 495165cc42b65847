"""Pinned host->device copy bandwidth on this box (the e2e input pipeline's bound)."""
import torch
for mb in (52, 104):
    n = mb * (1 << 20)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    print(f"H2D {mb} MB: {n * 10 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
