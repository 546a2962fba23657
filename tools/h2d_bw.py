"""Host link bandwidth on the box: pinned H2D / D2H copy rates (dev tool)."""
import torch
for mb in (38, 151, 605):
    n = mb * 2**20 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for direction in ("h2d", "d2h"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(4):
            if it == 1:
                e0.record()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{direction} {mb} MB: {ms:.3f} ms {n*8/ms/1e6:.1f} GB/s", flush=True)
