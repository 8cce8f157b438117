"""Pinned host<->device copy bandwidth at the e2e leg's sizes (diagnostic)."""
import torch
for mb in (16.8, 33.5, 5.0):
    nb = int(mb * 1e6) // 8
    h = torch.empty(nb, dtype=torch.float64).pin_memory()
    d = torch.empty(nb, dtype=torch.float64, device="cuda")
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            fn()
        t.record()
        t.synchronize()
        ms = s.elapsed_time(t) / 10
        print(f"{name} {mb:5.1f} MB: {ms:.3f} ms  {nb * 8 / ms / 1e6:.1f} GB/s")
