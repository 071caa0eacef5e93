"""Diagnostic (not collected): pinned host <-> device copy bandwidth (the
swap roofline denominator), large transfers, CUDA events."""
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    with torch.cuda.stream(s):
        for _ in range(2): fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5): fn()
        e1.record(s)
    torch.cuda.synchronize()
    print(f"{name}: {5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
