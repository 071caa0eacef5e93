"""Diagnostic (not collected): pinned host <-> device copy bandwidth (the
swap roofline denominator), large transfers, CUDA events; and whether H2D and
D2H on two streams overlap (full duplex) or serialise on one copy engine."""
import time
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    with torch.cuda.stream(s):
        for _ in range(2): fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5): fn()
        e1.record(s)
    torch.cuda.synchronize()
    res[name] = 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    print(f"{name}: {res[name]:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s):
    for _ in range(3): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(3): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
el = time.perf_counter() - t
print(f"h2d || d2h on two streams: {3 * n / el / 1e9:.1f} GB/s each direction "
      f"({'overlapped' if el < 1.5 * 3 * n / (res['h2d'] * 1e9) else 'serialised'})")
