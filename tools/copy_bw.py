"""Pinned host <-> device copy bandwidth on this box (diagnostic)."""
import torch
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
ms = t(lambda: d1.copy_(h1, non_blocking=True)); print(f"H2D {n / ms / 1e6:.1f} GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True)); print(f"D2H {n / ms / 1e6:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(both); print(f"H2D+D2H concurrent: {2 * n / ms / 1e6:.1f} GB/s total ({ms:.1f} ms for 1 GiB each way)")
