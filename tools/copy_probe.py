"""Host<->device copy bandwidth alone and with both directions concurrent (pinned, 256 MB)."""
import torch
n = 32 * 1000 * 1000  # 256 MB of fp64
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.randn(n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    torch.cuda.synchronize(); fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    with torch.cuda.stream(sa): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(sb): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {n * 8 / ms / 1e6:.1f} GB/s per direction")
