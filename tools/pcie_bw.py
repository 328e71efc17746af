"""Host<->device copy bandwidth on this box (pinned memory): H2D, D2H, and both
at once on two streams.  Informs the end-to-end path's floor."""
import time

import torch

n = 4 << 30  # 4 GiB
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()


def timeit(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


t_h2d = timeit(lambda: d1.copy_(h1, non_blocking=True))
t_d2h = timeit(lambda: h2.copy_(d2, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t_both = timeit(both)
print(f"H2D {n / t_h2d / 1e9:.1f} GB/s  D2H {n / t_d2h / 1e9:.1f} GB/s  both {2 * n / t_both / 1e9:.1f} GB/s total")
