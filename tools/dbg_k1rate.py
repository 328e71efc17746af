import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D, _native as N
n = 1 << 32
a = torch.empty(n, dtype=torch.int16, device='cuda'); D.synth_base(a, 5)
b = torch.empty_like(a); D.synth_mutate(a, b, 0.99, 64, 6)
plan = D.DevicePlan([(n, 4096)], int(n * 0.0102) + 65536)
plan.bind(0, [a]); plan.bind(1, [b])
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3): plan.scan(1, 0)
torch.cuda.synchronize(); ev[0].record()
for it in range(10): plan.scan(1, 0)
ev[1].record(); torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 10
print(sys.argv[1:], f"{ms:.3f} ms  {4*n/ms/1e6:.0f} GB/s", N.watchdog(), flush=True)
