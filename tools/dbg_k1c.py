import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D
for n in [1 << 28, 1 << 30, 1 << 31, 3 << 30]:
    a = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device='cuda')
    b = a ^ (torch.rand(n, device='cuda') < 0.01).to(torch.int16)
    plan = D.DevicePlan([(n, 8)], int(n * 0.012) + 1000)
    plan.bind(0, [a]); plan.bind(1, [b])
    for it in range(4):
        torch.cuda.synchronize(); t = time.time()
        plan.scan(1, 0); torch.cuda.synchronize()
        dt = time.time() - t
        print(n, it, f"{dt*1e3:.2f} ms", f"{4*n/dt/1e9:.0f} GB/s", flush=True)
    del a, b, plan
    torch.cuda.empty_cache()
