import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D
def run(sizes, dens, seed=0):
    g = torch.Generator(device='cuda').manual_seed(seed)
    prevs, currs = [], []
    for n in sizes:
        a = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device='cuda')
        flip = (torch.rand(n, device='cuda') < dens).to(torch.int16)
        prevs.append(a); currs.append(a ^ flip)
    plan = D.DevicePlan([(n, 8) for n in sizes], int(sum(sizes) * dens * 1.2) + 1000)
    plan.bind(0, prevs); plan.bind(1, currs)
    t = time.time()
    plan.scan(1, 0); torch.cuda.synchronize()
    print(len(sizes), sum(sizes), dens, 'scan ok', round(time.time() - t, 4), flush=True)
    p = plan.encode(1, 0, 1)
    idx, _ = plan.decode_indices(p)
    want = torch.cat([torch.nonzero(a != b).flatten() for a, b in zip(prevs, currs)])
    print('  changes', p.n_changes, want.numel(), torch.equal(idx, want), flush=True)
run([1 << 27], 0.01)
run([65536 * 3 + 8] * 300, 0.01)
run([1000 + 8 * i for i in range(2000)], 0.01)
run([1 << 28], 0.01)
