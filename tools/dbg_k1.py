import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D
def run(n, cols, dens, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 65536, n, dtype=np.uint16); b = a.copy()
    k = rng.random(n) < dens; b[k] ^= 1
    plan = D.DevicePlan([(n, cols)], max(16, n))
    plan.bind(0, [torch.from_numpy(a.view(np.int16)).cuda()]); plan.bind(1, [torch.from_numpy(b.view(np.int16)).cuda()])
    t = time.time()
    plan.scan(1, 0); torch.cuda.synchronize()
    s = plan.scan_summary_ptr()
    print(n, cols, dens, 'scan ok', time.time() - t, flush=True)
    p = plan.encode(1, 0, 1)
    idx, _ = plan.decode_indices(p)
    want = np.nonzero(a != b)[0]
    print('  changes', p.n_changes, len(want), np.array_equal(idx.cpu().numpy(), want), flush=True)
for args in [(64, 8, 0.1), (8192, 8, 0.01), (65536, 8, 0.01), (65536 * 3 + 8, 8, 0.01), (1 << 22, 8, 0.01), (1 << 22, 8, 0.5)]:
    run(*args)
