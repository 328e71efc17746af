import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D
from paper_2602_03839_b200.shapes import workload, numel
wl = sys.argv[1] if len(sys.argv) > 1 else 'qwen2.5-7b'
tensors = workload(wl)
sizes = [numel(s) for _, s in tensors]; Dn = sum(sizes)
prev = torch.empty(Dn, dtype=torch.int16, device='cuda'); curr = torch.empty_like(prev); w = torch.empty_like(prev)
D.synth_base(prev, seed=1002); n = D.synth_mutate(prev, curr, 0.99, 64, seed=1002); w.copy_(prev)
torch.cuda.synchronize(); print('synth', n, flush=True)
offs = np.concatenate([[0], np.cumsum(sizes)])
views = lambda b: [b[int(offs[i]):int(offs[i+1])] for i in range(len(sizes))]
plan = D.DevicePlan([(n_, s[-1]) for n_, (_, s) in zip(sizes, tensors)], int(Dn * 0.0102) + 65536)
plan.bind(0, views(prev)); plan.bind(1, views(curr)); plan.bind(2, views(w))
patch = plan.new_patch(0)
for it in range(6):
    cs, ps = (1, 0) if it % 2 == 0 else (0, 1)
    torch.cuda.synchronize(); t = time.time()
    plan.scan(cs, ps); torch.cuda.synchronize(); t1 = time.time()
    summ = torch.empty(0)
    plan.emit(patch); patch.fetch(); t2 = time.time()
    print(it, 'scan', round((t1 - t) * 1e3, 2), 'emit', round((t2 - t1) * 1e3, 2), 'status', patch.status, 'n', patch.n_changes, flush=True)
    res = D.parse_result(plan.apply(2, patch)); torch.cuda.synchronize(); t3 = time.time()
    print('   apply', round((t3 - t2) * 1e3, 2), 'status', int(res['status']), flush=True)
print('final ok', bool(torch.equal(w, prev)))
