import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D, _native as N
from paper_2602_03839_b200.shapes import workload, numel
tensors = workload('qwen2.5-7b')
sizes = [numel(s) for _, s in tensors]; Dn = sum(sizes)
prev = torch.empty(Dn, dtype=torch.int16, device='cuda'); curr = torch.empty_like(prev); w = torch.empty_like(prev)
D.synth_base(prev, seed=1002); n = D.synth_mutate(prev, curr, 0.99, 64, seed=1002); w.copy_(prev)
offs = np.concatenate([[0], np.cumsum(sizes)])
views = lambda b: [b[int(offs[i]):int(offs[i+1])] for i in range(len(sizes))]
plan = D.DevicePlan([(n_, s[-1]) for n_, (_, s) in zip(sizes, tensors)], int(Dn * 0.0102) + 65536)
plan.bind(0, views(prev)); plan.bind(1, views(curr)); plan.bind(2, views(w))
patch = plan.new_patch(0)
t = time.time()
for it in range(int(sys.argv[1])):
    cs, ps = (1, 0) if it % 2 == 0 else (0, 1)
    plan.scan(cs, ps)
    if it % 20 == 19:
        torch.cuda.synchronize()
        wd = N.watchdog()
        if wd: print('WATCHDOG', it, wd, flush=True); break
print('scans done', time.time() - t, flush=True)
bad = 0
for it in range(int(sys.argv[2])):
    cs, ps = (1, 0) if it % 2 == 0 else (0, 1)
    plan.scan(cs, ps); plan.emit(patch); patch.fetch(); res = plan.apply(2, patch)
    if it < 4:
        r = D.parse_result(res)
        ok = torch.equal(w, curr if it % 2 == 0 else prev)
        print('step', it, 'status', int(r['status']), 'ok', ok, flush=True)
        bad += not ok
torch.cuda.synchronize()
print('steps done', time.time() - t, N.watchdog(), bool(torch.equal(w, prev if int(sys.argv[2]) % 2 == 0 else curr)), flush=True)
