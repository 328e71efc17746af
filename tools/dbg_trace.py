import os, sys, time, ctypes as C, torch, numpy as np
os.environ['PULSE_TRACE'] = '1'
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import device as D, _native as N
from paper_2602_03839_b200.shapes import workload, numel
tensors = workload('qwen2.5-7b')
sizes = [numel(s) for _, s in tensors]; Dn = sum(sizes)
prev = torch.empty(Dn, dtype=torch.int16, device='cuda'); curr = torch.empty_like(prev)
D.synth_base(prev, seed=1002); D.synth_mutate(prev, curr, 0.99, 64, seed=1002)
offs = np.concatenate([[0], np.cumsum(sizes)])
views = lambda b: [b[int(offs[i]):int(offs[i+1])] for i in range(len(sizes))]
plan = D.DevicePlan([(n_, s[-1]) for n_, (_, s) in zip(sizes, tensors)], int(Dn * 0.0102) + 65536)
plan.bind(0, views(prev)); plan.bind(1, views(curr))
n = C.c_uint64(); tp = N.lib.pulse_plan_trace(plan._plan, C.byref(n))
print('tickets', n.value, flush=True)
for it in range(300):
    cs, ps = (1, 0) if it % 2 == 0 else (0, 1)
    plan.scan(cs, ps); torch.cuda.synchronize()
    wd = N.watchdog()
    if wd:
        print('WATCHDOG', it, wd, flush=True)
        tr = np.zeros(n.value, np.uint32)
        C.cdll.LoadLibrary('libcudart.so.12') if False else None
        torch.cuda.synchronize()
        t = torch.empty(n.value, dtype=torch.int32, device='cuda')
        # copy via torch: wrap raw pointer with cudaMemcpy from the runtime torch uses
        cudart = C.CDLL('/usr/local/cuda/lib64/libcudart.so')
        cudart.cudaMemcpy(C.c_void_p(tr.ctypes.data), C.c_void_p(tp), C.c_size_t(n.value * 4), 2)
        bad = np.nonzero((tr & 31) != 31)[0]
        print('incomplete tickets:', len(bad))
        for b in bad[:60]:
            print('  ticket', b, 'block', tr[b] >> 8, 'flags', bin(tr[b] & 31))
        blocks = set(int(tr[b] >> 8) for b in bad)
        for blk in sorted(blocks)[:10]:
            mine = np.nonzero((tr >> 8) == blk)[0]
            print('  block', blk, 'last tickets', [(int(x), bin(tr[x] & 31)) for x in mine[-6:]])
        break
else:
    print('no watchdog in 300 scans')
