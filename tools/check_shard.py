"""torchrun check: the sharded multi-GPU encode gathered to rank 0 (NCCL point-to-point,
shard.gather) is byte-identical to a single-GPU encode of the whole state dict and to
the reference's PULP body on the same bytes (all three representations), and sharded
apply reproduces `curr` on every rank.  Prints one JSON line with the gather time
(CUDA events on rank 0 around sp.gather, max over ranks).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/check_shard.py
"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03839_b200 import device as D
from paper_2602_03839_b200.shapes import workload, numel
from paper_2602_03839_b200.shard import ShardedPulse

local = int(os.environ.get('LOCAL_RANK', 0))
torch.cuda.set_device(local)
dist.init_process_group('nccl', device_id=torch.device('cuda', local))
rank, world = dist.get_rank(), dist.get_world_size()
tensors = workload(sys.argv[1] if len(sys.argv) > 1 else 'qwen2.5-1.5b')
sizes = [numel(s) for _, s in tensors]
offs = np.concatenate([[0], np.cumsum(sizes)])
prev = torch.empty(int(offs[-1]), dtype=torch.int16, device='cuda'); curr = torch.empty_like(prev)
D.synth_base(prev, seed=77); D.synth_mutate(prev, curr, 0.99, 64, seed=78)
sp = ShardedPulse(tensors)
lo, hi = sp.bounds[rank], sp.bounds[rank + 1]
view = lambda b: [b[int(offs[i]):int(offs[i + 1])] for i in range(lo, hi)]
w = prev.clone()
sp.bind(0, view(prev)); sp.bind(1, view(curr)); sp.bind(2, view(w))
ok = True
full = None
want = None
if rank == 0 and os.environ.get('PULSE_CHECK_REF', '1') == '1':
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
    from oracle.oracle import have_reference, reference
    import parity_util as PU
    if have_reference():
        st = lambda b: PU.DeviceState(tensors, b, offs)
        want = reference().encode_pulps(PU.host_checkpoint(st(curr), 1), PU.host_checkpoint(st(prev), 0))
gather_ms = {}
if rank == 0:
    full = D.DevicePlan([(n, s[-1]) for n, (_, s) in zip(sizes, tensors)], int(offs[-1] * 0.0102) + 65536)
    full.bind(0, [prev[int(offs[i]):int(offs[i + 1])] for i in range(len(sizes))])
    full.bind(1, [curr[int(offs[i]):int(offs[i + 1])] for i in range(len(sizes))])
for repr_ in (0, 1, 2):
    patch = sp.new_patch(repr_)
    sec = sp.encode(1, 0, patch)
    torch.cuda.synchronize(); dist.barrier()
    if repr_ == 0:  # untimed first gather: NCCL sets up its point-to-point connections lazily
        sp.gather(sec)
        torch.cuda.synchronize(); dist.barrier()
    g0 = torch.cuda.Event(enable_timing=True); g1 = torch.cuda.Event(enable_timing=True)
    g0.record()
    body, ents = sp.gather(sec)
    g1.record(); torch.cuda.synchronize()
    gt = torch.tensor([g0.elapsed_time(g1)], device='cuda'); dist.all_reduce(gt, op=dist.ReduceOp.MAX)
    gather_ms[repr_] = round(float(gt.item()), 3)
    w.copy_(prev)
    res = D.parse_result(sp.apply(2, sec))
    good = int(res['status']) == 0 and all(torch.equal(a, b) for a, b in zip(view(w), view(curr)))
    if rank == 0:
        ref = full.encode(1, 0, repr_)
        same_body = torch.equal(body, ref.body[:ref.body_bytes])
        same_ent = np.array_equal(ents, ref.host_entries[:ref.n_entries])
        same_ref = True
        if want is not None:
            hl = int.from_bytes(want[repr_][8:16], 'little')
            same_ref = body.cpu().numpy().tobytes() == want[repr_][16 + hl:]
        print(f'repr {repr_}: sections {list(sec.body_bytes)} gathered == single-GPU body: {same_body}, entries: {same_ent}, '
              f'== reference body: {same_ref if want is not None else "n/a"}, gather {gather_ms[repr_]} ms', flush=True)
        ok = ok and same_body and same_ent and same_ref
    t = torch.tensor([int(good)], device='cuda'); dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0: print(f'repr {repr_}: sharded apply exact on all ranks: {bool(t.item())}', flush=True)
    ok = ok and bool(t.item())
if rank == 0:
    import json
    print(json.dumps({"check": "sharded encode + NCCL gather to rank 0", "workload": sys.argv[1] if len(sys.argv) > 1 else 'qwen2.5-1.5b',
                      "world": world, "gather_ms": gather_ms, "reference_compared": want is not None, "pass": bool(ok)}), flush=True)
    print('CHECK_SHARD', 'PASS' if ok else 'FAIL', flush=True)
dist.destroy_process_group()
