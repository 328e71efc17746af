"""torchrun probe: CUDA IPC peer views of another rank's buffer, written by pulse_store_to_peers."""
import os, sys, traceback
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03839_b200 import device as D
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
buf = torch.zeros(16 * world, dtype=torch.uint8, device="cuda")
h = buf.untyped_storage()._share_cuda_()
hs = [None] * world
dist.all_gather_object(hs, h)
ptrs = []
for r in range(world):
    if r == rank:
        ptrs.append(buf.data_ptr()); continue
    dev, handle, size, off = hs[r][0], hs[r][1], hs[r][2], hs[r][3]
    hb = bytes(handle)
    hb = hb[2:] if len(hb) == 66 else hb
    base = D.ipc_open(hb, local)
    ptrs.append(base + off)
    print(rank, "peer", r, "dev", dev, "base", hex(base), "off", off, "size", size, flush=True)
src = torch.full((16,), rank + 1, dtype=torch.uint8, device="cuda")
try:
    D.store_to_peers(src, [p + 16 * rank for p in ptrs], 16)
    torch.cuda.synchronize()
    print(rank, "store ok", flush=True)
except Exception:
    traceback.print_exc()
dist.barrier(); torch.cuda.synchronize()
print(rank, "table", buf.cpu().tolist(), flush=True)
dist.destroy_process_group()
