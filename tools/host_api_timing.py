import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2602_03839_b200 import host as H
rng = np.random.default_rng(0)
# 7B-like changes: 76M entries spread over 339 tensors is heavy; use 1.5B shape (15M changes)
from paper_2602_03839_b200.shapes import workload, numel
ts = workload('qwen2.5-1.5b')
tensors = []
for name, shp in ts:
    n = numel(shp)
    m = max(1, n // 100)
    idx = np.unique(rng.integers(0, n, m)).astype(np.int64)
    tensors.append(H.TensorPatch(name, shp, idx, rng.integers(0, 65536, idx.size, dtype=np.uint16)))
p = H.SparsePatch(0, 1, 0, 0, 0, b"\0" * 32, tensors)
h = H.PatchHandle.from_patch(p)
for it in range(3):
    t = time.time(); w = H.write_patch_bytes(h); t1 = time.time()
    r = H.read_patch_handle(w); t2 = time.time()
    print('write', round(t1 - t, 3), 'read', round(t2 - t1, 3), len(w), flush=True)
