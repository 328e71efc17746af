"""K1 (diff + compaction) time on the 7B shape at a given sparsity, CUDA events,
median of 7 launches.  PULSE_K1_EXPERIMENT selects attribution variants
(see encode.cu K1Args::experiment).  Usage: python tools/k1_time.py [sparsity]"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03839_b200 import device as D  # noqa: E402
from paper_2602_03839_b200.shapes import numel, workload  # noqa: E402

sp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.99
tensors = workload("qwen2.5-7b")
sizes = [numel(s) for _, s in tensors]
n = sum(sizes)
prev = torch.empty(n, dtype=torch.int16, device="cuda")
curr = torch.empty_like(prev)
D.synth_base(prev, seed=1002)
D.synth_mutate(prev, curr, sp, int(os.environ.get("CW", "64")), seed=1002)
offs = np.concatenate([[0], np.cumsum(sizes)])
views = lambda b: [b[int(offs[i]):int(offs[i + 1])] for i in range(len(sizes))]
plan = D.DevicePlan([(m, s[-1]) for m, (_, s) in zip(sizes, tensors)], int(n * (1 - sp) * 1.02) + 65536)
plan.bind(0, views(prev))
plan.bind(1, views(curr))
ts = []
for it in range(9):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    plan.scan(1, 0)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"sparsity {sp} experiment {os.environ.get('PULSE_K1_EXPERIMENT', '0')}: K1 {statistics.median(ts[2:]):.3f} ms "
      f"({(4 * n) / (statistics.median(ts[2:]) / 1e3) / 1e12:.2f} TB/s of snapshot reads)")
