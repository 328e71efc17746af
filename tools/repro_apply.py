"""Runs encode + apply of every golden case (COO) once, outside pytest: a small repro for
debugging an apply build variant under cuda-gdb (PULSE_LIB=<variant.so>)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import json
import numpy as np
import torch
from oracle.oracle import Checkpoint, Tensor
from paper_2602_03839_b200 import device as D

G = os.path.join(ROOT, "tests", "golden")
man = json.load(open(os.path.join(G, "golden.json")))
snaps = np.load(os.path.join(G, "synth_cases.npz"))
repr_ = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for name, m in man["cases"].items():
    shapes = [tuple(s) for s in m["shapes"]]
    ck = lambda k: Checkpoint(0, [Tensor(n, s, snaps[f"{name}/{k}/{i}"]) for i, (n, s) in enumerate(zip(m["names"], shapes))]).sorted()
    prev, curr = ck("prev"), ck("curr")
    up = lambda ts: [torch.from_numpy(t.data.view(np.int16).copy()).cuda() for t in ts]
    pd, cd, wd = up(prev), up(curr), up(prev)
    plan = D.DevicePlan([(t.data.size, t.shape[-1]) for t in prev], max(16, sum(t.data.size for t in prev)))
    plan.bind(0, pd); plan.bind(1, cd); plan.bind(2, wd)
    p = plan.encode(1, 0, repr_)
    res = D.parse_result(plan.apply(2, p))
    ok = int(res["status"]) == 0 and all(torch.equal(a, b) for a, b in zip(wd, cd))
    print(name, "ok" if ok else f"MISMATCH {res}", flush=True)
