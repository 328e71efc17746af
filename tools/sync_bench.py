#!/usr/bin/env python
"""The sync path at BASELINE scale on one GPU: a publisher
resident holding W_t publishes W_{t+1} (device encode against the held weights,
PULP bytes straight from the device body, target hash once), and a consumer
resident holding W_t applies those bytes in place (apply_delta), without and
with the hash check.  Every step is checked bit-exact against the target.

  python tools/sync_bench.py [--workload qwen2.5-7b] [--steps 3] [--codec 0]
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_03839_b200 import device as D  # noqa: E402
from paper_2602_03839_b200 import host as H  # noqa: E402
from paper_2602_03839_b200.shapes import numel, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="qwen2.5-7b")
    ap.add_argument("--sparsity", type=float, default=0.99)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--codec", type=int, default=0)
    ap.add_argument("--repr", type=int, default=0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    tensors = workload(args.workload)
    names = [n for n, _ in tensors]
    shapes = [s for _, s in tensors]
    sizes = [numel(s) for s in shapes]
    offs = np.concatenate([[0], np.cumsum([(n + 7) // 8 * 8 for n in sizes])]).astype(np.int64)
    D_el = int(offs[-1])
    # a chain W_0 .. W_steps on the device (two buffers, generated step by step)
    a = torch.empty(D_el, dtype=torch.int16, device="cuda")
    b = torch.empty_like(a)
    D.synth_base(a, seed=11)
    views = lambda buf: [buf[int(offs[i]):int(offs[i]) + sizes[i]] for i in range(len(sizes))]
    cap = int(sum(sizes) * (1 - args.sparsity) * 1.05) + 4096
    pub = H.Resident.from_device(0, names, shapes, views(a), max_changes=cap)
    sub = H.Resident.from_device(0, names, shapes, views(a), max_changes=cap)
    sub_v = H.Resident.from_device(0, names, shapes, views(a), max_changes=cap)
    rows = []
    cur, nxt = a, b
    for step in range(1, args.steps + 1):
        D.synth_mutate(cur, nxt, args.sparsity, 64, seed=1000 + step)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wire, h = pub.publish(views(nxt), step, args.repr, args.codec, anchor_step=step - 1, advance=True)
        t1 = time.perf_counter()
        sub.apply(wire, step, expected_hash=h, verify=False)
        t2 = time.perf_counter()
        sub_v.apply(wire, step, expected_hash=h, verify=True)
        t3 = time.perf_counter()
        ok = True
        for r in (pub, sub, sub_v):
            for i in (0, len(sizes) // 2, len(sizes) - 1):
                got = _from_ptr(r.tensor_ptr(i), sizes[i])
                ok = ok and bool(torch.equal(got, views(nxt)[i]))
        ok = ok and pub.step == sub.step == sub_v.step == step and pub.weights_hash == sub_v.weights_hash == h
        rows.append({"publish_s": t1 - t0, "apply_s": t2 - t1, "apply_verify_s": t3 - t2, "pulp_bytes": len(wire),
                     "exact": ok})
        cur, nxt = nxt, cur
    d_bytes = 2 * sum(sizes)
    med = lambda k: float(np.median([r[k] for r in rows]))
    print(json.dumps({
        "tool": "sync_bench", "workload": args.workload, "elements": sum(sizes), "sparsity": args.sparsity,
        "representation": args.repr, "codec": args.codec, "steps": args.steps,
        "publish_s": round(med("publish_s"), 4), "apply_s": round(med("apply_s"), 4),
        "apply_verify_s": round(med("apply_verify_s"), 4),
        "apply_weight_gbs": round(d_bytes / med("apply_s") / 1e9, 2),
        "pulp_mb": round(rows[-1]["pulp_bytes"] / 1e6, 2), "exact": all(r["exact"] for r in rows),
        "note": "publish = device encode + D2H body + PULP assembly, overlapped with the SHA-256 of the target "
                "(host, one stream); apply = parse + upload + validate-then-scatter in HBM; apply_verify adds the "
                "index decode, undo copy and SHA-256 of the result (the reference's decode always verifies)",
    }))


def _from_ptr(ptr, n):
    """An int16 CUDA tensor viewing n elements at a raw device pointer (__cuda_array_interface__)."""
    class CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}
    return torch.as_tensor(CAI(), device="cuda")


if __name__ == "__main__":
    main()
