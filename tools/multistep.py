"""Multi-step patches across an off-policy delay k (BASELINE configs[3], SURVEY
8d C4): from W_0, k chained reference-style mutations give W_1..W_k (LSB
flips, so re-flips cancel: expected changed fraction (1-(1-2p)^k)/2).  Checks,
on the device path, that

  * the k chained single-step patches applied in order land on W_k exactly;
  * the direct k-step patch encode(W_k, W_0) applied once lands on W_k exactly

and reports timings and patch sizes as one JSON line per k.  Sharded by tensor
when launched under torchrun (one process per GPU):

  python tools/multistep.py --workload qwen2.5-7b --k 1 4 16
  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
      tools/multistep.py --workload qwen2.5-32b --k 1 4 16
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03839_b200 import device as D  # noqa: E402
from paper_2602_03839_b200.shapes import numel, workload  # noqa: E402
from paper_2602_03839_b200.shard import ShardedPulse  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="qwen2.5-7b")
    ap.add_argument("--k", type=int, nargs="+", default=[1, 4, 16])
    ap.add_argument("--p", type=float, default=0.01, help="per-step changed fraction")
    ap.add_argument("--repr", type=int, default=0)
    ap.add_argument("--seed", type=int, default=2024)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tensors = workload(args.workload)
    kmax = max(args.k)
    frac_max = (1 - (1 - 2 * args.p) ** kmax) / 2
    sp = ShardedPulse(tensors, max_change_frac=min(1.0, frac_max * 1.1 + 0.002))
    sizes = sp.sizes
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    d = int(offs[-1])
    views = lambda b: [b[int(offs[i]):int(offs[i + 1])] for i in range(len(sizes))]
    dev = torch.device("cuda", local)

    w0 = torch.empty(max(8, d), dtype=torch.int16, device=dev)
    D.synth_base(w0, seed=args.seed + 7919 * rank)
    cur, nxt = w0.clone(), torch.empty_like(w0)
    chained, direct = w0.clone(), torch.empty_like(w0)
    patch = sp.new_patch(args.repr)

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        return out, a.elapsed_time(b)

    def encode_apply(prev, curr, target):
        sp.bind(0, views(prev))
        sp.bind(1, views(curr))
        sp.bind(2, views(target))
        sec, t_enc = timed(lambda: sp.encode(1, 0, patch))
        if patch.status != 0:
            patch.raise_for_status([n for n, _ in sp.mine])
        _, t_app = timed(lambda: sp.apply(2, sec))
        res = sp.plan.last_result if hasattr(sp.plan, "last_result") else None
        return int(patch.n_changes), int(patch.body_bytes), t_enc, t_app, res

    results = []
    step = 0
    chain_ms = 0.0
    chain_changes = 0
    for k in sorted(args.k):
        while step < k:  # extend the chain to W_k, applying each single-step patch to `chained`
            D.synth_mutate(cur, nxt, 1 - args.p, 64, seed=args.seed + 1000 * (step + 1) + 104729 * rank)
            n, _, te, ta, _ = encode_apply(cur, nxt, chained)
            chain_ms += te + ta
            chain_changes += n
            cur, nxt = nxt, cur
            step += 1
        chain_ok = bool(torch.equal(chained, cur))
        direct.copy_(w0)
        n_direct, body, te, ta, _ = encode_apply(w0, cur, direct)
        direct_ok = bool(torch.equal(direct, cur))
        t = torch.tensor([te, ta, chain_ms, float(not (chain_ok and direct_ok)), float(n_direct), float(body),
                          float(chain_changes)], dtype=torch.float64, device=dev)
        if world > 1:
            mx = t[:4].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = t[4:].clone()
            dist.all_reduce(sm)
            t = torch.cat([mx, sm])
        te, ta, cms, bad, n_direct, body, cch = t.tolist()
        D_total = sum(numel(s) for _, s in tensors)
        line = {"workload": args.workload, "n_gpus": world, "k": k, "p": args.p,
                "representation": args.repr, "elements": D_total,
                "direct_changes": int(n_direct), "direct_changed_frac": round(n_direct / D_total, 5),
                "expected_frac": round((1 - (1 - 2 * args.p) ** k) / 2, 5),
                "direct_patch_mb": round(body / 1e6, 3), "direct_encode_ms": round(te, 3),
                "direct_apply_ms": round(ta, 3),
                "direct_weight_gbs": round(2 * D_total / ((te + ta) / 1e3) / 1e9, 1),
                "chain_steps": k, "chain_changes": int(cch), "chain_total_ms": round(cms, 3),
                "exact": not bool(bad)}
        results.append(line)
        if rank == 0:
            print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if all(r["exact"] for r in results) else 1


if __name__ == "__main__":
    sys.exit(main())
