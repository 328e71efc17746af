#!/usr/bin/env python
"""Full-size byte parity against the reference (oracle/_ref) at BASELINE.json's
configs, on ONE GPU, with the benchmark's own device-generated inputs.

  python tools/parity_full.py --workload qwen2.5-7b --ranks 1            # configs[2] (headline)
  python tools/parity_full.py --workload qwen2.5-7b --ranks 8 --sparsity 0.9999
  python tools/parity_full.py --workload qwen2.5-32b --ranks 8 --k 1,4,16  # configs[3]

The state dict is generated on the device (K5, seed --seed), then split into
--ranks contiguous name-ordered shards exactly as bench.py / shard.py would
(`shapes.shard`).  The N ranks run on one GPU without NCCL
(tests/parity_util.ShardedSim): each rank's K1 summary lands in a shared
`gathered` buffer, K2 emits with (n_ranks, rank), and apply takes the FLAT
carry from the gathered summaries on the device.  For every shard the
reference encodes the D2H copy of the SAME bytes and its PULP body must equal
that rank's section byte for byte (for FLAT_INT32 a shard's first u32 continues
the previous shard's gap stream, so it is checked against the carry instead).
Apply must then land on the target exactly.

--k K: multi-step (off-policy delay) patches.  The target is W_k, made by k
in-place reference-style mutations of W_0 (each changing 1 - sparsity of the
elements; re-flips cancel, so the patch density is (1 - (1 - 2p)^k) / 2), and
the direct k-step patch encode(W_k, W_0) is compared.

Test infrastructure: imports oracle/ (the reference) as the checker only.
Prints one JSON line per (k, representation) and writes them to --out.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import parity_util as PU  # noqa: E402
from oracle.oracle import Checkpoint, Tensor, reference  # noqa: E402
from paper_2602_03839_b200 import device as D  # noqa: E402
from paper_2602_03839_b200.shapes import numel, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="qwen2.5-7b")
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--sparsity", type=float, default=0.99)
    ap.add_argument("--cluster-width", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1002)
    ap.add_argument("--k", default="1")
    ap.add_argument("--reprs", default="0,1,2")
    ap.add_argument("--threads", type=int, default=3, help="shards encoded by the reference concurrently")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    R = reference()
    tensors = workload(args.workload)
    reprs = [int(x) for x in args.reprs.split(",")]
    ks = [int(x) for x in args.k.split(",")]
    sizes = [numel(s) for _, s in tensors]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    d = int(offs[-1])
    w0 = torch.empty(d, dtype=torch.int16, device="cuda")
    wk = torch.empty_like(w0)
    prev, curr = PU.DeviceState(tensors, w0, offs), PU.DeviceState(tensors, wk, offs)
    lines = []
    for k in ks:
        D.synth_base(w0, seed=args.seed)
        wk.copy_(w0)
        for j in range(k):
            D.synth_mutate(wk, wk, args.sparsity, args.cluster_width, seed=args.seed + 1 + j)
        torch.cuda.synchronize()
        density = 1 - args.sparsity
        cap = min(1.0, (1 - (1 - 2 * density) ** k) / 2 * 1.02 + 1e-4) if k > 1 else density * 1.02
        from paper_2602_03839_b200.shapes import shard
        b = shard(tensors, args.ranks)

        def ref_shard(r):
            lo, hi = b[r], b[r + 1]
            if lo == hi:
                return r, {x: None for x in reprs}, 0.0
            hp, hc = PU.host_checkpoint(prev, 0, lo, hi), PU.host_checkpoint(curr, 1, lo, hi)
            t0 = time.perf_counter()
            w = R.encode_pulps(hc, hp, reprs=tuple(reprs))
            return r, w, time.perf_counter() - t0

        ref_t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(max_workers=args.threads) as ex:
            ref = {r: (w, t) for r, w, t in ex.map(ref_shard, range(args.ranks))}
        ref_wall = time.perf_counter() - ref_t0
        for rp in reprs:
            # ranks one after another (one plan resident at a time, so the 32B shape at
            # k = 16 fits one GPU); a rank's K2 and its FLAT carry read only the summaries
            # of earlier ranks, which are already in `gathered`
            gathered = torch.zeros(32 * args.ranks, dtype=torch.uint8, device="cuda")
            ok, compared, changes, ref_bytes, body_bytes, enc_s = True, 0, 0, 0, 0, 0.0
            applied_ok, details = True, []
            for r in range(args.ranks):
                lo, hi = b[r], b[r + 1]
                mine = tensors[lo:hi]
                dr = sum(numel(s) for _, s in mine)
                plan = D.DevicePlan([(numel(s), s[-1]) for _, s in mine], int(dr * cap) + 65536)
                plan.bind(0, prev.views(lo, hi))
                plan.bind(1, curr.views(lo, hi))
                plan.bind(2, prev.views(lo, hi))  # apply in place onto W_0: it must become W_k
                t0 = time.perf_counter()
                plan.scan(1, 0, summary_out=gathered[32 * r:32 * r + 32])
                pt = plan.new_patch(rp)
                plan.emit(pt, gathered=gathered, n_ranks=args.ranks, rank=r)
                pt.fetch()
                enc_s += time.perf_counter() - t0
                pt.raise_for_status([n for n, _ in mine])
                sec = pt.body[: pt.body_bytes].cpu().numpy().tobytes()
                body_bytes += len(sec)
                wire = ref[r][0][rp]
                summ = gathered.cpu().numpy().view(D.N.SUMMARY_DTYPE)
                if wire is None:
                    ok = ok and sec == b""
                else:
                    header, body = PU.split_pulp(wire)
                    ref_bytes += len(body)
                    changes += sum(t["count"] for t in header["tensors"])
                    same = True
                    if rp == 2 and header["tensors"]:
                        # FLAT: the shard's first entry continues the previous shard's gap stream
                        carry = next((int(summ[q]["last_gap_base"]) for q in range(r - 1, -1, -1)
                                      if int(summ[q]["has_change"])), None)
                        if carry is not None:
                            same = int.from_bytes(sec[:4], "little") == \
                                (int.from_bytes(body[:4], "little") + carry) & 0xFFFFFFFF
                            body, sec = body[4:], sec[4:]
                    pe = pt.host_entries[: pt.n_entries]
                    same = same and sec == body and len(pe) == len(header["tensors"]) and all(
                        int(e["count"]) == h["count"] and int(e["idx_nbytes"]) == h["index_nbytes"]
                        and mine[int(e["tensor"])][0] == h["name"] for e, h in zip(pe, header["tensors"]))
                    details.append({"rank": r, "tensors": len(header["tensors"]), "bytes": len(body),
                                    "bit_exact": bool(same)})
                    ok = ok and same
                    compared += len(header["tensors"])
                carry_dev = None
                if rp == 2:
                    carry_dev = torch.zeros(16, dtype=torch.uint8, device="cuda")
                    D.flat_carry_from_summaries(gathered, r, carry_dev)
                res = D.parse_result(plan.apply_patch(2, pt, carry=carry_dev))
                applied_ok = applied_ok and int(res["status"]) == 0
                del plan, pt
            applied_ok = applied_ok and bool(torch.equal(w0, wk))
            D.synth_base(w0, seed=args.seed)  # restore W_0 for the next representation
            line = {"workload": args.workload, "ranks": args.ranks, "k": k, "sparsity": args.sparsity,
                    "representation": PU_REPR[rp], "elements": d, "changes": changes,
                    "patch_body_bytes": body_bytes, "reference_body_bytes": ref_bytes,
                    "tensors_compared": compared, "bit_exact_vs_reference": bool(ok), "apply_exact": applied_ok,
                    "device_encode_s_incl_fetch": round(enc_s, 4), "reference_encode_write_s_wall": round(ref_wall, 2),
                    "reference_threads": args.threads, "per_rank": details}
            print(json.dumps(line), flush=True)
            lines.append(line)
        del ref
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            for x in lines:
                f.write(json.dumps(x) + "\n")
    return 0 if all(x["bit_exact_vs_reference"] and x["apply_exact"] for x in lines) else 1


PU_REPR = {0: "COO_DOWNSCALED", 1: "COO_INT32", 2: "FLAT_INT32"}

if __name__ == "__main__":
    sys.exit(main())
