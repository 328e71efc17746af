#!/usr/bin/env python
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --small

Runs every hot-path kernel on small inputs: K1 (k1_tma, including the dense
element-mode tickets and the overfull-ticket re-stream), K2 (optimistic layout,
escape scan, exact re-run), the apply pipeline (layout, F1s aggregate, range
scan, F3 exact checks, F5 scatter), the escape-aware general decoder, and the
int64-index apply of the host API -- for all three representations, on
BASELINE configs[0] (16M, from the reference generator when oracle/_ref is
present), the escape-heavy golden cases and a corrupted patch.  Every result
is checked against the reference bytes, so a sanitizer-clean run is also a
correct one.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from oracle.oracle import IDENTITY, have_reference, reference, restatement  # noqa: E402
from paper_2602_03839_b200 import device as D  # noqa: E402
from paper_2602_03839_b200 import host as H  # noqa: E402


def golden_cases():
    import json
    g = os.path.join(ROOT, "tests", "golden")
    man = json.load(open(os.path.join(g, "golden.json")))
    snaps = np.load(os.path.join(g, "synth_cases.npz"))
    pat = np.load(os.path.join(g, "patches.npz"))
    for name in ("handcrafted", "esc_rows", "esc_cols", "h5_unchanged", "dense_all", "roundtrip_s0"):
        m = man["cases"][name]
        prev = [snaps[f"{name}/prev/{i}"] for i in range(len(m["names"]))]
        curr = [snaps[f"{name}/curr/{i}"] for i in range(len(m["names"]))]
        order = sorted(range(len(m["names"])), key=lambda i: m["names"][i].encode())
        yield name, [m["names"][i] for i in order], [tuple(m["shapes"][i]) for i in order], \
            [prev[i] for i in order], [curr[i] for i in order], \
            {r: pat[f"{name}/{r}/0"].tobytes() for r in (0, 1, 2)}


def run_case(name, names, shapes, prev, curr, want):
    up = lambda arrs: [torch.from_numpy(a.view(np.int16).copy()).cuda() for a in arrs]  # noqa: E731
    p_d, c_d, w_d = up(prev), up(curr), up(prev)
    n = sum(a.size for a in prev)
    plan = D.DevicePlan([(a.size, s[-1]) for a, s in zip(prev, shapes)], max(1024, n))
    plan.bind(0, p_d)
    plan.bind(1, c_d)
    plan.bind(2, w_d)
    for r in (0, 1, 2):
        p = plan.encode(1, 0, r)
        p.raise_for_status(names)
        hl = int.from_bytes(want[r][8:16], "little")
        assert p.body[: p.body_bytes].cpu().numpy().tobytes() == want[r][16 + hl:], (name, r)
        for a, b in zip(w_d, p_d):
            a.copy_(b)
        res = D.parse_result(plan.apply(2, p))
        assert int(res["status"]) == 0 and all(torch.equal(a, b) for a, b in zip(w_d, c_d)), (name, r)
        # a corrupted copy: validate-then-scatter reports and writes nothing
        if p.body_bytes > 8:
            bad = plan.new_patch(r)
            bad.body[: p.body_bytes].copy_(p.body[: p.body_bytes])
            bad.entries.copy_(p.entries)
            bad.host_entries = p.host_entries
            bad.host_result = p.host_result
            e = p.host_entries[p.n_entries - 1]
            bad.body[int(e["idx_off"]) + int(e["idx_nbytes"]) - 1] = 0xFF
            for a, b in zip(w_d, p_d):
                a.copy_(b)
            res = D.parse_result(plan.apply(2, bad))
            if int(res["status"]) != 0:  # rejected: nothing written
                assert all(torch.equal(a, b) for a, b in zip(w_d, p_d)), (name, r)
    # host API: encode -> write -> read -> decode (int64-index apply path)
    ck = lambda arrs, step: H.Checkpoint(step, [H.Tensor(nm, s, a) for nm, s, a in zip(names, shapes, arrs)])  # noqa
    for r in (0, 1, 2):
        h = H.encode_handle(ck(curr, 1), ck(prev, 0), r, IDENTITY)
        wire = H.write_patch_bytes(h)
        assert wire == want[r], (name, r)
        back = H.read_patch_bytes(wire)
        out = H.decode(ck(prev, 0), back, verify_hash=True)
        assert all(np.array_equal(t.data, c) for t, c in zip(out.tensors, curr))
    torch.cuda.synchronize()
    print(f"[sanitize] {name}: ok", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true", help="skip the 16M case (racecheck is slow)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for case in golden_cases():
        run_case(*case)
    if not args.small and have_reference():
        R = reference()
        prev, curr = R.generate_synthetic([(4096, 4096)], 0.99, 64, 7)
        want = R.encode_pulps(curr, prev)
        run_case("config1_16M", ["tensor_00"], [(4096, 4096)], [prev.tensors[0].data], [curr.tensors[0].data], want)
    # dense tickets: element-mode staging and overfull re-stream in K1
    rng = np.random.default_rng(4)
    a = rng.integers(0, 65536, 65536 * 5 + 77, dtype=np.uint16)
    b = a.copy()
    b[: 65536 * 2] ^= 1
    b[65536 * 3: 65536 * 3 + 20000] ^= 1
    b[rng.random(a.size) < 0.3] ^= 2
    S = restatement()
    want = {}
    from oracle.oracle import Checkpoint, Tensor
    cp, cc = Checkpoint(0, [Tensor("dense", (a.size,), a)]), Checkpoint(1, [Tensor("dense", (a.size,), b)])
    for r in (0, 1, 2):
        want[r] = S.write_patch_bytes_identity(S.encode(cc, cp, r, IDENTITY))
    run_case("dense_tickets", ["dense"], [(a.size,)], [a], [b], want)
    print("[sanitize] all cases ok")


if __name__ == "__main__":
    main()
