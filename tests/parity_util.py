"""Test helpers for parity at BASELINE sizes (test infrastructure only).

* `device_pair`: a name-sorted state dict generated on the device (K5, the
  benchmark's own inputs) in one arena, with per-tensor views (`DeviceState`).
* `host_checkpoint`: the D2H copy of such a state as an oracle Checkpoint, so
  the reference (oracle/_ref) encodes exactly the bytes the GPU encoded
  ("D2H copies of the *same* device inputs fed to the
  reference `pulse::encode`").
* `ShardedSim`: N ranks of `shard.ShardedPulse` simulated
  on ONE device without NCCL.  Each rank gets a DevicePlan over its contiguous
  name-ordered range (`shapes.shard`), its K1 summary lands in its slot of a
  shared `gathered` buffer (what the all-gather would produce), K2 runs with
  (n_ranks, rank), and the rank-major concatenation of the sections must be
  the reference PULP body; apply takes each rank's FLAT carry from the
  gathered summaries on the device, as the bench step does.
"""
from __future__ import annotations

import json
import struct

import numpy as np
import torch

from oracle.oracle import Checkpoint, Tensor
from paper_2602_03839_b200 import device as D
from paper_2602_03839_b200.shapes import numel, shard


def split_pulp(wire: bytes):
    assert wire[:4] == b"PULP"
    _, hlen = struct.unpack_from("<IQ", wire, 4)
    return json.loads(wire[16:16 + hlen]), wire[16 + hlen:]


class DeviceState:
    def __init__(self, tensors, buf: torch.Tensor, offs):
        self.tensors = list(tensors)
        self.buf = buf
        self.offs = offs

    def views(self, lo=0, hi=None):
        hi = len(self.tensors) if hi is None else hi
        return [self.buf[int(self.offs[i]):int(self.offs[i + 1])] for i in range(lo, hi)]


def device_pair(tensors, sparsity, cluster_width, seed, device="cuda"):
    """(prev, curr) DeviceStates: log-normal base + clustered LSB flips (K5)."""
    sizes = [numel(s) for _, s in tensors]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    prev = torch.empty(max(8, int(offs[-1])), dtype=torch.int16, device=device)
    curr = torch.empty_like(prev)
    D.synth_base(prev, seed=seed)
    D.synth_mutate(prev, curr, sparsity, cluster_width, seed=seed + 1)
    return DeviceState(tensors, prev, offs), DeviceState(tensors, curr, offs)


def host_checkpoint(st: DeviceState, step: int, lo=0, hi=None) -> Checkpoint:
    hi = len(st.tensors) if hi is None else hi
    host = st.buf[int(st.offs[lo]):int(st.offs[hi])].cpu().numpy().view(np.uint16)
    base = int(st.offs[lo])
    return Checkpoint(step, [Tensor(n, tuple(s), host[int(st.offs[i]) - base:int(st.offs[i + 1]) - base])
                             for i, (n, s) in enumerate(st.tensors[lo:hi], start=lo)])


class ShardedSim:
    """N ranks' plans over one device; see the module docstring."""

    def __init__(self, tensors, n_ranks: int, max_changes_frac: float = 0.0102):
        self.tensors = list(tensors)
        self.n = n_ranks
        self.bounds = shard(self.tensors, n_ranks)
        self.gathered = torch.zeros(32 * n_ranks, dtype=torch.uint8, device="cuda")
        self.plans = []
        for r in range(n_ranks):
            mine = self.tensors[self.bounds[r]:self.bounds[r + 1]]
            d = sum(numel(s) for _, s in mine)
            cap = int(d * max_changes_frac) + 65536
            # a rank with no tensors (more ranks than tensors) still runs, as ShardedPulse's would
            self.plans.append(D.DevicePlan([(numel(s), s[-1]) for _, s in mine], cap))

    def bind(self, slot: int, st: DeviceState):
        for r, p in enumerate(self.plans):
            if p is not None:
                p.bind(slot, st.views(self.bounds[r], self.bounds[r + 1]))

    def encode(self, repr_: int, curr_slot=1, prev_slot=0):
        """Returns (body bytes rank-major, entries with global tensor ids, patches)."""
        for r, p in enumerate(self.plans):
            if p is not None:
                p.scan(curr_slot, prev_slot, summary_out=self.gathered[32 * r:32 * r + 32])
        patches, bodies, ents = [], [], []
        for r, p in enumerate(self.plans):
            if p is None:
                patches.append(None)
                continue
            pt = p.new_patch(repr_)
            p.emit(pt, gathered=self.gathered, n_ranks=self.n, rank=r)
            pt.fetch()
            pt.raise_for_status([n for n, _ in self.tensors[self.bounds[r]:self.bounds[r + 1]]])
            bodies.append(pt.body[: pt.body_bytes].cpu().numpy().tobytes())
            e = pt.host_entries[: pt.n_entries].copy()
            e["tensor"] += np.uint32(self.bounds[r])
            ents.append(e)
            patches.append(pt)
        return b"".join(bodies), (np.concatenate(ents) if ents else np.zeros(0, D.N.ENTRY_DTYPE)), patches

    def apply(self, weights_slot: int, patches):
        """Every rank applies its section in place; returns the per-rank results."""
        out = []
        for r, (p, pt) in enumerate(zip(self.plans, patches)):
            if p is None:
                continue
            carry = None
            if pt.representation == 2:
                carry = torch.zeros(16, dtype=torch.uint8, device="cuda")
                D.flat_carry_from_summaries(self.gathered, r, carry)
            out.append(D.parse_result(p.apply_patch(weights_slot, pt, carry=carry)))
        return out

    def summaries(self):
        return self.gathered.cpu().numpy().view(D.N.SUMMARY_DTYPE)


def assert_entries_match_header(ents, header, tensors):
    assert len(ents) == len(header["tensors"]), (len(ents), len(header["tensors"]))
    for e, h in zip(ents, header["tensors"]):
        assert tensors[int(e["tensor"])][0] == h["name"]
        assert int(e["count"]) == h["count"]
        assert int(e["idx_nbytes"]) == h["index_nbytes"]
