"""Multi-GPU PULSE: the state dict sharded by tensor, one process per GPU.

The name-sorted tensor list is cut into contiguous, byte-balanced ranges
(`shapes.shard`), so the rank-major concatenation of the per-rank patch
sections *is* the PULP blob area in name order (patch_file.hpp:34-35, 76-82).
Every rank encodes and applies its own shard independently; NCCL over NVLink
carries only:

  1. an all-gather of the 32-byte per-rank scan summaries after K1 -- the
     FLAT_INT32 stream continues across ranks (patch.hpp:131-156: each rank's
     first gap is relative to the previous rank's last changed index);
  2. an all-gather of (body bytes, entries) after K2 -- the size exchange that
     places every section in the final patch;
  3. optionally, a gather of the sections to one rank (point-to-point
     send/recv; NCCL has no gatherv) to assemble the full PULP body there.

The exchange helpers take/return torch tensors and work with any
torch.distributed backend (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

from .shapes import numel, shard

SUMMARY_BYTES = 32  # pulse_scan_summary
SIZES_FIELDS = 2    # (body_bytes, n_entries)


# ---- exchange logic (device-agnostic) ---------------------------------------------------------
def flat_carry(summaries: np.ndarray, rank: int):
    """(has_prev, gap_base) for `rank` from all ranks' scan summaries
    (structured array with has_change / last_gap_base): the nearest earlier
    rank that emitted an index continues the FLAT_INT32 gap stream."""
    for q in range(rank - 1, -1, -1):
        if int(summaries[q]["has_change"]):
            return 1, int(summaries[q]["last_gap_base"])
    return 0, 0


def section_offsets(body_bytes, n_entries):
    """Byte offset and first entry index of every rank's section in the full
    patch (rank-major)."""
    b = np.asarray(body_bytes, dtype=np.int64)
    e = np.asarray(n_entries, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(b)])[:-1], np.concatenate([[0], np.cumsum(e)])[:-1]


def all_gather_bytes(local: torch.Tensor, world: int) -> torch.Tensor:
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local)
    return out


def exchange_sizes(body_bytes: int, n_entries: int, device) -> tuple[np.ndarray, np.ndarray]:
    """Size exchange: every rank learns every section's (body bytes, entries)."""
    world = dist.get_world_size()
    t = torch.tensor([body_bytes, n_entries], dtype=torch.int64, device=device)
    g = all_gather_bytes(t, world).view(world, SIZES_FIELDS).cpu().numpy()
    return g[:, 0], g[:, 1]


def gather_sections(section: torch.Tensor, sizes, root: int = 0):
    """Gather every rank's section (uint8, `sizes[r]` bytes) to `root`; returns
    the concatenation on root, None elsewhere."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank == root:
        total = int(np.sum(sizes))
        out = torch.empty(max(1, total), dtype=torch.uint8, device=section.device)
        offs, _ = section_offsets(sizes, np.zeros(len(sizes)))
        ops = []
        for q in range(world):
            n = int(sizes[q])
            if n == 0:
                continue
            dst = out[int(offs[q]):int(offs[q]) + n]
            if q == rank:
                dst.copy_(section[:n])
            else:
                ops.append(dist.P2POp(dist.irecv, dst, q))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return out[:total]
    n = int(sizes[rank])
    if n:
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, section[:n].contiguous(), root)]):
            r.wait()
    return None


# ---- the sharded driver ------------------------------------------------------------------------
@dataclass
class Section:
    patch: object                 # device.DevicePatch of this rank
    summaries: np.ndarray         # all ranks' scan summaries
    body_bytes: np.ndarray        # all ranks' section sizes
    n_entries: np.ndarray
    carry: tuple                  # this rank's FLAT carry (has_prev, gap_base)


class ShardedPulse:
    """One rank's view of a sharded state dict: its tensors, its plan, and the
    collectives that tie the sections together."""

    def __init__(self, tensors, max_change_frac: float = 0.0102, device=None):
        from . import device as D

        self.D = D
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.tensors = list(tensors)
        self.bounds = shard(self.tensors, self.world)
        self.mine = self.tensors[self.bounds[self.rank]:self.bounds[self.rank + 1]]
        self.sizes = [numel(s) for _, s in self.mine]
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        cap = int(sum(self.sizes) * max_change_frac) + 65536
        self.plan = D.DevicePlan([(n, s[-1]) for n, (_, s) in zip(self.sizes, self.mine)], cap)
        self.send = torch.zeros(SUMMARY_BYTES, dtype=torch.uint8, device=self.device)
        self.gathered = torch.zeros(SUMMARY_BYTES * self.world, dtype=torch.uint8, device=self.device)
        self.carry_dev = torch.zeros(16, dtype=torch.uint8, device=self.device)
        # device-side size exchange: bytes 8..24 of every rank's pulse_result
        # (body_bytes u64, n_entries u32, status i32)
        self.size_send = torch.zeros(16, dtype=torch.uint8, device=self.device)
        self.sizes_all = torch.zeros(16 * self.world, dtype=torch.uint8, device=self.device)
        self.apply_res = torch.zeros(72, dtype=torch.uint8, device=self.device)
        self._side = None
        # FLAT summaries over NVLink: 2 x world 64-byte slots per rank, an epoch per call
        self.sum_table = torch.zeros(2 * self.world * 64, dtype=torch.uint8, device=self.device)
        self.sum_epoch = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._peer_sizes = self._open_peer_sizes() if self.world > 1 else None
        self._peer_ptrs = None
        self._sum_ptrs = None
        if self._peer_sizes is not None:  # this rank's 16-byte slot in every rank's table
            self._peer_ptrs = [p + 16 * self.rank for p in self._peer_sizes]
        # FLAT_INT32's summary all-gather over NVLink (pulse_peer_allgather, device-side wait):
        # 2.67 vs 2.70-2.71 ms per step with NCCL at 2 GPUs, 1.43-1.52 vs 1.44-1.47 at 4 (one run
        # on another box: 2.04; profiles/r2l_peer_sizes.txt); PULSE_PEER_SUMMARIES=0 uses NCCL
        if self._peer_sizes is not None and os.environ.get("PULSE_PEER_SUMMARIES", "1") == "1":
            try:
                self._sum_ptrs = self._map_peers(self.sum_table)
                ok = torch.tensor([1], device=self.device)
            except Exception as exc:  # noqa: BLE001
                print(f"[shard] rank {self.rank}: NVLink summary table unavailable ({exc}); using NCCL",
                      file=sys.stderr)
                ok = torch.tensor([0], device=self.device)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) != 1:
                self._sum_ptrs = None

    def _map_peers(self, t: torch.Tensor):
        """Device addresses, valid for this device's kernels, of every rank's copy of `t`
        (same shape on every rank): CUDA IPC handles exchanged once with all_gather_object."""
        share = t.untyped_storage()._share_cuda_()  # (device, handle, size, offset, ...)
        handle = bytes(share[1])
        # torch's caching allocator prefixes the 64-byte cudaIpcMemHandle_t with a format
        # version byte and the segment kind, b"c" for a cudaMalloc segment (expandable
        # segments would need the cuMem API: not supported here, NCCL is used instead)
        if len(handle) == 66 and handle[1:2] == b"c":
            handle = handle[2:]
        if len(handle) != 64:
            raise ValueError(f"unsupported CUDA IPC handle ({len(handle)} bytes)")
        shares = [None] * self.world
        dist.all_gather_object(shares, (handle, int(share[3])))
        return [t.data_ptr() if r == self.rank else self.D.ipc_open(shares[r][0], self.device.index) + shares[r][1]
                for r in range(self.world)]

    def _open_peer_sizes(self):
        """Device addresses of every rank's `sizes_all`, mapped for this device over NVLink
        (CUDA IPC handles exchanged once with all_gather_object), so the per-step size
        exchange is world-1 16-byte peer stores instead of an NCCL all-gather: in the step graphs the
        collective cost 0.02-0.75 ms at 4 GPUs (its kernel waits behind the apply grids and
        the slowest rank).  None -> NCCL (PULSE_PEER_SIZES=0, or IPC / peer access missing)."""
        if os.environ.get("PULSE_PEER_SIZES", "1") == "0":
            return None
        try:
            ptrs = self._map_peers(self.sizes_all)
            ok = torch.tensor([1], device=self.device)
        except Exception as exc:  # noqa: BLE001  (no IPC / peer access: every rank falls back together)
            print(f"[shard] rank {self.rank}: NVLink size table unavailable ({type(exc).__name__}: {exc}); "
                  "using NCCL", file=sys.stderr)
            ptrs, ok = None, torch.tensor([0], device=self.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        return ptrs if int(ok.item()) == 1 else None

    def bind(self, slot: int, local_tensors):
        self.plan.bind(slot, local_tensors)

    def new_patch(self, representation: int):
        return self.plan.new_patch(representation)

    def encode(self, curr_slot: int, prev_slot: int, patch, sizes: bool = True) -> Section:
        """K1 -> all-gather summaries -> K2 (FLAT continued across ranks) ->
        D2H of this section's entry table -> size exchange."""
        self.plan.scan(curr_slot, prev_slot, summary_out=self.send)
        return self.encode_after_scan(patch, sizes)

    def encode_after_scan(self, patch, sizes: bool = True) -> Section:
        if self.world > 1:
            dist.all_gather_into_tensor(self.gathered, self.send)
            self.plan.emit(patch, gathered=self.gathered, n_ranks=self.world, rank=self.rank)
        else:
            self.plan.emit(patch)
        patch.fetch()
        if self.world > 1:
            summ = self.gathered.cpu().numpy().view(self.D.N.SUMMARY_DTYPE)
        else:
            summ = self.send.cpu().numpy().view(self.D.N.SUMMARY_DTYPE)
        carry = flat_carry(summ, self.rank)
        if sizes and self.world > 1:
            bb, ne = exchange_sizes(patch.body_bytes, patch.n_entries, self.device)
        else:
            bb, ne = np.array([patch.body_bytes]), np.array([patch.n_entries])
        return Section(patch, summ, bb, ne, carry)

    def apply(self, weights_slot: int, sec: Section):
        """Validate-then-scatter this rank's section into its resident shard."""
        carry = None
        if sec.patch.representation == 2 and sec.carry[0]:
            # a fresh device buffer per call (synchronous copy from pageable memory):
            # a later apply cannot overwrite the carry an earlier queued apply reads
            carry = torch.from_numpy(np.array(sec.carry, np.uint64).view(np.uint8)).to(self.device)
        return self.plan.apply(weights_slot, sec.patch, carry=carry)

    # ---- fully device-side step (no host round trip) ---------------------------------------------
    def emit_async(self, patch):
        """After scan(): K2 and the size exchange, stream-ordered, nothing read
        back to the host.  Only FLAT_INT32 needs other ranks before K2 (its gap
        stream continues across shards): it all-gathers the scan summaries and
        derives the carry on the device.  The other representations emit
        independently, and the (body bytes, entries) exchange runs on a side
        stream, overlapped with apply (join with `join()`)."""
        if self.world == 1:
            self.plan.emit(patch)
            return
        main = torch.cuda.current_stream(self.device)
        if patch.representation == 2:
            if self._sum_ptrs is not None:  # device-side all-gather over NVLink (no collective)
                self.D.peer_allgather(self.send, self._sum_ptrs, self.rank, SUMMARY_BYTES, self.sum_epoch,
                                      self.gathered)
            else:
                dist.all_gather_into_tensor(self.gathered, self.send)
            self.plan.emit(patch, gathered=self.gathered, n_ranks=self.world, rank=self.rank)
            self.D.flat_carry_from_summaries(self.gathered, self.rank, self.carry_dev)
        else:
            self.plan.emit(patch)
        if os.environ.get("PULSE_SKIP_SIZE_EXCHANGE"):  # attribution experiment only
            return
        if self._peer_ptrs is not None:
            # this rank's (body bytes, entries, status) stored straight into every rank's
            # table over NVLink by one kernel; readers look after a device sync + barrier
            self.D.store_to_peers(patch.result[8:24], self._peer_ptrs, 16)
            return
        self.size_send.copy_(patch.result[8:24])
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        self._side.wait_stream(main)
        with torch.cuda.stream(self._side):
            dist.all_gather_into_tensor(self.sizes_all, self.size_send)

    def join(self):
        """Make the current stream wait for the side-stream size exchange."""
        if self._side is not None:
            torch.cuda.current_stream(self.device).wait_stream(self._side)

    def apply_async(self, weights_slot: int, patch):
        """Apply this rank's section with the entry count read on the device."""
        carry = self.carry_dev if (self.world > 1 and patch.representation == 2) else None
        return self.plan.apply_patch(weights_slot, patch, carry=carry, result=self.apply_res)

    def exchanged_sizes(self):
        """Host view of the last device-side size exchange: (body_bytes, n_entries, status) per rank.
        With peer stores, call after every rank synchronised its device (e.g. synchronize + barrier)."""
        raw = self.sizes_all.cpu().numpy().reshape(self.world, 16)
        body = raw[:, 0:8].copy().view(np.uint64)[:, 0]
        ent = raw[:, 8:12].copy().view(np.uint32)[:, 0]
        st = raw[:, 12:16].copy().view(np.int32)[:, 0]
        return body, ent, st

    def gather(self, sec: Section, root: int = 0):
        """Full PULP body and entry table (global tensor ids) on `root`."""
        body = gather_sections(sec.patch.body, sec.body_bytes, root)
        n = int(sec.patch.n_entries)
        ent = torch.from_numpy(sec.patch.host_entries[:n].view(np.uint8).copy()).to(self.device)
        # entries are variable-count per rank: pad to the max and all-gather
        mx = int(np.max(sec.n_entries)) if len(sec.n_entries) else 0
        pad = torch.zeros(max(1, mx) * 40, dtype=torch.uint8, device=self.device)
        pad[: ent.numel()] = ent
        allent = all_gather_bytes(pad, self.world).cpu().numpy() if self.world > 1 else pad.cpu().numpy()
        if self.rank != root:
            return None, None
        boffs, _ = section_offsets(sec.body_bytes, sec.n_entries)
        rows = []
        per = max(1, mx) * 40
        for q in range(self.world):
            e = allent[q * per:q * per + int(sec.n_entries[q]) * 40].view(self.D.N.ENTRY_DTYPE).copy()
            e["tensor"] += np.uint32(self.bounds[q])
            e["idx_off"] += np.uint64(boffs[q])
            e["val_off"] += np.uint64(boffs[q])
            rows.append(e)
        return body, (np.concatenate(rows) if rows else np.zeros(0, self.D.N.ENTRY_DTYPE))
