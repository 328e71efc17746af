"""Device-resident PULSE: encode/apply over bf16 snapshots already in HBM.

torch supplies device memory and streams (plumbing only); every kernel is in
libpulse_cuda.so.  Typical use on one GPU:

    plan = DevicePlan([(numel, cols), ...], max_changes)      # name-sorted tensors
    plan.bind(0, prev_tensors); plan.bind(1, curr_tensors); plan.bind(2, weights)
    patch = plan.encode(curr_slot=1, prev_slot=0, representation=COO_DOWNSCALED)
    plan.apply(2, patch)        # weights[slot 2] := curr, bit-exact, in place

`DevicePatch` is the device image of a PULP body: per changed tensor
[index payload][value payload] in name order (patch_file.hpp:76-82, identity
codec) plus the entry table that the PULP JSON header is written from.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._native import COO_DOWNSCALED, COO_INT32, FLAT_INT32, PulseError  # noqa: F401


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class DevicePatch:
    representation: int
    body: torch.Tensor          # uint8 [capacity] on device
    entries: torch.Tensor       # uint8 [n_tensors * 40] on device (pulse_patch_entry[])
    result: torch.Tensor        # uint8 [72] on device (pulse_result)
    host_result: np.ndarray | None = None
    host_entries: np.ndarray | None = None

    def fetch(self, stream=None) -> "DevicePatch":
        """D2H of the result and entry table (small); synchronizes the stream."""
        r = self.result.to("cpu", non_blocking=False).numpy().view(N.RESULT_DTYPE)[0]
        wd = N.watchdog()
        if wd is not None:
            raise PulseError(14, f"device watchdog fired: kind={wd[1]} block={wd[2]} thread={wd[3]} "
                                 f"a={wd[4]} b={wd[5]} c={wd[6]:#x}")
        self.host_result = r
        n = int(r["n_entries"])
        self.host_entries = self.entries[: n * 40].to("cpu").numpy().view(N.ENTRY_DTYPE).copy()
        return self

    @property
    def status(self) -> int:
        return int(self.host_result["status"])

    @property
    def n_entries(self) -> int:
        return int(self.host_result["n_entries"])

    @property
    def body_bytes(self) -> int:
        return int(self.host_result["body_bytes"])

    @property
    def n_changes(self) -> int:
        return int(self.host_result["n_changes"])

    def raise_for_status(self, names=None):
        r = self.host_result
        if int(r["status"]) != 0:
            t = int(r["err_tensor"])
            where = names[t] if names is not None and t < len(names) else f"#{t}"
            raise PulseError(int(r["status"]), f"{N.CHECK_NAMES.get(int(r['err_check']), '?')} in tensor '{where}' "
                                               f"(element {int(r['err_elem'])}; required {int(r['required'])})")


class DevicePlan:
    def __init__(self, geoms, max_changes: int, device: int | None = None):
        self.device = torch.cuda.current_device() if device is None else device
        self.geoms = [(int(n), int(c)) for n, c in geoms]
        self.n_tensors = len(self.geoms)
        self.max_changes = int(max_changes)
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib.pulse_context_create(self.device, C.byref(ctx)))
            self._ctx = ctx
            arr = (N.TensorGeom * max(1, self.n_tensors))(*[N.TensorGeom(n, c) for n, c in self.geoms])
            plan = C.c_void_p()
            N.check(N.lib.pulse_plan_create(ctx, arr, self.n_tensors, self.max_changes, C.byref(plan)))
        self._plan = plan
        self._bound = {}

    def close(self):
        if getattr(self, "_plan", None):
            N.lib.pulse_plan_destroy(self._plan)
            self._plan = None
        if getattr(self, "_ctx", None):
            N.lib.pulse_context_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- binding ------------------------------------------------------------------------
    def bind(self, slot: int, tensors):
        """Bind one device tensor per plan tensor (bf16 / int16 / uint16, contiguous)."""
        tensors = list(tensors)
        if len(tensors) != self.n_tensors:
            raise ValueError("one tensor per plan tensor")
        for t, (n, _) in zip(tensors, self.geoms):
            if t.numel() != n or t.element_size() != 2 or not t.is_contiguous() or t.device.index != self.device:
                raise ValueError("tensor does not match plan geometry / device / layout")
        ptrs = (C.c_void_p * max(1, self.n_tensors))(*[t.data_ptr() for t in tensors])
        N.check(N.lib.pulse_plan_bind(self._plan, slot, ptrs))
        self._bound[slot] = tensors  # keep alive

    # ---- buffers ------------------------------------------------------------------------
    def body_capacity(self, representation: int) -> int:
        per = 9 if representation == COO_DOWNSCALED else 6  # worst case index + value bytes
        return per * self.max_changes + 16

    def new_patch(self, representation: int, body_capacity: int | None = None) -> DevicePatch:
        cap = body_capacity or self.body_capacity(representation)
        dev = torch.device("cuda", self.device)
        return DevicePatch(representation,
                           torch.empty(cap, dtype=torch.uint8, device=dev),
                           torch.zeros(max(1, self.n_tensors) * 40, dtype=torch.uint8, device=dev),
                           torch.zeros(72, dtype=torch.uint8, device=dev))

    # ---- encode -------------------------------------------------------------------------
    def scan(self, curr_slot: int, prev_slot: int, summary_out: torch.Tensor | None = None, stream=None):
        """K1.  `summary_out` (32-byte uint8 device tensor) receives a copy of the
        pulse_scan_summary, e.g. an NCCL all-gather send buffer."""
        N.check(N.lib.pulse_encode_scan(self._plan, curr_slot, prev_slot, _ptr(summary_out), _stream_ptr(stream)))

    def scan_summary_ptr(self) -> int:
        return N.lib.pulse_plan_scan_summary(self._plan)

    def emit(self, patch: DevicePatch, gathered: torch.Tensor | None = None, n_ranks: int = 1, rank: int = 0,
             stream=None):
        N.check(N.lib.pulse_encode_emit(self._plan, patch.representation, _ptr(gathered), n_ranks, rank,
                                        _ptr(patch.body), patch.body.numel(), _ptr(patch.entries),
                                        _ptr(patch.result), _stream_ptr(stream)))

    def encode(self, curr_slot: int, prev_slot: int, representation: int = COO_DOWNSCALED,
               patch: DevicePatch | None = None, stream=None, fetch=True) -> DevicePatch:
        patch = patch or self.new_patch(representation)
        patch.representation = representation
        self.scan(curr_slot, prev_slot, stream=stream)
        self.emit(patch, stream=stream)
        if fetch:
            patch.fetch(stream)
        return patch

    # ---- apply / decode -----------------------------------------------------------------
    def apply(self, weights_slot: int, patch: DevicePatch, n_entries: int | None = None,
              carry: torch.Tensor | None = None, result: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Validate-then-scatter `patch` into the tensors bound at `weights_slot`.
        Returns the device pulse_result (72 bytes)."""
        n = patch.n_entries if n_entries is None else n_entries
        res = result if result is not None else torch.zeros(72, dtype=torch.uint8, device=patch.body.device)
        N.check(N.lib.pulse_apply(self._plan, weights_slot, patch.representation, _ptr(patch.body),
                                  _ptr(patch.entries), n, _ptr(carry), _ptr(res), _stream_ptr(stream)))
        return res

    def apply_patch(self, weights_slot: int, patch: DevicePatch, carry: torch.Tensor | None = None,
                    result: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """apply() with the entry count read on the device from the patch's
        encode result (no host round trip; a failed encode applies nothing)."""
        res = result if result is not None else torch.zeros(72, dtype=torch.uint8, device=patch.body.device)
        N.check(N.lib.pulse_apply_patch(self._plan, weights_slot, patch.representation, _ptr(patch.body),
                                        _ptr(patch.entries), _ptr(patch.result), _ptr(carry), _ptr(res),
                                        _stream_ptr(stream)))
        return res

    def decode_indices(self, patch: DevicePatch, n_entries: int | None = None, carry: torch.Tensor | None = None,
                       stream=None):
        n = patch.n_entries if n_entries is None else n_entries
        total = int(sum(int(e["count"]) for e in patch.host_entries[:n])) if patch.host_entries is not None else self.max_changes
        out = torch.empty(max(1, total), dtype=torch.int64, device=patch.body.device)
        res = torch.zeros(72, dtype=torch.uint8, device=patch.body.device)
        N.check(N.lib.pulse_decode_indices(self._plan, patch.representation, _ptr(patch.body), _ptr(patch.entries), n,
                                           _ptr(carry), _ptr(out), _ptr(res), _stream_ptr(stream)))
        return out[:total], res


def flat_carry_from_summaries(gathered: torch.Tensor, rank: int, out: torch.Tensor, stream=None):
    """Device-side FLAT carry (16-byte pulse_flat_carry in `out`) of shard `rank`."""
    N.check(N.lib.pulse_flat_carry_from_summaries(_ptr(gathered), rank, _ptr(out), _stream_ptr(stream)))
    return out


def store_to_peers(src: torch.Tensor, dst_ptrs, nbytes: int, stream=None):
    """`nbytes` of device `src` stored at every device address in `dst_ptrs` (ints, e.g.
    peer-mapped over NVLink), one kernel on `stream` (peer access enabled on first use)."""
    arr = (C.c_void_p * max(1, len(dst_ptrs)))(*[C.c_void_p(int(p)) for p in dst_ptrs])
    N.check(N.lib.pulse_store_to_peers(_ptr(src), arr, len(dst_ptrs), nbytes, src.device.index,
                                       _stream_ptr(stream)))


def peer_allgather(src: torch.Tensor, table_ptrs, rank: int, nbytes: int, epoch: torch.Tensor, out: torch.Tensor,
                   stream=None):
    """One `nbytes` record per rank gathered into `out` through peer-mapped slot tables
    (pulse_peer_allgather): no collective, graph-capturable."""
    arr = (C.c_void_p * max(1, len(table_ptrs)))(*[C.c_void_p(int(p)) for p in table_ptrs])
    N.check(N.lib.pulse_peer_allgather(_ptr(src), arr, len(table_ptrs), rank, nbytes, _ptr(epoch), _ptr(out),
                                       src.device.index, _stream_ptr(stream)))


def ipc_open(handle: bytes, device: int) -> int:
    """Device address of another process's allocation (its 64-byte CUDA IPC handle), mapped
    for kernels on `device` (peer access over NVLink)."""
    ptr = C.c_void_p()
    buf = C.create_string_buffer(bytes(handle), 64)
    N.check(N.lib.pulse_ipc_open(buf, int(device), C.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int, device: int):
    N.check(N.lib.pulse_ipc_close(C.c_void_p(ptr), int(device)))


def parse_result(res: torch.Tensor):
    return res.to("cpu").numpy().view(N.RESULT_DTYPE)[0]


def synth_base(out: torch.Tensor, seed: int, median: float = 0.0117, sigma: float = 1.0, stream=None):
    N.check(N.lib.pulse_synth_base(_ptr(out), out.numel(), seed, median, sigma, _stream_ptr(stream)))


_SYNTH_CTX = {}


def synth_mutate(base: torch.Tensor, out: torch.Tensor, sparsity: float, cluster_width: int, seed: int,
                 stream=None) -> int:
    dev = base.device.index
    if dev not in _SYNTH_CTX:
        ctx = C.c_void_p()
        N.check(N.lib.pulse_context_create(dev, C.byref(ctx)))
        _SYNTH_CTX[dev] = ctx
    changed = C.c_uint64()
    N.check(N.lib.pulse_synth_mutate(_SYNTH_CTX[dev], _ptr(base), _ptr(out), base.numel(), sparsity, cluster_width,
                                     seed, C.byref(changed), _stream_ptr(stream)))
    return changed.value
