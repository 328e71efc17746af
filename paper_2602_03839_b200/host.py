"""Python mirror of the reference's host-buffer API (patch.hpp, patch_file.hpp,
index_coding.hpp, compression.hpp, sha256.hpp) over the C ABI of
libpulse_cuda.so -- the same functions the C++ drop-in headers
(include/pulse/*.hpp) wrap.  Per-element work runs in the CUDA kernels.

Checkpoints are lists of (name, shape, uint16 ndarray of bf16 bit patterns).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import COO_DOWNSCALED, COO_INT32, FLAT_INT32, IDENTITY, LZ4, ZSTD1, ZSTD3, GZIP6, PulseError  # noqa: F401


@dataclass
class Tensor:
    name: str
    shape: tuple
    data: np.ndarray  # uint16, flat


@dataclass
class Checkpoint:
    step: int = 0
    tensors: list = field(default_factory=list)


@dataclass
class TensorPatch:
    name: str
    shape: tuple
    indices: np.ndarray  # int64
    values: np.ndarray   # uint16


@dataclass
class SparsePatch:
    base_step: int = 0
    target_step: int = 0
    anchor_step: int = 0
    representation: int = COO_DOWNSCALED
    codec: int = ZSTD1
    target_hash: bytes = b"\0" * 32
    tensors: list = field(default_factory=list)

    def total_changes(self) -> int:
        return sum(int(t.indices.size) for t in self.tensors)


# ---- C views ----------------------------------------------------------------------------------
class CheckpointView:
    """pulse_checkpoint over Python/numpy memory (kept alive by this object)."""

    def __init__(self, ck: Checkpoint):
        self._keep = []
        arr = (N.Tensor * max(1, len(ck.tensors)))()
        for i, t in enumerate(ck.tensors):
            shp = np.ascontiguousarray(t.shape, dtype=np.int64)
            data = np.ascontiguousarray(t.data).view(np.uint16)
            name = t.name.encode()
            self._keep += [shp, data, name]
            arr[i] = N.Tensor(name, shp.ctypes.data_as(C.POINTER(C.c_int64)), len(t.shape), data.ctypes.data, data.size)
        self._arr = arr
        self.c = N.CheckpointC(ck.step, arr, len(ck.tensors))


class PatchHandle:
    """Owns a library pulse_patch*."""

    def __init__(self, ptr=None):
        if ptr is None:
            ptr = C.c_void_p()
            N.check(N.lib.pulse_patch_new(C.byref(ptr)))
        self.ptr = ptr

    def __del__(self):
        if getattr(self, "ptr", None):
            N.lib.pulse_patch_free(self.ptr)
            self.ptr = None

    @classmethod
    def from_patch(cls, p: SparsePatch, with_indices=True):
        h = cls()
        hd = N.PatchHeader(p.base_step, p.target_step, p.anchor_step, p.representation, p.codec,
                           (C.c_uint8 * 32)(*bytes(p.target_hash)))
        N.check(N.lib.pulse_patch_set_header(h.ptr, C.byref(hd)))
        for tp in p.tensors:
            shp = np.ascontiguousarray(tp.shape, dtype=np.int64)
            idx = np.ascontiguousarray(tp.indices, dtype=np.int64)
            val = np.ascontiguousarray(tp.values, dtype=np.uint16)
            v = N.TensorPatchC(tp.name.encode(), shp.ctypes.data_as(C.POINTER(C.c_int64)), len(tp.shape),
                               idx.ctypes.data_as(C.POINTER(C.c_int64)), idx.size if with_indices else 0,
                               val.ctypes.data_as(C.POINTER(C.c_uint16)), val.size)
            N.check(N.lib.pulse_patch_add_tensor(h.ptr, C.byref(v)))
        return h

    def to_patch(self) -> SparsePatch:
        hd = N.PatchHeader()
        N.check(N.lib.pulse_patch_get_header(self.ptr, C.byref(hd)))
        p = SparsePatch(hd.base_step, hd.target_step, hd.anchor_step, hd.representation, hd.codec, bytes(hd.target_hash))
        for i in range(N.lib.pulse_patch_num_tensors(self.ptr)):
            v = N.TensorPatchC()
            N.check(N.lib.pulse_patch_get_tensor(self.ptr, i, C.byref(v)))
            idx = np.ctypeslib.as_array(v.indices, (v.n_indices,)).copy() if v.n_indices else np.zeros(0, np.int64)
            val = np.ctypeslib.as_array(v.values, (v.n_values,)).copy() if v.n_values else np.zeros(0, np.uint16)
            p.tensors.append(TensorPatch(v.name.decode(), tuple(v.shape[k] for k in range(v.rank)), idx, val))
        return p


def _take(b) -> bytes:
    n = N.lib.pulse_bytes_size(b)
    out = C.string_at(N.lib.pulse_bytes_data(b), n) if n else b""
    N.lib.pulse_bytes_free(b)
    return out


# ---- the reference API ---------------------------------------------------------------------------
def encode_handle(current: Checkpoint, previous: Checkpoint, representation=COO_DOWNSCALED, codec=ZSTD1,
                  views=None) -> PatchHandle:
    cv, pv = views or (CheckpointView(current), CheckpointView(previous))
    out = C.c_void_p()
    N.check(N.lib.pulse_encode(C.byref(cv.c), C.byref(pv.c), representation, codec, C.byref(out)))
    return PatchHandle(out)


def encode(current: Checkpoint, previous: Checkpoint, representation=COO_DOWNSCALED, codec=ZSTD1) -> SparsePatch:
    """patch.hpp:264-307"""
    return encode_handle(current, previous, representation, codec).to_patch()


def decode_into(previous: Checkpoint, patch, out_arrays, verify_hash=True, view=None) -> int:
    """patch.hpp:309-348 into caller arrays (one per tensor of `previous`); returns the step."""
    pv = view or CheckpointView(previous)
    h = patch if isinstance(patch, PatchHandle) else PatchHandle.from_patch(patch)
    ptrs = (C.c_void_p * max(1, len(out_arrays)))(*[a.ctypes.data for a in out_arrays])
    step = C.c_uint64()
    N.check(N.lib.pulse_decode(C.byref(pv.c), h.ptr, int(verify_hash), ptrs, C.byref(step)))
    return step.value


def decode(previous: Checkpoint, patch, verify_hash=True) -> Checkpoint:
    outs = [np.empty(t.data.size, np.uint16) for t in previous.tensors]
    step = decode_into(previous, patch, outs, verify_hash)
    return Checkpoint(step, [Tensor(t.name, t.shape, o) for t, o in zip(previous.tensors, outs)])


def encode_index_payloads(patch: SparsePatch) -> list:
    """patch.hpp:116-174"""
    h = PatchHandle.from_patch(patch)
    sizes = (C.c_uint64 * max(1, len(patch.tensors)))()
    b = C.c_void_p()
    N.check(N.lib.pulse_encode_index_payloads(h.ptr, C.byref(b), sizes))
    blob = _take(b)
    out, off = [], 0
    for i in range(len(patch.tensors)):
        out.append(blob[off:off + sizes[i]])
        off += sizes[i]
    return out


def decode_index_payloads(patch: SparsePatch, payloads: list) -> SparsePatch:
    """patch.hpp:178-262 (counts = len(values)); returns the patch with indices."""
    h = PatchHandle.from_patch(patch, with_indices=False)
    bufs = [C.create_string_buffer(p, len(p)) for p in payloads]
    ptrs = (C.c_void_p * max(1, len(bufs)))(*[C.addressof(b) for b in bufs])
    sizes = (C.c_uint64 * max(1, len(bufs)))(*[len(p) for p in payloads])
    N.check(N.lib.pulse_decode_index_payloads(h.ptr, ptrs, sizes, len(payloads)))
    return h.to_patch()


def write_patch_bytes(patch) -> bytes:
    """patch_file.hpp:30-83"""
    h = patch if isinstance(patch, PatchHandle) else PatchHandle.from_patch(patch)
    b = C.c_void_p()
    N.check(N.lib.pulse_write_patch_bytes(h.ptr, C.byref(b)))
    return _take(b)



def write_patch_array(patch) -> np.ndarray:
    """write_patch_bytes as a uint8 ndarray (the reference's Bytes is a byte
    vector) viewing the library's buffer directly -- no copy of the 100s of MB;
    the buffer is freed when the array (and any view of it) is."""
    h = patch if isinstance(patch, PatchHandle) else PatchHandle.from_patch(patch)
    b = C.c_void_p()
    N.check(N.lib.pulse_write_patch_bytes(h.ptr, C.byref(b)))
    n = N.lib.pulse_bytes_size(b)
    if not n:
        N.lib.pulse_bytes_free(b)
        return np.empty(0, np.uint8)
    raw = (C.c_uint8 * n).from_address(N.lib.pulse_bytes_data(b))
    weakref.finalize(raw, N.lib.pulse_bytes_free, b)
    return np.frombuffer(raw, np.uint8)


def read_patch_handle(data) -> PatchHandle:
    """read_patch_bytes into a library patch handle; `data` is bytes or a uint8 ndarray."""
    out = C.c_void_p()
    if isinstance(data, np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.uint8)
        N.check(N.lib.pulse_read_patch_bytes(C.cast(a.ctypes.data, C.c_char_p), a.size, C.byref(out)))
    else:
        N.check(N.lib.pulse_read_patch_bytes(data, len(data), C.byref(out)))
    return PatchHandle(out)


def read_patch_bytes(data: bytes) -> SparsePatch:
    """patch_file.hpp:85-147"""
    return read_patch_handle(data).to_patch()


def hash_weights(ck: Checkpoint) -> bytes:
    """sha256.hpp:93-116"""
    v = CheckpointView(ck)
    out = C.create_string_buffer(32)
    N.check(N.lib.pulse_hash_weights(C.byref(v.c), out))
    return out.raw


def delta_encode_indices(idx) -> np.ndarray:
    a = np.ascontiguousarray(idx, np.int64)
    out = np.empty_like(a)
    N.check(N.lib.pulse_delta_encode_indices(a.ctypes.data_as(C.POINTER(C.c_int64)), a.size,
                                             out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def delta_decode_indices(gaps) -> np.ndarray:
    a = np.ascontiguousarray(gaps, np.int64)
    out = np.empty_like(a)
    N.check(N.lib.pulse_delta_decode_indices(a.ctypes.data_as(C.POINTER(C.c_int64)), a.size,
                                             out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def downscale_coo(rows, cols) -> bytes:
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    b = C.c_void_p()
    N.check(N.lib.pulse_downscale_coo(r.ctypes.data_as(C.POINTER(C.c_int64)), r.size,
                                      c.ctypes.data_as(C.POINTER(C.c_int64)), c.size, C.byref(b)))
    return _take(b)


def upscale_coo(data: bytes, count: int):
    rows = np.empty(count, np.int64)
    cols = np.empty(count, np.int64)
    N.check(N.lib.pulse_upscale_coo(data, len(data), count, rows.ctypes.data_as(C.POINTER(C.c_int64)),
                                    cols.ctypes.data_as(C.POINTER(C.c_int64))))
    return rows, cols


def compress(data: bytes, codec: int) -> bytes:
    b = C.c_void_p()
    N.check(N.lib.pulse_compress(data, len(data), codec, C.byref(b)))
    return _take(b)


def decompress(data: bytes, codec: int) -> bytes:
    b = C.c_void_p()
    N.check(N.lib.pulse_decompress(data, len(data), codec, C.byref(b)))
    return _take(b)


@dataclass
class SparsityReport:
    k: int = 1
    changed: int = 0
    total: int = 0
    sparsity: float = 1.0


def sparsity(a: Checkpoint, b: Checkpoint, k: int = 1) -> SparsityReport:
    """absorption.hpp:55-78 (one device pass over both snapshots)."""
    va, vb = CheckpointView(a), CheckpointView(b)
    r = N.SparsityReportC()
    N.check(N.lib.pulse_sparsity(C.byref(va.c), C.byref(vb.c), k, C.byref(r)))
    return SparsityReport(r.k, r.changed, r.total, r.sparsity)


def frozen_fraction(c: Checkpoint, threshold: float) -> float:
    """absorption.hpp:38-46 (one device pass)."""
    v = CheckpointView(c)
    out = C.c_double()
    N.check(N.lib.pulse_frozen_fraction(C.byref(v.c), threshold, C.byref(out)))
    return out.value


def transfer_stats(reset=False):
    """(h2d_bytes, d2h_bytes) the host API has copied so far in this process."""
    a, b = C.c_uint64(), C.c_uint64()
    N.lib.pulse_transfer_stats(C.byref(a), C.byref(b), int(reset))
    return a.value, b.value


# ---- container.hpp: the PULC checkpoint container --------------------------------------------
def _buf(data):
    """(pointer, length, keep-alive) of bytes / a uint8 ndarray."""
    if isinstance(data, np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.uint8)
        return a.ctypes.data, a.size, a
    b = bytes(data)
    return C.cast(C.c_char_p(b), C.c_void_p).value, len(b), b


def write_checkpoint_bytes(ck: Checkpoint) -> bytes:
    """container.hpp:58-90 (canonical: equal checkpoints give equal bytes)."""
    v = CheckpointView(ck)
    out = C.c_void_p()
    N.check(N.lib.pulse_write_checkpoint_bytes(C.byref(v.c), 0, C.byref(out)))
    return _take(out)


class Container:
    """A parsed PULC container (container.hpp:92-142 checks); tensors refer to
    the caller's bytes by payload offset."""

    def __init__(self, data):
        self._ptr, self._n, self._keep = _buf(data)
        h = C.c_void_p()
        N.check(N.lib.pulse_container_parse(self._ptr, self._n, C.byref(h)))
        self.h = h
        self.step = int(N.lib.pulse_container_step(h))
        self.tensors = []
        for i in range(N.lib.pulse_container_num_tensors(h)):
            t = N.ContainerTensorC()
            N.check(N.lib.pulse_container_get_tensor(h, i, C.byref(t)))
            self.tensors.append((t.name.decode(), tuple(t.shape[k] for k in range(t.rank)), int(t.numel),
                                 int(t.payload_offset)))

    def __del__(self):
        if getattr(self, "h", None):
            N.lib.pulse_container_free(self.h)
            self.h = None

    def copy_out(self, dst_ptrs, device: bool):
        arr = (C.c_void_p * max(1, len(dst_ptrs)))(*dst_ptrs)
        N.check(N.lib.pulse_container_copy_out(self.h, self._ptr, self._n, int(device), arr))


def read_checkpoint_bytes(data) -> Checkpoint:
    """container.hpp:92-142"""
    c = Container(data)
    out = Checkpoint(c.step, [Tensor(n, s, np.empty(k, np.uint16)) for n, s, k, _ in c.tensors])
    c.copy_out([t.data.ctypes.data for t in out.tensors], device=False)
    return out


def read_checkpoint_to_device(data, device_tensors) -> Container:
    """Parse + check like read_checkpoint_bytes, then copy tensor i's payload
    straight into device_tensors[i] (a CUDA tensor of numel 2-byte elements)."""
    c = Container(data)
    if len(device_tensors) != len(c.tensors):
        raise PulseError(2, "one device tensor per container tensor required")
    for t, (name, _, k, _) in zip(device_tensors, c.tensors):
        if not t.is_cuda or t.element_size() != 2 or t.numel() != k or not t.is_contiguous():
            raise PulseError(2, f"device tensor for {name} must be a contiguous CUDA tensor of {k} 2-byte elements")
    c.copy_out([t.data_ptr() for t in device_tensors], device=True)
    return c


def write_checkpoint_bytes_from_device(step: int, names, shapes, device_tensors) -> bytes:
    """PULC bytes of a checkpoint resident in HBM (payloads copied straight out of the device)."""
    keep, arr = [], (N.Tensor * max(1, len(names)))()
    for i, (name, shape, t) in enumerate(zip(names, shapes, device_tensors)):
        shp = np.ascontiguousarray(shape, dtype=np.int64)
        nm = name.encode()
        keep += [shp, nm]
        arr[i] = N.Tensor(nm, shp.ctypes.data_as(C.POINTER(C.c_int64)), len(shape), t.data_ptr(), t.numel())
    ck = N.CheckpointC(step, arr, len(names))
    out = C.c_void_p()
    N.check(N.lib.pulse_write_checkpoint_bytes(C.byref(ck), 1, C.byref(out)))
    return _take(out)


# ---- resident checkpoints: the sync path on the device (sync.hpp) -----------------------------
class Resident:
    """A checkpoint held in HBM with its step and weights hash (the consumer's
    SyncState, sync.hpp:78-92, and the publisher's last published snapshot).
    apply / walk = apply_delta / walk_deltas (sync.hpp:308-352) straight from
    PULP bytes; publish = publish_checkpoint's patch (sync.hpp:166-181) encoded
    on the device against the held weights."""

    def __init__(self, ck: Checkpoint, max_changes: int = 1 << 20):
        v = CheckpointView(ck)
        h = C.c_void_p()
        N.check(N.lib.pulse_resident_create(C.byref(v.c), max_changes, C.byref(h)))
        self.h = h
        self.names = [t.name for t in ck.tensors]
        self.shapes = [tuple(t.shape) for t in ck.tensors]

    @classmethod
    def from_device(cls, step: int, names, shapes, device_tensors, max_changes: int = 1 << 20):
        """A resident copy of a checkpoint already in HBM (CUDA tensors of 2-byte elements)."""
        keep, arr = [], (N.Tensor * max(1, len(names)))()
        for i, (name, shape, t) in enumerate(zip(names, shapes, device_tensors)):
            shp = np.ascontiguousarray(shape, dtype=np.int64)
            nm = name.encode()
            keep += [shp, nm]
            arr[i] = N.Tensor(nm, shp.ctypes.data_as(C.POINTER(C.c_int64)), len(shape), t.data_ptr(), t.numel())
        ck = N.CheckpointC(step, arr, len(names))
        self = cls.__new__(cls)
        h = C.c_void_p()
        N.check(N.lib.pulse_resident_create_device(C.byref(ck), max_changes, C.byref(h)))
        self.h = h
        self.names = list(names)
        self.shapes = [tuple(s) for s in shapes]
        return self

    def __del__(self):
        if getattr(self, "h", None):
            N.lib.pulse_resident_destroy(self.h)
            self.h = None

    @property
    def step(self) -> int:
        return int(N.lib.pulse_resident_step(self.h))

    @property
    def last_anchor_step(self) -> int:
        return int(N.lib.pulse_resident_last_anchor_step(self.h))

    @property
    def weights_hash(self) -> bytes:
        out = C.create_string_buffer(32)
        N.check(N.lib.pulse_resident_hash(self.h, out))
        return out.raw

    def tensor_ptr(self, i: int) -> int:
        p = C.c_void_p()
        N.check(N.lib.pulse_resident_tensor(self.h, i, C.byref(p)))
        return int(p.value)

    def download(self) -> Checkpoint:
        outs = [np.empty(int(np.prod(s)), np.uint16) for s in self.shapes]
        arr = (C.c_void_p * max(1, len(outs)))(*[o.ctypes.data for o in outs])
        N.check(N.lib.pulse_resident_download(self.h, arr))
        return Checkpoint(self.step, [Tensor(n, s, o) for n, s, o in zip(self.names, self.shapes, outs)])

    def apply(self, pulp, step: int, expected_hash: bytes | None = None, verify: bool = True):
        ptr, n, keep = _buf(pulp)
        N.check(N.lib.pulse_resident_apply(self.h, ptr, n, step, expected_hash, int(verify)))
        del keep

    def walk(self, pulps, verify: bool = True) -> int:
        bufs = [_buf(p) for p in pulps]
        ptrs = (C.c_void_p * max(1, len(bufs)))(*[b[0] for b in bufs])
        sizes = (C.c_uint64 * max(1, len(bufs)))(*[b[1] for b in bufs])
        applied = C.c_uint32()
        try:
            N.check(N.lib.pulse_resident_walk(self.h, ptrs, sizes, len(bufs), int(verify), C.byref(applied)))
        finally:
            self.last_walk_applied = applied.value
        return applied.value

    def publish(self, device_tensors, step: int, representation=COO_DOWNSCALED, codec=ZSTD1,
                anchor_step: int | None = None, advance: bool = True):
        """(PULP bytes, target hash) of the snapshot in `device_tensors` (CUDA
        tensors, this checkpoint's tensor order) at `step` = held step + 1."""
        arr = (C.c_void_p * max(1, len(device_tensors)))(*[t.data_ptr() for t in device_tensors])
        out = C.c_void_p()
        hsh = C.create_string_buffer(32)
        anchor = self.step if anchor_step is None else anchor_step
        N.check(N.lib.pulse_resident_publish(self.h, arr, step, representation, codec, anchor, int(advance),
                                             C.byref(out), hsh))
        return _take(out), hsh.raw


# ---- end-to-end benchmark leg ---------------------------------------------------------------------
def bench_e2e(args, mine, prev_dev, curr_dev, world, rank, steps=None, warmup=3):
    """The benchmark metric measured end to end through the public host API.

    Every step runs encode -> write_patch_bytes -> read_patch_bytes ->
    decode(verify_hash=False) on snapshots held in pinned host memory, so it
    includes all host->device copies of the inputs and device->host reads of
    the results (and encode's SHA-256 target hash, as the reference's encode
    does).  The snapshots are the same bytes as the device-resident run
    (copied out once, untimed).  Wall-clock per step, max over ranks; the
    bytes moved are the library's own counters (pulse_transfer_stats)."""
    import os
    import sys
    import time

    import torch
    import torch.distributed as dist

    from .shapes import numel

    sizes = [numel(s) for _, s in mine]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    hp = torch.empty(prev_dev.numel(), dtype=torch.int16).pin_memory()
    hc = torch.empty(curr_dev.numel(), dtype=torch.int16).pin_memory()
    ho = torch.empty(prev_dev.numel(), dtype=torch.int16).pin_memory()
    hp.copy_(prev_dev.view(torch.int16))
    hc.copy_(curr_dev.view(torch.int16))
    a_prev, a_curr, a_out = (t.numpy().view(np.uint16) for t in (hp, hc, ho))

    def mk(a, step):
        return Checkpoint(step, [Tensor(n, s, a[int(offs[i]):int(offs[i + 1])]) for i, (n, s) in enumerate(mine)])

    ck = {0: mk(a_prev, 0), 1: mk(a_curr, 1)}
    views = {k: CheckpointView(v) for k, v in ck.items()}
    outs = [a_out[int(offs[i]):int(offs[i + 1])] for i in range(len(sizes))]
    steps = steps or max(1, min(args.steps, 3))

    parts = {"encode": 0.0, "write": 0.0, "read": 0.0, "decode": 0.0}

    def step(k, timed=False):
        # alternate direction like the device run: prev->curr, then curr->prev
        c, p = (1, 0) if k % 2 == 0 else (0, 1)
        t0 = time.perf_counter()
        h = encode_handle(ck[c], ck[p], args.repr, IDENTITY, views=(views[c], views[p]))
        t1 = time.perf_counter()
        wire = write_patch_array(h)
        t2 = time.perf_counter()
        if os.environ.get("PULSE_TIMING"):
            print(f"[pulse timing] e2e write (incl. copy to bytes) {1e3 * (t2 - t1):.1f} ms", file=sys.stderr)
        back = read_patch_handle(wire)
        t3 = time.perf_counter()
        decode_into(ck[p], back, outs, verify_hash=False, view=views[p])
        t4 = time.perf_counter()
        if timed:
            for key, dt_ in zip(parts, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
                parts[key] += dt_
        return c

    for k in range(warmup):
        step(k)
    if world > 1:
        dist.barrier()
    transfer_stats(reset=True)
    t0 = time.perf_counter()
    for k in range(steps):
        last = step(k, timed=True)
    dt = time.perf_counter() - t0
    h2d, d2h = transfer_stats()
    ok = bool(np.array_equal(a_out, (a_curr if last == 1 else a_prev)))
    t = torch.tensor([dt / steps, float(offs[-1]), float(ok)], dtype=torch.float64)
    if world > 1:
        t = t.cuda()
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = t[1:].clone()
        dist.all_reduce(tot)
        s_step, d_total, n_ok = float(mx.item()), float(tot[0].item()), int(tot[1].item())
        ok = n_ok == world
    else:
        s_step, d_total = float(t[0]), float(t[1])
    return {"value": round(2 * d_total / s_step / 1e9, 4), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d // steps), "d2h_bytes_per_step": int(d2h // steps),
            "steps": steps, "warmup": warmup, "s_per_step": round(s_step, 4), "verified": ok,
            "parts_s": {k_: round(v / steps, 4) for k_, v in parts.items()},
            "path": "pulse_encode -> pulse_write_patch_bytes (into a uint8 array) -> pulse_read_patch_bytes -> "
                    "pulse_decode(verify_hash=false); identity codec; pinned host snapshots; wall clock"}
