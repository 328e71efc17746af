"""ORACLE / TEST INFRASTRUCTURE ONLY -- never imported by the product package.

Two CPU checkers for the CUDA path, both loaded with ctypes:

* ``Reference`` wraps ``oracle/_ref/libpulse_ref.so``: the unmodified reference
  headers (/root/reference/proj/include/pulse) behind ``oracle/ref_shim.cpp``.
  It is the ground truth where it exists (built here, shipped prebuilt to the
  GPU box).
* ``Restatement`` wraps ``oracle/liboracle.so`` (``oracle/pulse_oracle.c``), a
  plain-C restatement of the reference arithmetic, plus the PULP identity
  writer restated below in Python (patch_file.hpp:30-83).  It is pinned by
  tests/test_oracle.py against the reference's own known-answer vectors and the
  golden fixtures in tests/golden/.

Only tests/, ``__graft_entry__.smoke()`` and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpulse_ref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

# Representation / codec numbering: patch.hpp:20-24, compression.hpp:31-37.
COO_DOWNSCALED, COO_INT32, FLAT_INT32 = 0, 1, 2
REPR_NAMES = {0: "COO_DOWNSCALED", 1: "COO_INT32", 2: "FLAT_INT32"}
IDENTITY, LZ4, ZSTD1, ZSTD3, GZIP6 = 0, 1, 2, 3, 4

# include/pulse_cuda.h status numbering (shared with ref_shim.cpp).
STATUS_NAMES = {
    1: "Error", 2: "ArgumentError", 3: "FormatError", 4: "BadMagicError", 5: "VersionError",
    6: "TruncationError", 7: "CorruptStreamError", 8: "ModelMismatchError",
    9: "ShapeMismatchError", 10: "TensorSetError", 11: "IndexRangeError",
    12: "DimensionError", 13: "HashMismatchError",
}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))
        self.msg = msg


@dataclass
class Tensor:
    name: str
    shape: tuple
    data: np.ndarray  # uint16 bit patterns, flat


@dataclass
class Checkpoint:
    step: int
    tensors: list = field(default_factory=list)

    def total_elements(self) -> int:
        return sum(int(t.data.size) for t in self.tensors)

    def sorted(self):
        return sorted(self.tensors, key=lambda t: t.name.encode())


@dataclass
class TensorPatch:
    name: str
    shape: tuple
    indices: np.ndarray  # int64
    values: np.ndarray  # uint16


@dataclass
class Patch:
    base_step: int = 0
    target_step: int = 0
    anchor_step: int = 0
    representation: int = COO_DOWNSCALED
    codec: int = ZSTD1
    target_hash: bytes = b"\0" * 32
    tensors: list = field(default_factory=list)

    def total_changes(self) -> int:
        return sum(int(tp.indices.size) for tp in self.tensors)


# ------------------------------------------------------------------------------------------
# The reference itself
# ------------------------------------------------------------------------------------------
class Reference:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.L = C.CDLL(path)
        vp, u64, i64, u32, u16 = C.c_void_p, C.c_uint64, C.c_int64, C.c_uint32, C.c_uint16
        pp = C.POINTER
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_ckpt_new": (vp, [u64]),
            "ref_ckpt_free": (None, [vp]),
            "ref_ckpt_add": (None, [vp, C.c_char_p, pp(i64), u32, vp, u64]),
            "ref_ckpt_step": (u64, [vp]),
            "ref_ckpt_num_tensors": (u32, [vp]),
            "ref_ckpt_tensor": (None, [vp, u32, pp(C.c_char_p), pp(pp(i64)), pp(u32), pp(vp), pp(u64)]),
            "ref_generate_synthetic": (C.c_int, [pp(i64), pp(u32), u32, C.c_double, i64, u64, pp(vp), pp(vp)]),
            "ref_mutate": (C.c_int, [vp, C.c_double, i64, u64, u64, pp(vp)]),
            "ref_round_to_bf16": (u16, [C.c_double]),
            "ref_hash_weights": (C.c_int, [vp, C.c_char_p]),
            "ref_sha256": (None, [C.c_char_p, u64, C.c_char_p]),
            "ref_patch_free": (None, [vp]),
            "ref_patch_new": (vp, []),
            "ref_patch_header": (None, [vp, pp(i64), pp(u32), pp(u32), C.c_char_p]),
            "ref_patch_set_header": (None, [vp, pp(i64), u32, u32, C.c_char_p]),
            "ref_patch_num_tensors": (u32, [vp]),
            "ref_patch_tensor": (None, [vp, u32, pp(C.c_char_p), pp(pp(i64)), pp(u32), pp(pp(i64)), pp(u64), pp(vp), pp(u64)]),
            "ref_patch_add_tensor": (None, [vp, C.c_char_p, pp(i64), u32, pp(i64), u64, vp, u64]),
            "ref_encode": (C.c_int, [vp, vp, u32, u32, pp(vp)]),
            "ref_decode": (C.c_int, [vp, vp, C.c_int, pp(vp)]),
            "ref_buf_free": (None, [vp]),
            "ref_buf_data": (vp, [vp]),
            "ref_buf_size": (u64, [vp]),
            "ref_write_patch_bytes": (C.c_int, [vp, pp(vp)]),
            "ref_read_patch_bytes": (C.c_int, [C.c_char_p, u64, pp(vp)]),
            "ref_encode_index_payloads": (C.c_int, [vp, pp(vp), pp(u64)]),
            "ref_decode_index_payloads": (C.c_int, [vp, C.c_char_p, pp(u64)]),
            "ref_downscale_coo": (C.c_int, [pp(i64), u64, pp(i64), u64, pp(vp)]),
            "ref_upscale_coo": (C.c_int, [C.c_char_p, u64, u64, pp(i64), pp(i64)]),
            "ref_delta_encode": (C.c_int, [pp(i64), u64, pp(i64)]),
            "ref_delta_decode": (C.c_int, [pp(i64), u64, pp(i64)]),
            "ref_compress": (C.c_int, [C.c_char_p, u64, u32, pp(vp)]),
            "ref_decompress": (C.c_int, [C.c_char_p, u64, u32, pp(vp)]),
            "ref_write_checkpoint_bytes": (C.c_int, [vp, pp(vp)]),
            "ref_read_checkpoint_bytes": (C.c_int, [C.c_char_p, u64, pp(vp)]),
            "ref_sparsity": (C.c_int, [vp, vp, pp(u64), pp(u64)]),
            "ref_frozen_fraction": (C.c_int, [vp, C.c_double, pp(C.c_double)]),
            "ref_time_step": (C.c_int, [vp, vp, u32, u32, C.c_int] + [pp(C.c_double)] * 5 + [pp(u64), pp(u64)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # -- plumbing -----------------------------------------------------------------------
    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.L.ref_last_error().decode(errors="replace"))

    def _take_buf(self, h) -> bytes:
        n = self.L.ref_buf_size(h)
        # (ctypes.string_at takes a C int size: buffers of 2 GiB and more go through an array view)
        out = bytes((C.c_char * n).from_address(self.L.ref_buf_data(h))) if n else b""
        self.L.ref_buf_free(h)
        return out

    @staticmethod
    def _i64(a):
        a = np.ascontiguousarray(a, dtype=np.int64)
        return a, a.ctypes.data_as(C.POINTER(C.c_int64))

    def ckpt_handle(self, ck: Checkpoint):
        h = self.L.ref_ckpt_new(ck.step)
        for t in ck.tensors:
            shp, shp_p = self._i64(t.shape)
            d = np.ascontiguousarray(t.data, dtype=np.uint16)
            self.L.ref_ckpt_add(h, t.name.encode(), shp_p, len(t.shape), d.ctypes.data, d.size)
        return h

    def ckpt_from_handle(self, h, free=True) -> Checkpoint:
        ck = Checkpoint(step=int(self.L.ref_ckpt_step(h)))
        for i in range(self.L.ref_ckpt_num_tensors(h)):
            name, shp, rank, data, numel = C.c_char_p(), C.POINTER(C.c_int64)(), C.c_uint32(), C.c_void_p(), C.c_uint64()
            self.L.ref_ckpt_tensor(h, i, C.byref(name), C.byref(shp), C.byref(rank), C.byref(data), C.byref(numel))
            shape = tuple(shp[k] for k in range(rank.value))
            arr = np.empty(numel.value, dtype=np.uint16)
            if numel.value:
                C.memmove(arr.ctypes.data, data.value, numel.value * 2)
            ck.tensors.append(Tensor(name.value.decode(), shape, arr))
        if free:
            self.L.ref_ckpt_free(h)
        return ck

    def patch_handle(self, p: Patch):
        h = self.L.ref_patch_new()
        steps = (C.c_int64 * 3)(p.base_step, p.target_step, p.anchor_step)
        self.L.ref_patch_set_header(h, steps, p.representation, p.codec, bytes(p.target_hash))
        for tp in p.tensors:
            shp, shp_p = self._i64(tp.shape)
            idx, idx_p = self._i64(tp.indices)
            v = np.ascontiguousarray(tp.values, dtype=np.uint16)
            self.L.ref_patch_add_tensor(h, tp.name.encode(), shp_p, len(tp.shape), idx_p, idx.size, v.ctypes.data, v.size)
        return h

    def patch_from_handle(self, h, free=True) -> Patch:
        steps = (C.c_int64 * 3)()
        repr_, codec = C.c_uint32(), C.c_uint32()
        hb = C.create_string_buffer(32)
        self.L.ref_patch_header(h, steps, C.byref(repr_), C.byref(codec), hb)
        p = Patch(steps[0], steps[1], steps[2], repr_.value, codec.value, hb.raw)
        for i in range(self.L.ref_patch_num_tensors(h)):
            name, shp, rank = C.c_char_p(), C.POINTER(C.c_int64)(), C.c_uint32()
            idx, nidx, val, nval = C.POINTER(C.c_int64)(), C.c_uint64(), C.c_void_p(), C.c_uint64()
            self.L.ref_patch_tensor(h, i, C.byref(name), C.byref(shp), C.byref(rank), C.byref(idx), C.byref(nidx), C.byref(val), C.byref(nval))
            ia = np.ctypeslib.as_array(idx, shape=(nidx.value,)).copy() if nidx.value else np.empty(0, np.int64)
            va = np.empty(nval.value, dtype=np.uint16)
            if nval.value:
                C.memmove(va.ctypes.data, val.value, nval.value * 2)
            p.tensors.append(TensorPatch(name.value.decode(), tuple(shp[k] for k in range(rank.value)), ia, va))
        if free:
            self.L.ref_patch_free(h)
        return p

    # -- reference API ------------------------------------------------------------------
    def generate_synthetic(self, shapes, sparsity=0.99, cluster_width=64, seed=0):
        flat = [int(x) for s in shapes for x in s]
        shp, shp_p = self._i64(flat)
        ranks = (C.c_uint32 * len(shapes))(*[len(s) for s in shapes])
        a, b = C.c_void_p(), C.c_void_p()
        self._check(self.L.ref_generate_synthetic(shp_p, ranks, len(shapes), sparsity, cluster_width, seed, C.byref(a), C.byref(b)))
        return self.ckpt_from_handle(a.value), self.ckpt_from_handle(b.value)

    def mutate(self, base: Checkpoint, sparsity, cluster_width, seed, new_step) -> Checkpoint:
        h = self.ckpt_handle(base)
        out = C.c_void_p()
        try:
            self._check(self.L.ref_mutate(h, sparsity, cluster_width, seed, new_step, C.byref(out)))
        finally:
            self.L.ref_ckpt_free(h)
        return self.ckpt_from_handle(out.value)

    def round_to_bf16(self, x: float) -> int:
        return int(self.L.ref_round_to_bf16(x))

    def hash_weights(self, ck: Checkpoint) -> bytes:
        h = self.ckpt_handle(ck)
        out = C.create_string_buffer(32)
        try:
            self._check(self.L.ref_hash_weights(h, out))
        finally:
            self.L.ref_ckpt_free(h)
        return out.raw

    def sha256(self, data: bytes) -> bytes:
        out = C.create_string_buffer(32)
        self.L.ref_sha256(data, len(data), out)
        return out.raw

    def encode(self, cur: Checkpoint, prev: Checkpoint, repr_=COO_DOWNSCALED, codec=ZSTD1) -> Patch:
        hc, hp = self.ckpt_handle(cur), self.ckpt_handle(prev)
        out = C.c_void_p()
        try:
            self._check(self.L.ref_encode(hc, hp, repr_, codec, C.byref(out)))
        finally:
            self.L.ref_ckpt_free(hc)
            self.L.ref_ckpt_free(hp)
        return self.patch_from_handle(out.value)

    def encode_pulps(self, cur: Checkpoint, prev: Checkpoint, reprs=(COO_DOWNSCALED, COO_INT32, FLAT_INT32),
                     codec=IDENTITY):
        """{representation: write_patch_bytes(encode(cur, prev, repr, codec))}: one
        reference encode (the patch's indices and values do not depend on the
        representation, patch.hpp:296-301), then the representation field is
        switched on the same patch object before each write."""
        hc, hp = self.ckpt_handle(cur), self.ckpt_handle(prev)
        out = C.c_void_p()
        try:
            self._check(self.L.ref_encode(hc, hp, reprs[0], codec, C.byref(out)))
        finally:
            self.L.ref_ckpt_free(hc)
            self.L.ref_ckpt_free(hp)
        h = out.value
        try:
            steps = (C.c_int64 * 3)()
            r_, c_ = C.c_uint32(), C.c_uint32()
            hb = C.create_string_buffer(32)
            self.L.ref_patch_header(h, steps, C.byref(r_), C.byref(c_), hb)
            wires = {}
            for r in reprs:
                self.L.ref_patch_set_header(h, steps, r, codec, hb.raw)
                buf = C.c_void_p()
                self._check(self.L.ref_write_patch_bytes(h, C.byref(buf)))
                wires[r] = self._take_buf(buf.value)
            return wires
        finally:
            self.L.ref_patch_free(h)

    def decode(self, prev: Checkpoint, patch: Patch, verify=True) -> Checkpoint:
        hp, hq = self.ckpt_handle(prev), self.patch_handle(patch)
        out = C.c_void_p()
        try:
            self._check(self.L.ref_decode(hp, hq, int(verify), C.byref(out)))
        finally:
            self.L.ref_ckpt_free(hp)
            self.L.ref_patch_free(hq)
        return self.ckpt_from_handle(out.value)

    def write_patch_bytes(self, patch: Patch) -> bytes:
        h = self.patch_handle(patch)
        out = C.c_void_p()
        try:
            self._check(self.L.ref_write_patch_bytes(h, C.byref(out)))
        finally:
            self.L.ref_patch_free(h)
        return self._take_buf(out.value)

    def read_patch_bytes(self, data: bytes) -> Patch:
        out = C.c_void_p()
        self._check(self.L.ref_read_patch_bytes(data, len(data), C.byref(out)))
        return self.patch_from_handle(out.value)

    def encode_index_payloads(self, patch: Patch) -> list:
        h = self.patch_handle(patch)
        sizes = (C.c_uint64 * max(1, len(patch.tensors)))()
        out = C.c_void_p()
        try:
            self._check(self.L.ref_encode_index_payloads(h, C.byref(out), sizes))
        finally:
            self.L.ref_patch_free(h)
        blob = self._take_buf(out.value)
        res, off = [], 0
        for i in range(len(patch.tensors)):
            res.append(blob[off:off + sizes[i]])
            off += sizes[i]
        return res

    def decode_index_payloads(self, patch: Patch, payloads: list) -> Patch:
        """Fills indices from payloads (counts = len(values)); returns a new Patch."""
        h = self.patch_handle(patch)
        sizes = (C.c_uint64 * max(1, len(payloads)))(*[len(p) for p in payloads])
        try:
            self._check(self.L.ref_decode_index_payloads(h, b"".join(payloads), sizes))
            return self.patch_from_handle(h, free=False)
        finally:
            self.L.ref_patch_free(h)

    def downscale_coo(self, rows, cols) -> bytes:
        r, rp = self._i64(rows)
        c, cp = self._i64(cols)
        out = C.c_void_p()
        self._check(self.L.ref_downscale_coo(rp, r.size, cp, c.size, C.byref(out)))
        return self._take_buf(out.value)

    def upscale_coo(self, data: bytes, count: int):
        rows = np.empty(count, np.int64)
        cols = np.empty(count, np.int64)
        self._check(self.L.ref_upscale_coo(data, len(data), count, rows.ctypes.data_as(C.POINTER(C.c_int64)), cols.ctypes.data_as(C.POINTER(C.c_int64))))
        return rows, cols

    def delta_encode(self, idx):
        a, ap = self._i64(idx)
        out = np.empty(a.size, np.int64)
        self._check(self.L.ref_delta_encode(ap, a.size, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def delta_decode(self, gaps):
        a, ap = self._i64(gaps)
        out = np.empty(a.size, np.int64)
        self._check(self.L.ref_delta_decode(ap, a.size, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def compress(self, data: bytes, codec: int) -> bytes:
        out = C.c_void_p()
        self._check(self.L.ref_compress(data, len(data), codec, C.byref(out)))
        return self._take_buf(out.value)

    def decompress(self, data: bytes, codec: int) -> bytes:
        out = C.c_void_p()
        self._check(self.L.ref_decompress(data, len(data), codec, C.byref(out)))
        return self._take_buf(out.value)

    def write_checkpoint_bytes(self, ck: Checkpoint) -> bytes:
        h = self.ckpt_handle(ck)
        out = C.c_void_p()
        try:
            self._check(self.L.ref_write_checkpoint_bytes(h, C.byref(out)))
        finally:
            self.L.ref_ckpt_free(h)
        return self._take_buf(out.value)

    def read_checkpoint_bytes(self, data: bytes) -> Checkpoint:
        out = C.c_void_p()
        self._check(self.L.ref_read_checkpoint_bytes(data, len(data), C.byref(out)))
        return self.ckpt_from_handle(out.value)

    def sparsity(self, a: Checkpoint, b: Checkpoint):
        """absorption.hpp:55-78 -> (changed, total)"""
        ha, hb = self.ckpt_handle(a), self.ckpt_handle(b)
        ch, tot = C.c_uint64(), C.c_uint64()
        try:
            self._check(self.L.ref_sparsity(ha, hb, C.byref(ch), C.byref(tot)))
        finally:
            self.L.ref_ckpt_free(ha)
            self.L.ref_ckpt_free(hb)
        return ch.value, tot.value

    def frozen_fraction(self, c: Checkpoint, threshold: float) -> float:
        """absorption.hpp:38-46"""
        h = self.ckpt_handle(c)
        out = C.c_double()
        try:
            self._check(self.L.ref_frozen_fraction(h, threshold, C.byref(out)))
        finally:
            self.L.ref_ckpt_free(h)
        return out.value

    def time_step(self, prev_h, curr_h, repr_=COO_DOWNSCALED, codec=IDENTITY, verify=False):
        """Times one reference step on prebuilt handles (see ref_shim.cpp ref_time_step)."""
        t = [C.c_double() for _ in range(5)]
        nbytes, changes = C.c_uint64(), C.c_uint64()
        self._check(self.L.ref_time_step(prev_h, curr_h, repr_, codec, int(verify), *[C.byref(x) for x in t], C.byref(nbytes), C.byref(changes)))
        keys = ("encode", "write", "read", "decode", "hash")
        return dict(zip(keys, [x.value for x in t])), nbytes.value, changes.value


# ------------------------------------------------------------------------------------------
# The restatement
# ------------------------------------------------------------------------------------------
class Restatement:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        vp, u64, i64, u32 = C.c_void_p, C.c_uint64, C.c_int64, C.c_uint32
        L.po_diff.restype = u64
        L.po_diff.argtypes = [vp, vp, u64, vp, vp]
        for n in ("po_delta_encode", "po_delta_decode"):
            getattr(L, n).restype = C.c_int
            getattr(L, n).argtypes = [vp, u64, vp]
        L.po_payload_coo_int32.restype = C.c_int
        L.po_payload_coo_int32.argtypes = [vp, u64, u64, vp, C.POINTER(u64)]
        L.po_payload_flat.restype = C.c_int
        L.po_payload_flat.argtypes = [u32, vp, vp, vp, vp, vp]
        L.po_downscale_coo.restype = C.c_int
        L.po_downscale_coo.argtypes = [vp, vp, u64, vp, C.POINTER(u64)]
        L.po_payload_coo_ds.restype = C.c_int
        L.po_payload_coo_ds.argtypes = [vp, u64, i64, vp, vp, vp, C.POINTER(u64)]
        L.po_upscale_coo.restype = C.c_int
        L.po_upscale_coo.argtypes = [vp, u64, u64, vp, vp]
        L.po_decode_payloads.restype = C.c_int
        L.po_decode_payloads.argtypes = [u32, u32, vp, vp, vp, vp, vp, vp, vp, vp, C.POINTER(u32)]
        L.po_apply.restype = C.c_int
        L.po_apply.argtypes = [vp, u64, vp, vp, u64]
        L.po_sha256_ctx_size.restype = u64
        L.po_sha256_init.argtypes = [vp]
        L.po_sha256_update.argtypes = [vp, vp, u64]
        L.po_sha256_final.argtypes = [vp, vp]

    @staticmethod
    def _raise(rc, what=""):
        if rc:
            raise OracleError(rc, what)

    # patch.hpp:296-301
    def diff(self, prev: np.ndarray, curr: np.ndarray):
        prev = np.ascontiguousarray(prev, np.uint16)
        curr = np.ascontiguousarray(curr, np.uint16)
        n = self.L.po_diff(prev.ctypes.data, curr.ctypes.data, prev.size, None, None)
        idx = np.empty(n, np.int64)
        val = np.empty(n, np.uint16)
        self.L.po_diff(prev.ctypes.data, curr.ctypes.data, prev.size, idx.ctypes.data, val.ctypes.data)
        return idx, val

    # patch.hpp:264-307 (hash via the restated SHA-256)
    def encode(self, cur: Checkpoint, prev: Checkpoint, repr_=COO_DOWNSCALED, codec=ZSTD1) -> Patch:
        p = Patch(prev.step, cur.step, prev.step, repr_, codec, self.hash_weights(cur))
        for c, q in zip(cur.sorted(), prev.sorted()):
            assert c.name == q.name and tuple(c.shape) == tuple(q.shape)
            idx, val = self.diff(q.data, c.data)
            if idx.size:
                p.tensors.append(TensorPatch(c.name, tuple(c.shape), idx, val))
        return p

    def delta_encode(self, idx):
        a = np.ascontiguousarray(idx, np.int64)
        out = np.empty_like(a)
        self._raise(self.L.po_delta_encode(a.ctypes.data, a.size, out.ctypes.data))
        return out

    def delta_decode(self, gaps):
        a = np.ascontiguousarray(gaps, np.int64)
        out = np.empty_like(a)
        self._raise(self.L.po_delta_decode(a.ctypes.data, a.size, out.ctypes.data))
        return out

    def downscale_coo(self, rows, cols) -> bytes:
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(cols, np.int64)
        if r.size != c.size:
            raise OracleError(2, "row and column lists differ in length")
        buf = np.empty(10 * r.size + 1, np.uint8)
        nb = C.c_uint64()
        self._raise(self.L.po_downscale_coo(r.ctypes.data, c.ctypes.data, r.size, buf.ctypes.data, C.byref(nb)))
        return buf[: nb.value].tobytes()

    def upscale_coo(self, data: bytes, count: int):
        rows = np.empty(count, np.int64)
        cols = np.empty(count, np.int64)
        d = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
        self._raise(self.L.po_upscale_coo(d.ctypes.data, len(data), count, rows.ctypes.data, cols.ctypes.data))
        return rows, cols

    # patch.hpp:116-174
    def encode_index_payloads(self, patch: Patch) -> list:
        out = []
        if patch.representation == FLAT_INT32:
            n = len(patch.tensors)
            idx = [np.ascontiguousarray(tp.indices, np.int64) for tp in patch.tensors]
            ptrs = (C.c_void_p * max(1, n))(*[a.ctypes.data for a in idx])
            counts = (C.c_uint64 * max(1, n))(*[a.size for a in idx])
            numel = (C.c_uint64 * max(1, n))(*[int(np.prod(tp.shape)) for tp in patch.tensors])
            sizes = (C.c_uint64 * max(1, n))()
            buf = np.empty(4 * sum(a.size for a in idx) + 1, np.uint8)
            self._raise(self.L.po_payload_flat(n, ptrs, counts, numel, buf.ctypes.data, sizes))
            off = 0
            for i in range(n):
                out.append(buf[off:off + sizes[i]].tobytes())
                off += sizes[i]
            return out
        for tp in patch.tensors:
            idx = np.ascontiguousarray(tp.indices, np.int64)
            nb = C.c_uint64()
            if patch.representation == COO_INT32:
                buf = np.empty(4 * idx.size + 1, np.uint8)
                self._raise(self.L.po_payload_coo_int32(idx.ctypes.data, idx.size, int(np.prod(tp.shape)), buf.ctypes.data, C.byref(nb)))
            else:
                buf = np.empty(10 * idx.size + 1, np.uint8)
                rt = np.empty(max(1, idx.size), np.int64)
                ct = np.empty(max(1, idx.size), np.int64)
                self._raise(self.L.po_payload_coo_ds(idx.ctypes.data, idx.size, int(tp.shape[-1]), rt.ctypes.data, ct.ctypes.data, buf.ctypes.data, C.byref(nb)))
            out.append(buf[: nb.value].tobytes())
        return out

    # patch.hpp:178-262
    def decode_index_payloads(self, repr_, shapes, counts, payloads):
        n = len(shapes)
        bufs = [np.frombuffer(p, np.uint8) if len(p) else np.zeros(1, np.uint8) for p in payloads]
        outs = [np.empty(max(1, c), np.int64) for c in counts]
        mx = max([1] + list(counts))
        rt, ct = np.empty(mx, np.int64), np.empty(mx, np.int64)
        arr = lambda t, xs: (t * max(1, n))(*xs)
        err_t = C.c_uint32()
        rc = self.L.po_decode_payloads(
            repr_, n, arr(C.c_void_p, [b.ctypes.data for b in bufs]), arr(C.c_uint64, [len(p) for p in payloads]),
            arr(C.c_uint64, counts), arr(C.c_uint64, [int(np.prod(s)) for s in shapes]),
            arr(C.c_int64, [int(s[-1]) for s in shapes]), arr(C.c_void_p, [o.ctypes.data for o in outs]),
            rt.ctypes.data, ct.ctypes.data, C.byref(err_t))
        if rc:
            raise OracleError(rc, f"tensor {err_t.value}")
        return [o[:c] for o, c in zip(outs, counts)]

    # patch.hpp:309-348 (verify via the restated SHA-256)
    def decode(self, prev: Checkpoint, patch: Patch, verify=True) -> Checkpoint:
        out = Checkpoint(patch.target_step, [Tensor(t.name, t.shape, t.data.copy()) for t in prev.tensors])
        by_name = {t.name: t for t in out.tensors}
        for tp in patch.tensors:
            t = by_name.get(tp.name)
            if t is None:
                raise OracleError(10, "unknown tensor")
            if tuple(t.shape) != tuple(tp.shape):
                raise OracleError(9, "shape")
            if tp.indices.size != tp.values.size:
                raise OracleError(2, "count")
            idx = np.ascontiguousarray(tp.indices, np.int64)
            val = np.ascontiguousarray(tp.values, np.uint16)
            self._raise(self.L.po_apply(t.data.ctypes.data, t.data.size, idx.ctypes.data, val.ctypes.data, idx.size))
        if verify and self.hash_weights(out) != patch.target_hash:
            raise OracleError(13, "hash mismatch")
        return out

    def sha256_stream(self, chunks) -> bytes:
        ctx = C.create_string_buffer(self.L.po_sha256_ctx_size())
        self.L.po_sha256_init(ctx)
        for ch in chunks:
            a = np.ascontiguousarray(np.frombuffer(ch, np.uint8) if isinstance(ch, (bytes, bytearray)) else ch)
            if a.nbytes:
                self.L.po_sha256_update(ctx, a.ctypes.data, a.nbytes)
        out = C.create_string_buffer(32)
        self.L.po_sha256_final(ctx, out)
        return out.raw

    def sha256(self, data: bytes) -> bytes:
        return self.sha256_stream([data])

    # sha256.hpp:93-116: raw LE bf16 bytes, tensors in ascending (bytewise) name order
    def hash_weights(self, ck: Checkpoint) -> bytes:
        return self.sha256_stream([np.ascontiguousarray(t.data, np.uint16).view(np.uint8) for t in ck.sorted()])

    # patch_file.hpp:30-83, identity codec: magic, u32 version 1, u64 header length,
    # nlohmann dump() of a sorted-key object, then [index blob][value blob] per tensor.
    def write_patch_bytes_identity(self, patch: Patch) -> bytes:
        payloads = self.encode_index_payloads(patch)
        header = pulp_header_json(patch, [len(p) for p in payloads], [2 * tp.values.size for tp in patch.tensors])
        body = b"".join(p + np.ascontiguousarray(tp.values, np.uint16).tobytes() for p, tp in zip(payloads, patch.tensors))
        return b"PULP" + struct.pack("<IQ", 1, len(header)) + header + body


def pulp_header_json(patch: Patch, index_nbytes, value_nbytes) -> bytes:
    """The PULP JSON header exactly as nlohmann::json::dump() renders it
    (patch_file.hpp:52-74): std::map key order, no whitespace."""
    tensors = []
    for tp, inb, vnb in zip(patch.tensors, index_nbytes, value_nbytes):
        e = {"name": tp.name, "shape": [int(x) for x in tp.shape], "count": int(tp.indices.size),
             "index_nbytes": int(inb), "value_nbytes": int(vnb)}
        if patch.representation == COO_DOWNSCALED:
            e["row_bits"] = 8
            e["col_bits"] = 16
        tensors.append(e)
    obj = {"anchor_step": int(patch.anchor_step), "base_step": int(patch.base_step),
           "target_step": int(patch.target_step), "target_hash": bytes(patch.target_hash).hex(),
           "codec": int(patch.codec), "representation": REPR_NAMES[patch.representation],
           "tensors": tensors}
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), ensure_ascii=False).encode()


_REF = None
_RES = None


def reference() -> Reference:
    global _REF
    if _REF is None:
        _REF = Reference()
    return _REF


def restatement() -> Restatement:
    global _RES
    if _RES is None:
        _RES = Restatement()
    return _RES


def have_reference() -> bool:
    return os.path.exists(REF_SO)
