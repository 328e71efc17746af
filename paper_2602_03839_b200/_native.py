"""ctypes binding of libpulse_cuda.so (include/pulse_cuda.h).

The shared library is the product: every per-element step of encode/apply
runs in its CUDA kernels.  There is no Python or CPU fallback -- if the .so is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PULSE_LIB: an alternative build of the same library (experiment variants)
LIB_PATH = os.environ.get("PULSE_LIB") or os.path.join(HERE, "libpulse_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2602_03839_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

# ---- status codes (pulse_status) ---------------------------------------------------------
STATUS = {
    0: "OK", 1: "Error", 2: "ArgumentError", 3: "FormatError", 4: "BadMagicError", 5: "VersionError",
    6: "TruncationError", 7: "CorruptStreamError", 8: "ModelMismatchError", 9: "ShapeMismatchError",
    10: "TensorSetError", 11: "IndexRangeError", 12: "DimensionError", 13: "HashMismatchError",
    14: "CudaError", 15: "CapacityError", 16: "ProtocolViolationError",
}
COO_DOWNSCALED, COO_INT32, FLAT_INT32 = 0, 1, 2
IDENTITY, LZ4, ZSTD1, ZSTD3, GZIP6 = 0, 1, 2, 3, 4


class PulseError(Exception):
    """Raised for any non-OK pulse_status; `.kind` is the reference exception
    class name (error.hpp)."""

    def __init__(self, status: int, msg: str = ""):
        self.status = int(status)
        self.kind = STATUS.get(self.status, str(status))
        super().__init__(f"{self.kind}: {msg}" if msg else self.kind)


def check(status: int):
    if status != 0:
        raise PulseError(status, lib.pulse_last_error().decode(errors="replace"))


# ---- structs -------------------------------------------------------------------------------
class TensorGeom(C.Structure):
    _fields_ = [("numel", C.c_uint64), ("cols", C.c_uint64)]


class FlatCarry(C.Structure):
    _fields_ = [("has_prev", C.c_uint64), ("gap_base", C.c_uint64)]


class ScanSummary(C.Structure):
    _fields_ = [("n_changes", C.c_uint64), ("has_change", C.c_uint64), ("last_gap_base", C.c_uint64),
                ("status", C.c_uint64)]


class PatchEntry(C.Structure):
    _fields_ = [("tensor", C.c_uint32), ("reserved", C.c_uint32), ("count", C.c_uint64),
                ("idx_off", C.c_uint64), ("idx_nbytes", C.c_uint64), ("val_off", C.c_uint64)]


class Result(C.Structure):
    _fields_ = [("n_changes", C.c_uint64), ("body_bytes", C.c_uint64), ("n_entries", C.c_uint32),
                ("status", C.c_int32), ("err_check", C.c_uint32), ("err_stage", C.c_uint32),
                ("err_tensor", C.c_uint64), ("err_elem", C.c_uint64), ("required", C.c_uint64),
                ("carry_out", FlatCarry)]


ENTRY_DTYPE = np.dtype([("tensor", "<u4"), ("reserved", "<u4"), ("count", "<u8"), ("idx_off", "<u8"),
                        ("idx_nbytes", "<u8"), ("val_off", "<u8")])
RESULT_DTYPE = np.dtype([("n_changes", "<u8"), ("body_bytes", "<u8"), ("n_entries", "<u4"), ("status", "<i4"),
                         ("err_check", "<u4"), ("err_stage", "<u4"), ("err_tensor", "<u8"), ("err_elem", "<u8"),
                         ("required", "<u8"), ("carry_has_prev", "<u8"), ("carry_gap_base", "<u8")])
SUMMARY_DTYPE = np.dtype([("n_changes", "<u8"), ("has_change", "<u8"), ("last_gap_base", "<u8"), ("status", "<u8")])
assert C.sizeof(PatchEntry) == ENTRY_DTYPE.itemsize == 40
assert C.sizeof(Result) == RESULT_DTYPE.itemsize == 72
assert C.sizeof(ScanSummary) == SUMMARY_DTYPE.itemsize == 32

# Which reference check failed (PULSE_CHECK_*), for messages.
CHECK_NAMES = {
    1: "truncated", 2: "zero index gap", 3: "non-positive column gap within a row",
    4: "column index out of range", 5: "index out of range", 6: "trailing bytes",
    7: "negative index", 8: "indices must be strictly increasing", 9: "index gap exceeds 32 bits",
    10: "row gap exceeds 32 bits", 11: "column entry exceeds 32 bits",
    12: "too large for 32-bit indices", 13: "indices are not strictly increasing", 14: "index out of range",
    15: "capacity",
}

class Tensor(C.Structure):
    _fields_ = [("name", C.c_char_p), ("shape", C.POINTER(C.c_int64)), ("rank", C.c_uint32),
                ("data", C.c_void_p), ("numel", C.c_uint64)]


class CheckpointC(C.Structure):
    _fields_ = [("step", C.c_uint64), ("tensors", C.POINTER(Tensor)), ("n_tensors", C.c_uint32)]


class PatchHeader(C.Structure):
    _fields_ = [("base_step", C.c_int64), ("target_step", C.c_int64), ("anchor_step", C.c_int64),
                ("representation", C.c_uint32), ("codec", C.c_uint32), ("target_hash", C.c_uint8 * 32)]


class TensorPatchC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("shape", C.POINTER(C.c_int64)), ("rank", C.c_uint32),
                ("indices", C.POINTER(C.c_int64)), ("n_indices", C.c_uint64),
                ("values", C.POINTER(C.c_uint16)), ("n_values", C.c_uint64)]


class ContainerTensorC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("shape", C.POINTER(C.c_int64)), ("rank", C.c_uint32),
                ("numel", C.c_uint64), ("payload_offset", C.c_uint64)]


class SparsityReportC(C.Structure):
    _fields_ = [("k", C.c_uint64), ("changed", C.c_uint64), ("total", C.c_uint64), ("sparsity", C.c_double)]


vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
_SIGS = {
    "pulse_last_error": (C.c_char_p, []),
    "pulse_version": (C.c_char_p, []),
    "pulse_watchdog": (C.c_int, [C.POINTER(C.c_uint64)]),
    "pulse_context_create": (i32, [C.c_int, C.POINTER(vp)]),
    "pulse_context_destroy": (None, [vp]),
    "pulse_plan_create": (i32, [vp, C.POINTER(TensorGeom), u32, u64, C.POINTER(vp)]),
    "pulse_plan_destroy": (None, [vp]),
    "pulse_plan_bind": (i32, [vp, u32, C.POINTER(vp)]),
    "pulse_encode_scan": (i32, [vp, u32, u32, vp, vp]),
    "pulse_plan_scan_summary": (vp, [vp]),
    "pulse_plan_trace": (vp, [vp, C.POINTER(u64)]),
    "pulse_encode_emit": (i32, [vp, u32, vp, u32, u32, vp, u64, vp, vp, vp]),
    "pulse_apply": (i32, [vp, u32, u32, vp, vp, u32, vp, vp, vp]),
    "pulse_apply_patch": (i32, [vp, u32, u32, vp, vp, vp, vp, vp, vp]),
    "pulse_flat_carry_from_summaries": (i32, [vp, u32, vp, vp]),
    "pulse_store_to_peers": (i32, [vp, vp, u32, u32, C.c_int, vp]),
    "pulse_peer_allgather": (i32, [vp, vp, u32, u32, u32, vp, vp, C.c_int, vp]),
    "pulse_ipc_open": (i32, [vp, C.c_int, C.POINTER(vp)]),
    "pulse_ipc_close": (i32, [vp, C.c_int]),
    "pulse_decode_indices": (i32, [vp, u32, vp, vp, u32, vp, vp, vp, vp]),
    "pulse_synth_base": (i32, [vp, u64, u64, C.c_double, C.c_double, vp]),
    "pulse_synth_mutate": (i32, [vp, vp, vp, u64, C.c_double, u64, u64, C.POINTER(u64), vp]),
    # host-buffer API
    "pulse_patch_new": (i32, [C.POINTER(vp)]),
    "pulse_patch_free": (None, [vp]),
    "pulse_patch_get_header": (i32, [vp, C.POINTER(PatchHeader)]),
    "pulse_patch_set_header": (i32, [vp, C.POINTER(PatchHeader)]),
    "pulse_patch_num_tensors": (u32, [vp]),
    "pulse_patch_get_tensor": (i32, [vp, u32, C.POINTER(TensorPatchC)]),
    "pulse_patch_add_tensor": (i32, [vp, C.POINTER(TensorPatchC)]),
    "pulse_bytes_data": (vp, [vp]),
    "pulse_bytes_size": (u64, [vp]),
    "pulse_bytes_free": (None, [vp]),
    "pulse_encode": (i32, [C.POINTER(CheckpointC), C.POINTER(CheckpointC), u32, u32, C.POINTER(vp)]),
    "pulse_decode": (i32, [C.POINTER(CheckpointC), vp, C.c_int, C.POINTER(vp), C.POINTER(u64)]),
    "pulse_encode_index_payloads": (i32, [vp, C.POINTER(vp), C.POINTER(u64)]),
    "pulse_decode_index_payloads": (i32, [vp, C.POINTER(vp), C.POINTER(u64), u32]),
    "pulse_write_patch_bytes": (i32, [vp, C.POINTER(vp)]),
    "pulse_read_patch_bytes": (i32, [C.c_char_p, u64, C.POINTER(vp)]),
    "pulse_count_changed": (i32, [vp, u32, u32, vp, vp]),
    "pulse_count_above": (i32, [vp, u32, u32, vp, vp]),
    "pulse_sparsity": (i32, [C.POINTER(CheckpointC), C.POINTER(CheckpointC), u64, C.POINTER(SparsityReportC)]),
    "pulse_frozen_fraction": (i32, [C.POINTER(CheckpointC), C.c_double, C.POINTER(C.c_double)]),
    "pulse_transfer_stats": (None, [C.POINTER(u64), C.POINTER(u64), C.c_int]),
    "pulse_hash_weights": (i32, [C.POINTER(CheckpointC), C.c_char_p]),
    "pulse_sha256_new": (i32, [C.POINTER(vp)]),
    "pulse_sha256_update": (i32, [vp, C.c_char_p, u64]),
    "pulse_sha256_final": (i32, [vp, C.c_char_p]),
    "pulse_sha256_free": (None, [vp]),
    "pulse_delta_encode_indices": (i32, [C.POINTER(C.c_int64), u64, C.POINTER(C.c_int64)]),
    "pulse_delta_decode_indices": (i32, [C.POINTER(C.c_int64), u64, C.POINTER(C.c_int64)]),
    "pulse_downscale_coo": (i32, [C.POINTER(C.c_int64), u64, C.POINTER(C.c_int64), u64, C.POINTER(vp)]),
    "pulse_upscale_coo": (i32, [C.c_char_p, u64, u64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pulse_compress": (i32, [C.c_char_p, u64, u32, C.POINTER(vp)]),
    "pulse_decompress": (i32, [C.c_char_p, u64, u32, C.POINTER(vp)]),
    # PULC container
    "pulse_write_checkpoint_bytes": (i32, [C.POINTER(CheckpointC), C.c_int, C.POINTER(vp)]),
    "pulse_container_parse": (i32, [vp, u64, C.POINTER(vp)]),
    "pulse_container_free": (None, [vp]),
    "pulse_container_step": (u64, [vp]),
    "pulse_container_num_tensors": (u32, [vp]),
    "pulse_container_get_tensor": (i32, [vp, u32, C.POINTER(ContainerTensorC)]),
    "pulse_container_copy_out": (i32, [vp, vp, u64, C.c_int, C.POINTER(vp)]),
    # resident checkpoints (sync path)
    "pulse_resident_create": (i32, [C.POINTER(CheckpointC), u64, C.POINTER(vp)]),
    "pulse_resident_create_device": (i32, [C.POINTER(CheckpointC), u64, C.POINTER(vp)]),
    "pulse_resident_destroy": (None, [vp]),
    "pulse_resident_step": (u64, [vp]),
    "pulse_resident_last_anchor_step": (u64, [vp]),
    "pulse_resident_hash": (i32, [vp, C.c_char_p]),
    "pulse_resident_num_tensors": (u32, [vp]),
    "pulse_resident_tensor": (i32, [vp, u32, C.POINTER(vp)]),
    "pulse_resident_download": (i32, [vp, C.POINTER(vp)]),
    "pulse_resident_apply": (i32, [vp, vp, u64, u64, C.c_char_p, C.c_int]),
    "pulse_resident_walk": (i32, [vp, C.POINTER(vp), C.POINTER(u64), u32, C.c_int, C.POINTER(u32)]),
    "pulse_resident_publish": (i32, [vp, C.POINTER(vp), u64, u32, u32, u64, C.c_int, C.POINTER(vp), C.c_char_p]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def watchdog():
    """None, or the 7 words of a fired device watchdog (kind, block, thread, a, b, c)."""
    out = (C.c_uint64 * 7)()
    if lib.pulse_watchdog(out):
        return list(out)
    return None


def exported_symbols():
    """Names declared by include/pulse_cuda.h that this binding resolves."""
    return sorted(_SIGS)
