/*
 * pulse_cuda.h -- C ABI of libpulse_cuda.so, the B200-native PULSE hot path.
 *
 * The reference (arxiv 2602.03839, /root/reference/proj/include/pulse) is a
 * header-only C++20 library with no FFI; its drop-in surface for this path is
 * the set of functions in patch.hpp, index_coding.hpp, patch_file.hpp,
 * compression.hpp and sha256.hpp.  This header is the C boundary those
 * functions are re-expressed over: plain pointers, sizes and status codes, no
 * C++ or torch types.  The headers in include/pulse/ re-create the reference's C++ API
 * on top of it, and paper_2602_03839_b200/_native.py binds it with ctypes.
 *
 * Two families of entry points:
 *   pulse_encode / pulse_decode / pulse_*_payloads / pulse_*_patch_bytes ...
 *       host-buffer calls that mirror the reference functions one for one
 *       (the reference interface each replaces is cited on the declaration);
 *       inputs are staged to the GPU, every per-element step runs in CUDA.
 *   pulse_plan_* / pulse_encode_scan / pulse_encode_emit / pulse_apply ...
 *       device-resident calls over snapshots already in HBM, asynchronous on
 *       a caller-supplied cudaStream_t (passed as void*).  These are what the
 *       throughput numbers measure and what the multi-GPU driver shards.
 *
 * Errors: every function returns a pulse_status; the numbering maps one to one
 * onto the reference exception classes (error.hpp:10-115).  No exception
 * crosses the ABI.  pulse_last_error() returns the thread-local message of the
 * last failing call on the calling thread.
 */
#ifndef PULSE_CUDA_H
#define PULSE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pulse_status {
    PULSE_OK = 0,
    PULSE_E_ERROR = 1,           /* pulse::Error                 error.hpp:10  */
    PULSE_E_ARGUMENT = 2,        /* pulse::ArgumentError         error.hpp:16  */
    PULSE_E_FORMAT = 3,          /* pulse::FormatError           error.hpp:22  */
    PULSE_E_BAD_MAGIC = 4,       /* pulse::BadMagicError         error.hpp:27  */
    PULSE_E_VERSION = 5,         /* pulse::VersionError          error.hpp:32  */
    PULSE_E_TRUNCATION = 6,      /* pulse::TruncationError       error.hpp:37  */
    PULSE_E_CORRUPT_STREAM = 7,  /* pulse::CorruptStreamError    error.hpp:42  */
    PULSE_E_MODEL_MISMATCH = 8,  /* pulse::ModelMismatchError    error.hpp:49  */
    PULSE_E_SHAPE_MISMATCH = 9,  /* pulse::ShapeMismatchError    error.hpp:54  */
    PULSE_E_TENSOR_SET = 10,     /* pulse::TensorSetError        error.hpp:59  */
    PULSE_E_INDEX_RANGE = 11,    /* pulse::IndexRangeError       error.hpp:64  */
    PULSE_E_DIMENSION = 12,      /* pulse::DimensionError        error.hpp:71  */
    PULSE_E_HASH_MISMATCH = 13,  /* pulse::HashMismatchError     error.hpp:77  */
    PULSE_E_CUDA = 14,           /* device/runtime failure (no reference analogue) */
    PULSE_E_CAPACITY = 15,       /* caller arena too small; see `required` */
    PULSE_E_PROTOCOL = 16        /* pulse::ProtocolViolationError error.hpp:112 */
} pulse_status;

/* SparseRepresentation (patch.hpp:20-24) and CodecId (compression.hpp:31-37). */
enum { PULSE_COO_DOWNSCALED = 0, PULSE_COO_INT32 = 1, PULSE_FLAT_INT32 = 2 };
enum { PULSE_IDENTITY = 0, PULSE_LZ4 = 1, PULSE_ZSTD1 = 2, PULSE_ZSTD3 = 3, PULSE_GZIP6 = 4 };

const char* pulse_last_error(void);
const char* pulse_version(void);

/* Device spin-wait watchdog: returns 1 (and clears it) if some kernel gave up
 * a wait after the spin limit; out7 = {fired, kind, block, thread, a, b, c}.
 * A fired watchdog means the results of that launch are invalid. */
int pulse_watchdog(uint64_t* out7);

/* ======================================================================= */
/* Device-resident API                                                      */
/* ======================================================================= */

typedef struct pulse_context pulse_context;
typedef struct pulse_plan pulse_plan;

/* One context per device; callable from one host thread per GPU. */
pulse_status pulse_context_create(int device, pulse_context** out);
void pulse_context_destroy(pulse_context* ctx);

/* Geometry of one tensor of a name-sorted state dict (checkpoint.hpp:18-28). */
typedef struct pulse_tensor_geom {
    uint64_t numel; /* elements, > 0 */
    uint64_t cols;  /* shape.back(): COO_DOWNSCALED column extent (patch.hpp:105-109) */
} pulse_tensor_geom;

/* A plan fixes the tensor table (in ascending name order, the PULP order,
 * patch_file.hpp:34-35) and owns the device scratch for up to `max_changes`
 * changed elements per encode/apply.  Tensors may exceed 2^32 elements. */
pulse_status pulse_plan_create(pulse_context* ctx, const pulse_tensor_geom* tensors,
                               uint32_t n_tensors, uint64_t max_changes, pulse_plan** out);
void pulse_plan_destroy(pulse_plan* plan);

/* Binds one device pointer per tensor (bf16 data, 16-byte aligned) to slot
 * 0..3.  Encode reads two slots; apply writes one. */
enum { PULSE_MAX_SLOTS = 4 };
pulse_status pulse_plan_bind(pulse_plan* plan, uint32_t slot, const void* const* dev_ptrs);

/* FLAT_INT32 threads one gap stream across tensors (patch.hpp:131-156); when a
 * state dict is sharded across ranks, each rank's stream continues from the
 * previous rank's last emitted index.  gap_base = numel(last changed tensor)
 * - last index in it; the first entry of the next shard is idx + gap_base. */
typedef struct pulse_flat_carry {
    uint64_t has_prev;
    uint64_t gap_base;
} pulse_flat_carry;

/* Per-shard summary after the diff scan; all-gathered across ranks so each
 * rank can place its section and continue the FLAT stream. */
typedef struct pulse_scan_summary {
    uint64_t n_changes;
    uint64_t has_change;
    uint64_t last_gap_base; /* numel - last index of this shard's last changed tensor */
    uint64_t status;        /* 0 or PULSE_E_CAPACITY */
} pulse_scan_summary;

/* One entry per changed tensor, in name order -- the device image of the PULP
 * per-tensor header record (patch_file.hpp:63-71) and its two blobs. */
typedef struct pulse_patch_entry {
    uint32_t tensor; /* plan tensor index */
    uint32_t reserved;
    uint64_t count;      /* changed elements = values */
    uint64_t idx_off;    /* byte offset of the raw index payload in the body */
    uint64_t idx_nbytes; /* patch.hpp:116-174 payload length */
    uint64_t val_off;    /* byte offset of the u16 LE value payload (2*count B) */
} pulse_patch_entry;

/* The reference check behind a failure (ordered as the reference evaluates
 * them); lets the host rebuild the reference's exception message. */
enum {
    PULSE_CHECK_TRUNCATED = 1,     /* wire.hpp:58-60 */
    PULSE_CHECK_ZERO_GAP = 2,      /* patch.hpp:201-203, 225-227 */
    PULSE_CHECK_ZERO_COL_GAP = 3,  /* index_coding.hpp:147-149 */
    PULSE_CHECK_COL_RANGE = 4,     /* patch.hpp:247-250 */
    PULSE_CHECK_INDEX_RANGE = 5,   /* patch.hpp:206-208, 231-233, 252-254 */
    PULSE_CHECK_TRAILING = 6,      /* patch.hpp:211-213, index_coding.hpp:154-156 */
    PULSE_CHECK_NEGATIVE = 7,      /* index_coding.hpp:19-21, 118 */
    PULSE_CHECK_ORDER = 8,         /* index_coding.hpp:22-24, 119-121; patch.hpp:142-144 */
    PULSE_CHECK_FLAT_GAP = 9,      /* patch.hpp:145-147 */
    PULSE_CHECK_ROW_GAP = 10,      /* index_coding.hpp:69-71 */
    PULSE_CHECK_COL_ENTRY = 11,    /* index_coding.hpp:80-82 */
    PULSE_CHECK_INT32 = 12,        /* patch.hpp:99-103 */
    PULSE_CHECK_APPLY_ORDER = 13,  /* patch.hpp:329-332 */
    PULSE_CHECK_APPLY_RANGE = 14,  /* patch.hpp:333-336 */
    PULSE_CHECK_CAPACITY = 15
};

typedef struct pulse_result {
    uint64_t n_changes;
    uint64_t body_bytes; /* encode: bytes written to the body */
    uint32_t n_entries;  /* encode: changed tensors */
    int32_t status;      /* pulse_status of the device pipeline */
    uint32_t err_check;  /* which reference check failed first (PULSE_CHECK_*) */
    uint32_t err_stage;
    uint64_t err_tensor; /* plan tensor (encode) / patch entry (apply) of the first failure */
    uint64_t err_elem;   /* element / entry ordinal of the first failure */
    uint64_t required;   /* bytes or changes needed when status == PULSE_E_CAPACITY */
    pulse_flat_carry carry_out;
} pulse_result;

/* K1: bitwise diff of slot `curr_slot` against `prev_slot` and ordered
 * compaction (decoupled look-back) of every changed element -- the loop at
 * patch.hpp:296-301.  Writes the plan's scan summary and, when
 * `dev_summary_out` is non-NULL, a copy of it there (e.g. straight into an
 * NCCL all-gather send buffer). */
pulse_status pulse_encode_scan(pulse_plan* plan, uint32_t curr_slot, uint32_t prev_slot,
                               pulse_scan_summary* dev_summary_out, void* stream);
/* Device pointer to the plan's pulse_scan_summary (for NCCL all-gather). */
pulse_scan_summary* pulse_plan_scan_summary(pulse_plan* plan);
/* Debug: K1 per-ticket progress trace (device, NULL unless PULSE_TRACE is set). */
uint32_t* pulse_plan_trace(pulse_plan* plan, uint64_t* n);

/* K2: index coding (patch.hpp:116-174, index_coding.hpp:14-128) and the PULP
 * body layout: for each changed tensor, [index payload][value payload]
 * concatenated in name order (the identity-codec blob area of
 * patch_file.hpp:76-82).  `gathered`/`n_ranks`/`rank` (device array of all
 * ranks' scan summaries) continue a sharded FLAT_INT32 stream and offset the
 * section; pass NULL/1/0 on one GPU.  Writes `dev_entries[n_tensors]`,
 * `dev_result`. */
pulse_status pulse_encode_emit(pulse_plan* plan, uint32_t representation,
                               const pulse_scan_summary* gathered, uint32_t n_ranks,
                               uint32_t rank, uint8_t* dev_body, uint64_t body_capacity,
                               pulse_patch_entry* dev_entries, pulse_result* dev_result,
                               void* stream);

/* Apply a device-resident patch body in place to slot `weights_slot`:
 * parse + validate every entry first (patch.hpp:178-262, 325-336), then
 * scatter (patch.hpp:337) only if nothing failed, so a bad patch never
 * half-applies.  `carry` continues a sharded FLAT_INT32 stream (NULL on one
 * GPU).  Writes `dev_result`. */
pulse_status pulse_apply(pulse_plan* plan, uint32_t weights_slot, uint32_t representation,
                         const uint8_t* dev_body, const pulse_patch_entry* dev_entries,
                         uint32_t n_entries, const pulse_flat_carry* dev_carry,
                         pulse_result* dev_result, void* stream);

/* pulse_apply with the entry count taken from the encode's device result
 * (`dev_patch_result`, as written by pulse_encode_emit) instead of the host:
 * a sharded encode -> apply step then needs no host round trip.  If the
 * encode failed (status != 0) nothing is applied and its error is reported
 * in `dev_result`. */
pulse_status pulse_apply_patch(pulse_plan* plan, uint32_t weights_slot, uint32_t representation,
                               const uint8_t* dev_body, const pulse_patch_entry* dev_entries,
                               const pulse_result* dev_patch_result, const pulse_flat_carry* dev_carry,
                               pulse_result* dev_result, void* stream);

/* Device-side FLAT_INT32 carry of shard `rank` from the all-gathered scan
 * summaries of every rank (the nearest earlier rank that emitted an index). */
pulse_status pulse_flat_carry_from_summaries(const pulse_scan_summary* dev_gathered, uint32_t rank,
                                             pulse_flat_carry* dev_out, void* stream);

/* Stores `nbytes` (<= 256) device bytes from `dev_src` at each of the `n_dst` (<= 64)
 * device addresses in the host array `dsts`, from one kernel on `stream` (a stream of
 * `device`, which gets peer access to every device it can reach on first use; call it
 * once outside stream capture before capturing it):
 * with peer-mapped destinations (CUDA IPC, NVLink) this is a one-sided exchange of small
 * per-step tables between ranks -- the sharded driver's (body bytes, entries, status)
 * table -- without a collective. Ordering for the readers is the caller's (e.g. device
 * synchronize + barrier before reading). */
pulse_status pulse_store_to_peers(const void* dev_src, void* const* dsts, uint32_t n_dst, uint32_t nbytes,
                                  int device, void* stream);

/* All-gather of one `nbytes` (<= 48) record per rank through peer-mapped tables, inside a
 * stream / CUDA graph (no collective): `tables[r]` is rank r's table of 2 x world 64-byte
 * slots (zeroed once; tables[rank] is this rank's own), `dev_epoch` a device u64 (zeroed
 * once) that every rank advances once per call. The record goes to this rank's slot in
 * every table tagged with the new epoch; the call then waits on the device until all
 * ranks' slots carry it and copies the records to `dev_out` (world x nbytes, rank order).
 * Slots alternate with the epoch's parity, so a rank one call ahead never overwrites a
 * record its peers have not read. Every rank must make the same sequence of calls. */
pulse_status pulse_peer_allgather(const void* dev_src, void* const* tables, uint32_t world, uint32_t rank,
                                  uint32_t nbytes, uint64_t* dev_epoch, void* dev_out, int device, void* stream);

/* Maps another process's device allocation (a 64-byte cudaIpcMemHandle_t, e.g. from torch's
 * storage sharing) into the context of `device` in this process, with peer access enabled,
 * so kernels on `device` can load / store it over NVLink; pulse_ipc_close unmaps it. */
pulse_status pulse_ipc_open(const void* ipc_handle, int device, void** dev_ptr);
pulse_status pulse_ipc_close(void* dev_ptr, int device);

/* Analyses (absorption.hpp:38-78) on bound snapshots, one HBM pass each:
 * elements whose bit patterns differ between two slots (the count behind
 * sparsity(), :55-78), and elements whose bf16 magnitude pattern (bits &
 * 0x7FFF) is above `magnitude_bits` and not NaN (frozen_fraction(), :38-46;
 * the host maps the threshold to the largest magnitude pattern <= it).
 * `dev_count` is one device uint64. */
pulse_status pulse_count_changed(pulse_plan* plan, uint32_t slot_a, uint32_t slot_b, uint64_t* dev_count,
                                 void* stream);
pulse_status pulse_count_above(pulse_plan* plan, uint32_t slot, uint32_t magnitude_bits, uint64_t* dev_count,
                               void* stream);

/* Decode only: parse the payloads to flat int64 indices (dev_indices, in
 * entry order) without touching weights. */
pulse_status pulse_decode_indices(pulse_plan* plan, uint32_t representation,
                                  const uint8_t* dev_body, const pulse_patch_entry* dev_entries,
                                  uint32_t n_entries, const pulse_flat_carry* dev_carry,
                                  int64_t* dev_indices, pulse_result* dev_result, void* stream);

/* Synthetic snapshots on device (fixture; the reference generator's knobs,
 * synthetic.hpp:21-28,62-107): log-normal |w| (median, sigma), random sign,
 * then exactly llround((1-sparsity)*n) changed positions in half-density
 * windows of `cluster_width`, each an LSB flip.  Counter-based RNG, so the
 * bytes are a function of (seed, n) only. */
pulse_status pulse_synth_base(uint16_t* dev_out, uint64_t n, uint64_t seed, double median,
                              double sigma, void* stream);
pulse_status pulse_synth_mutate(pulse_context* ctx, const uint16_t* dev_base, uint16_t* dev_out,
                                uint64_t n, double sparsity, uint64_t cluster_width,
                                uint64_t seed, uint64_t* changed_out, void* stream);

/* ======================================================================= */
/* Host-buffer API: the reference's functions over host memory              */
/* ======================================================================= */

/* One named bf16 tensor, row-major (checkpoint.hpp:18-28 TensorRecord). */
typedef struct pulse_tensor {
    const char* name;     /* NUL-terminated */
    const int64_t* shape;
    uint32_t rank;
    const uint16_t* data; /* numel bf16 bit patterns */
    uint64_t numel;       /* data length; validated against shape */
} pulse_tensor;

/* A snapshot at one optimizer step (checkpoint.hpp:32-71 Checkpoint). */
typedef struct pulse_checkpoint {
    uint64_t step;
    const pulse_tensor* tensors;
    uint32_t n_tensors;
} pulse_checkpoint;

/* SparsePatch (patch.hpp:54-70), library-owned. */
typedef struct pulse_patch pulse_patch;
typedef struct pulse_patch_header {
    int64_t base_step, target_step, anchor_step;
    uint32_t representation, codec;
    uint8_t target_hash[32];
} pulse_patch_header;
/* TensorPatch view (patch.hpp:45-52); pointers stay valid until the patch is freed. */
typedef struct pulse_tensor_patch {
    const char* name;
    const int64_t* shape;
    uint32_t rank;
    const int64_t* indices;
    uint64_t n_indices;
    const uint16_t* values;
    uint64_t n_values;
} pulse_tensor_patch;

pulse_status pulse_patch_new(pulse_patch** out);
void pulse_patch_free(pulse_patch* patch);
pulse_status pulse_patch_get_header(const pulse_patch* patch, pulse_patch_header* out);
pulse_status pulse_patch_set_header(pulse_patch* patch, const pulse_patch_header* header);
uint32_t pulse_patch_num_tensors(const pulse_patch* patch);
pulse_status pulse_patch_get_tensor(const pulse_patch* patch, uint32_t i, pulse_tensor_patch* out);
pulse_status pulse_patch_add_tensor(pulse_patch* patch, const pulse_tensor_patch* tensor); /* copies */

/* Library-owned byte buffer (the reference's Bytes, wire.hpp:15). */
typedef struct pulse_bytes pulse_bytes;
const uint8_t* pulse_bytes_data(const pulse_bytes* b);
uint64_t pulse_bytes_size(const pulse_bytes* b);
void pulse_bytes_free(pulse_bytes* b);

/* encode(current, previous, repr, codec) -- patch.hpp:264-307.  Bitwise diff
 * and compaction on the GPU (K1); target_hash = SHA-256 of `current`
 * (sha256.hpp:93-116) on a host thread in parallel. */
pulse_status pulse_encode(const pulse_checkpoint* current, const pulse_checkpoint* previous,
                          uint32_t representation, uint32_t codec, pulse_patch** out);

/* decode(previous, patch, verify_hash) -- patch.hpp:309-348.  The result has
 * previous's tensors (same order, same shapes); out_data[i] receives tensor i's
 * numel values.  Validation precedes any scatter (IndexRangeError etc.). */
pulse_status pulse_decode(const pulse_checkpoint* previous, const pulse_patch* patch, int verify_hash,
                          uint16_t* const* out_data, uint64_t* out_step);

/* encode_index_payloads -- patch.hpp:116-174.  All payloads concatenated in
 * patch order; sizes[i] = payload i's length (array of num_tensors). */
pulse_status pulse_encode_index_payloads(const pulse_patch* patch, pulse_bytes** concat, uint64_t* sizes);

/* decode_index_payloads -- patch.hpp:178-262.  Fills each tensor's indices;
 * each tensor's count is its number of values. */
pulse_status pulse_decode_index_payloads(pulse_patch* patch, const uint8_t* const* payloads,
                                         const uint64_t* sizes, uint32_t n_payloads);

/* write_patch_bytes / read_patch_bytes -- patch_file.hpp:30-83 / 85-147. */
pulse_status pulse_write_patch_bytes(const pulse_patch* patch, pulse_bytes** out);
pulse_status pulse_read_patch_bytes(const uint8_t* data, uint64_t n, pulse_patch** out);

/* Bytes the host-buffer API has copied host->device and device->host in this
 * process (all threads); a benchmark/diagnostic aid with no reference
 * counterpart.  reset != 0 zeroes the counters after reading them. */
void pulse_transfer_stats(uint64_t* h2d_bytes, uint64_t* d2h_bytes, int reset);

/* sparsity -- absorption.hpp:55-78 (k is metadata, as in the reference). */
typedef struct pulse_sparsity_report {
    uint64_t k;
    uint64_t changed;
    uint64_t total;
    double sparsity; /* 1 - changed / total; 1.0 when total == 0 */
} pulse_sparsity_report;
pulse_status pulse_sparsity(const pulse_checkpoint* a, const pulse_checkpoint* b, uint64_t k,
                            pulse_sparsity_report* out);
/* frozen_fraction -- absorption.hpp:38-46: fraction of weights with |w| > threshold. */
pulse_status pulse_frozen_fraction(const pulse_checkpoint* checkpoint, double threshold, double* out);

/* hash_weights -- sha256.hpp:93-116; Sha256 -- sha256.hpp:51-87. */
pulse_status pulse_hash_weights(const pulse_checkpoint* checkpoint, uint8_t* out32);
typedef struct pulse_sha256_ctx pulse_sha256_ctx;
pulse_status pulse_sha256_new(pulse_sha256_ctx** out);
pulse_status pulse_sha256_update(pulse_sha256_ctx* ctx, const uint8_t* data, uint64_t n);
pulse_status pulse_sha256_final(pulse_sha256_ctx* ctx, uint8_t* out32);
void pulse_sha256_free(pulse_sha256_ctx* ctx);

/* Index helpers -- index_coding.hpp:14-50 (delta) and 108-158 (COO downscale). */
pulse_status pulse_delta_encode_indices(const int64_t* indices, uint64_t n, int64_t* gaps_out);
pulse_status pulse_delta_decode_indices(const int64_t* gaps, uint64_t n, int64_t* indices_out);
pulse_status pulse_downscale_coo(const int64_t* rows, uint64_t n_rows, const int64_t* cols, uint64_t n_cols,
                                 pulse_bytes** out);
pulse_status pulse_upscale_coo(const uint8_t* payload, uint64_t n, uint64_t count, int64_t* rows_out,
                               int64_t* cols_out);

/* Codec envelope -- compression.hpp:119-204 (host libzstd / liblz4 / zlib). */
pulse_status pulse_compress(const uint8_t* raw, uint64_t n, uint32_t codec, pulse_bytes** out);
pulse_status pulse_decompress(const uint8_t* enveloped, uint64_t n, uint32_t codec, pulse_bytes** out);

/* ======================================================================= */
/* PULC checkpoint container -- container.hpp:18-150                        */
/* ======================================================================= */

/* write_checkpoint_bytes -- container.hpp:58-90: "PULC", u32 1, u64 header
 * length, JSON tensor table (sorted keys), then every tensor's LE bf16 payload
 * at a 64-byte aligned offset from the 64-byte aligned payload base, tensors in
 * insertion order.  device_data != 0: the tensors' `data` pointers are DEVICE
 * pointers of the current device, and each payload is copied straight out of
 * HBM into its place in the file (no host Checkpoint in between). */
pulse_status pulse_write_checkpoint_bytes(const pulse_checkpoint* checkpoint, int device_data, pulse_bytes** out);

/* read_checkpoint_bytes -- container.hpp:92-142, in two steps: parse (the
 * header, every payload bound and Checkpoint::validate, with the reference's
 * checks, order and exception classes), then copy the payloads out to host or
 * device memory.  The parsed table refers to the caller's bytes by offset. */
typedef struct pulse_container pulse_container;
typedef struct pulse_container_tensor {
    const char* name;
    const int64_t* shape;
    uint32_t rank;
    uint64_t numel;
    uint64_t payload_offset; /* absolute byte offset of the LE bf16 payload in the container */
} pulse_container_tensor;
pulse_status pulse_container_parse(const uint8_t* data, uint64_t n, pulse_container** out);
void pulse_container_free(pulse_container* container);
uint64_t pulse_container_step(const pulse_container* container);
uint32_t pulse_container_num_tensors(const pulse_container* container);
pulse_status pulse_container_get_tensor(const pulse_container* container, uint32_t i, pulse_container_tensor* out);
/* Copies tensor i's payload (numel * 2 bytes) from `data` -- the bytes that
 * were parsed, `n` long -- to dst[i]: host memory (device == 0) or device
 * memory of the current device (device != 0; DMA straight from `data` when it
 * is page-locked, else through pinned staging).  Returns when the copies are
 * complete. */
pulse_status pulse_container_copy_out(const pulse_container* container, const uint8_t* data, uint64_t n,
                                      int device, void* const* dst);

/* ======================================================================= */
/* Resident checkpoints: the sync path on device (sync.hpp:78-92, 166-211, */
/* 308-352)                                                                */
/* ======================================================================= */

/* A checkpoint held in HBM of the current device, with its step and weights
 * hash -- the consumer's SyncState (sync.hpp:78-92) and the publisher's last
 * published snapshot.  PULP patches are applied to it in place straight from
 * their blobs (no int64 index round trip), and new patches are encoded from
 * it against device-resident weights and written straight from the device
 * body, hashing the target once (sync.hpp:176 and patch.hpp:282 hash it
 * twice). */
typedef struct pulse_resident pulse_resident;

/* checkpoint_to_state: uploads `checkpoint` (validated; host data) and hashes
 * it.  `max_changes` sizes the device scratch (grown on demand). */
pulse_status pulse_resident_create(const pulse_checkpoint* checkpoint, uint64_t max_changes, pulse_resident** out);
/* The same from a checkpoint already in HBM: `checkpoint` gives names, shapes
 * and step, its `data` pointers are device pointers of the current device
 * (copied device to device; the hash is taken from HBM).  The call first waits
 * for all work already queued on the device (cudaDeviceSynchronize), so writes
 * to those buffers pending on any caller stream complete before they are read. */
pulse_status pulse_resident_create_device(const pulse_checkpoint* checkpoint, uint64_t max_changes,
                                          pulse_resident** out);
void pulse_resident_destroy(pulse_resident* r);
uint64_t pulse_resident_step(const pulse_resident* r);
uint64_t pulse_resident_last_anchor_step(const pulse_resident* r);
pulse_status pulse_resident_hash(const pulse_resident* r, uint8_t* out32);
uint32_t pulse_resident_num_tensors(const pulse_resident* r);
/* Device pointer of tensor i (the checkpoint's insertion order). */
pulse_status pulse_resident_tensor(const pulse_resident* r, uint32_t i, void** dev_ptr);
/* Copies every tensor to host memory out[i] (numel values each). */
pulse_status pulse_resident_download(const pulse_resident* r, uint16_t* const* out);

/* apply_delta (sync.hpp:308-329) for the PULP bytes of the delta to `step`:
 * patch.base_step must equal the held step and patch.target_step `step`, and
 * patch.target_hash `expected_hash32` when non-NULL (the manifest's weights
 * hash) -- else PULSE_E_PROTOCOL; tensor names / shapes as decode checks them
 * (patch.hpp:314-324); then validate-then-scatter in place.  verify_hash != 0
 * re-hashes the result (decode's check, patch.hpp:341-346) and on a mismatch
 * puts the overwritten values back before failing with HashMismatchError, so
 * a failed apply never changes the held state. */
pulse_status pulse_resident_apply(pulse_resident* r, const uint8_t* pulp, uint64_t n, uint64_t step,
                                  const uint8_t* expected_hash32, int verify_hash);
/* walk_deltas (sync.hpp:331-352): the deltas to steps held+1 .. held+k, in
 * order; the next patch is parsed and uploaded while the current one applies.
 * Returns the number applied in *applied (stops at the first failure). */
pulse_status pulse_resident_walk(pulse_resident* r, const uint8_t* const* pulps, const uint64_t* sizes, uint32_t k,
                                 int verify_hash, uint32_t* applied);
/* publish_checkpoint's patch (sync.hpp:166-181): `dev_current` (device
 * pointers, insertion order, same tensors as the held checkpoint) at step
 * held+1 is encoded against the held weights on the device; the PULP bytes
 * come straight from the device body (codec on host threads) with
 * anchor_step as given; the target hash (sha256 of dev_current, computed
 * once) goes to out_hash32.  advance != 0 then applies the patch to the held
 * weights, so the resident becomes the new last-published snapshot.  Like
 * create_device, it waits for all queued device work before reading
 * `dev_current`, so a snapshot still being written on another stream is
 * never encoded or hashed half-updated. */
pulse_status pulse_resident_publish(pulse_resident* r, const void* const* dev_current, uint64_t step,
                                    uint32_t representation, uint32_t codec, uint64_t anchor_step, int advance,
                                    pulse_bytes** out_pulp, uint8_t* out_hash32);

#ifdef __cplusplus
}
#endif

#endif /* PULSE_CUDA_H */
