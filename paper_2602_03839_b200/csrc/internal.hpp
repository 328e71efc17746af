// Internal interface between the plan/ABI layer (plan.cu) and the kernel
// translation units (encode.cu, decode.cu, synth.cu).
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/pulse_cuda.h"

namespace pulse {
namespace dev {

// K1 tile: 8192 bf16 of each snapshot (16 KiB + 16 KiB) inside one segment.
constexpr uint32_t kTileElems = 8192;
// Segments split tensors so that a compacted u32 index (relative to the
// segment) always fits; tiles never straddle segments (nor tensors).
constexpr uint64_t kSegElems = 1ull << 31;
// K2 / decode chunk: 2048 entries = 256 threads x 8.
constexpr uint32_t kChunkEntries = 2048;
constexpr uint32_t kEntriesPerThread = 8;
// COO_DOWNSCALED parse tiles: 256 threads x 16 bytes.
constexpr uint32_t kParseBytes = 16;
constexpr uint32_t kParseTile = 256 * kParseBytes;

struct SegDesc {
    uint64_t elem_off;     // element offset of the segment inside its tensor
    uint64_t tile_start;   // first global K1 tile id (8192-element tiles)
    uint64_t ticket_start; // first global K1 ticket id (65536-element TMA tickets)
    uint32_t tensor;       // tensor index in the plan
    uint32_t numel;        // elements in the segment (<= 2^31)
};
constexpr uint32_t kTicketElems = 65536;
constexpr uint32_t kK2RangeEntries = 1024;  // K2 warp range (index_code.cu kRangeEntries)

// Division by a tensor's column extent (COO_DOWNSCALED view, patch.hpp:105-109):
// q = (umulhi(n, magic) + n) >> shift for 32-bit n when cols < 2^32.
struct ColDiv {
    uint64_t cols;
    uint32_t cols32, magic, shift, wide;
};

inline ColDiv make_coldiv(uint64_t cols) {
    ColDiv d{};
    d.cols = cols;
    d.wide = cols >= (1ull << 32);
    if (!d.wide) {
        d.cols32 = uint32_t(cols);
        uint32_t l = 0;
        while ((1ull << l) < cols) ++l;  // ceil(log2(cols))
        d.shift = l;
        d.magic = uint32_t(((unsigned __int128)1 << 32) * ((1ull << l) - cols) / cols + 1);
    }
    return d;
}

// Per-tensor encode layout (written by the layout kernel).
struct TensorLayout {
    uint64_t idx_off;     // byte offset of the index payload in the body
    uint64_t val_off;     // byte offset of the value payload in the body
    uint64_t row_bytes;   // COO_DOWNSCALED: bytes of the row stream
    uint64_t rts;         // row escapes before this tensor (global)
    uint64_t cts;         // col escapes before this tensor (global)
    uint64_t gap_base;    // FLAT: numel - last of the previous changed tensor
    uint32_t has_prev;    // FLAT: an earlier index exists in the stream
    uint32_t count_nz;    // tensor has changes
};

// Per-entry decode layout (one per patch entry).
struct EntryLayout {
    uint64_t tensor;      // plan tensor index
    uint64_t count;
    uint64_t idx_off, idx_nbytes, val_off;
    uint64_t es;          // first entry ordinal (exclusive scan of counts)
    uint64_t ck;          // first parse chunk (row grammar)
    uint64_t numel, cols;
    uint64_t flat_base;   // FLAT: sum of numel of earlier patch entries
    uint64_t col_start;   // COO_DS: byte offset (within idx blob) where the col stream starts
    uint64_t cu;          // COO_DS: first col-grammar chunk
};

// Everything the kernels need, as device pointers.
struct PlanDev {
    uint32_t n_tensors, n_segs;
    uint64_t n_tiles, cap;
    const SegDesc* segs;
    const uint32_t* tile_seg;   // [n_tiles] segment of each K1 tile
    uint64_t tma_tiles;         // number of 65536-element tickets
    uint32_t k1_dense;          // K1 staging shape from the capacity: 4 sparse (< 1.5%), 0 sparse (< 2.2%), 1 dense (>= 2.2%), 2 denser (>= 4.5%), 3 (>= 5.6%)
    ulonglong2* k1_defer;       // [tma_tiles] (ticket, output offset) of the tickets K1b writes
    const uint32_t* tma_tile_seg;  // [tma_tiles] segment of each ticket
    uint32_t* trace;            // [tma_tiles] optional K1 progress trace (PULSE_TRACE=1)
    const uint32_t* seg_first;  // [T+1] first segment of each tensor
    const uint64_t* numel;      // [T]
    const uint64_t* cols;       // [T]
    uint16_t* const* slot[PULSE_MAX_SLOTS];  // device arrays of T data pointers

    // encode scratch
    uint32_t* idx32;            // [cap]
    uint16_t* val16;            // [cap]
    uint64_t* seg_start;        // [S+1] entry offset of each segment
    uint64_t* k1_status;        // [n_tiles]
    uint64_t* counters;         // [8] tickets
    pulse_scan_summary* scan;   // device
    const ColDiv* coldiv;       // [T]
    uint64_t* range_cnt;        // [cap/kK2RangeEntries + 2] packed (row | col << 32) escapes per K2 warp range
    ulonglong2* range_pre;      // [cap/kK2RangeEntries + 2] global (row, col) escapes before each range
    uint32_t* t_resc;           // [T]
    uint32_t* t_cesc;           // [T]
    TensorLayout* tlay;         // [T]
    uint64_t* err;              // first-error key
    pulse_result* result;       // device (internal copy)

    // mode-B (host int64 indices) entry map: one segment per tensor
    const SegDesc* id_segs;     // [T]
    const uint32_t* id_first;   // [T+1] = 0..T
    uint64_t* id_start;         // [T+1] entry offsets, uploaded per call

    // decode scratch
    EntryLayout* elay;          // [T]
    uint64_t* d_es;             // [T+1] first entry ordinal of each patch entry
    uint64_t* d_ck;             // [T+1] first row-grammar chunk
    uint64_t* d_cu;             // [T+1] first col-grammar chunk
    uint32_t* rowgap;           // [cap]
    uint32_t* colent;           // [cap]
    uint64_t* flat;             // [cap]
    uint64_t* d_status;         // look-back status words, 4 regions of d_status_len
    uint64_t d_status_len;      // words per region
    uint64_t dec_bytes_cap;     // max index-payload bytes a decode may parse
    uint64_t* d_totals;         // [16] totals + tickets
    uint32_t* d_flags;          // [4] flags[0]: patch needs the general (escape-aware) decoder
};

// ---- launchers (stream-ordered, no host sync) -------------------------------------------
void launch_encode_scan(const PlanDev& p, uint32_t curr_slot, uint32_t prev_slot, pulse_scan_summary* copy_out,
                        cudaStream_t s);
void launch_encode_emit(const PlanDev& p, uint32_t repr, const pulse_scan_summary* gathered,
                        uint32_t n_ranks, uint32_t rank, uint8_t* body, uint64_t body_cap,
                        pulse_patch_entry* entries, pulse_result* result, cudaStream_t s);
void launch_decode(const PlanDev& p, uint32_t repr, const uint8_t* body,
                   const pulse_patch_entry* entries, uint32_t n_entries,
                   const pulse_flat_carry* carry, int weights_slot, int64_t* out_indices,
                   pulse_result* result, cudaStream_t s, const pulse_result* patch_result = nullptr);
void launch_flat_carry(const pulse_scan_summary* gathered, uint32_t rank, pulse_flat_carry* out, cudaStream_t s);
struct PeerPtrs {
    void* p[64];
};
void launch_store_to_peers(const void* src, const PeerPtrs& dst, uint32_t n_dst, uint32_t nbytes, cudaStream_t s);
void launch_peer_allgather(const void* src, const PeerPtrs& tables, const void* my_table, uint32_t world,
                           uint32_t rank, uint32_t nbytes, unsigned long long* epoch, void* out, cudaStream_t s);
// Validate caller-provided int64 indices (decode over an in-memory SparsePatch,
// patch.hpp:325-336) and scatter values into `weights_slot`.
void launch_apply_fast(const PlanDev& p, uint32_t repr, const uint8_t* body, uint32_t n_entries,
                       const pulse_flat_carry* carry, int weights_slot, int64_t* out_indices, uint32_t* flags,
                       cudaStream_t s);
void launch_apply_idx64(const PlanDev& p, const int64_t* idx64, const uint16_t* vals,
                        const pulse_patch_entry* entries, uint32_t n_entries, int weights_slot,
                        pulse_result* result, cudaStream_t s);

// Host-index encode (index coding of caller-provided int64 indices, the
// reference's encode_index_payloads over a host SparsePatch).
void launch_encode_emit_idx64(const PlanDev& p, uint32_t repr, const int64_t* idx64, const uint16_t* vals,
                              uint8_t* body, uint64_t body_cap, pulse_patch_entry* entries,
                              pulse_result* result, cudaStream_t s);

int sm_count();
// Per-device one-time launch configuration: function attributes (the dynamic
// shared-memory opt-in) and occupancy are per device, so caches index by the
// current device.  A race only repeats an idempotent setup.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & (kMaxDevices - 1);
}
struct PerDeviceInt {
    int v[kMaxDevices] = {};
    int& here() { return v[current_device()]; }
};
// PULSE_DEBUG_SYNC=1: synchronise after every launch and report the first
// failing kernel by name on stderr (debugging aid; off by default).
void debug_sync(const char* kernel, cudaStream_t s);
// gate.cu: `body` (launches on the stream it is given) runs only if *flag != 0
// when the stream gets there -- a conditional graph node under stream capture.
void launch_gated(cudaStream_t s, const uint32_t* flag, const std::function<void(cudaStream_t)>& body);
// ... only if a first-error key has been recorded (*err_key != kNoError).
void launch_gated_on_error(cudaStream_t s, const uint64_t* err_key, const std::function<void(cudaStream_t)>& body);
#define PULSE_LAUNCHED(name, stream) ::pulse::dev::debug_sync(name, stream)
// helpers.cu (host-buffer API support)
void launch_export_indices(const PlanDev& p, int64_t* out, cudaStream_t s);
void launch_gather_values(const PlanDev& p, int slot, const pulse_patch_entry* ents, const uint64_t* start,
                          uint32_t n_e, const int64_t* idx, uint16_t* out, cudaStream_t s);
void launch_delta_encode(const int64_t* in, uint64_t n, int64_t* out, uint64_t* err, cudaStream_t s);
void launch_delta_decode(const int64_t* in, uint64_t n, int64_t* out, uint64_t* err, cudaStream_t s);
void launch_coo_pack(const int64_t* rows, const int64_t* cols, uint64_t n, uint8_t* out, uint64_t* nbytes,
                     uint64_t* err, cudaStream_t s);
void launch_coo_unpack_par(const PlanDev& p, const uint8_t* body, const pulse_patch_entry* entry, int64_t* rows,
                           int64_t* cols, pulse_result* result, cudaStream_t s);
void set_watchdog_helpers(unsigned long long* slot);
void set_watchdog_encode(unsigned long long* slot);
void set_watchdog_decode(unsigned long long* slot);
void set_watchdog_synth(unsigned long long* slot);
void set_watchdog_index(unsigned long long* slot);
void set_watchdog_apply(unsigned long long* slot);
void set_watchdog_reduce(unsigned long long* slot);
// reduce.cu (absorption.hpp analyses)
void launch_count_changed(const PlanDev& p, uint32_t slot_a, uint32_t slot_b, uint64_t* out, cudaStream_t s);
void launch_count_above(const PlanDev& p, uint32_t slot, uint32_t magnitude_bits, uint64_t* out, cudaStream_t s);

}  // namespace dev
}  // namespace pulse
