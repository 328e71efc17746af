// PULSE decode / apply on sm_100a.
//
// Input: a device-resident patch body (per changed tensor [index payload]
// [value payload], the identity-codec PULP blob area, patch_file.hpp:76-82)
// and its entry table.  Output: flat indices (decode_index_payloads,
// patch.hpp:178-262) and, for apply, the values scattered in place into the
// resident weights (patch.hpp:337) -- but only after every entry validated,
// so a corrupt patch never half-applies (the reference validates on a copy,
// patch.hpp:311).
//
//   D0 d_layout      one CTA: entry offsets, parse-chunk offsets, FLAT bases,
//                    size checks that need no parsing.
//   D1 d_fixed       COO_INT32 / FLAT_INT32: u32 gaps -> (segmented) prefix
//                    sum via decoupled look-back -> flat indices + checks.
//   D2 d_rows        COO_DOWNSCALED row stream (u8, 0xFF + u32 escapes):
//                    parallel parse.  A byte position p is an entry boundary
//                    whenever none of bytes p-4..p-1 is 0xFF (an escape marker
//                    can only sit there), so every 16-byte chunk resynchronises
//                    locally and entry ordinals come from a segmented count
//                    scan (index_coding.hpp:136-139).  Finds where the column
//                    stream starts (after `count` row entries).
//   D3 d_col_layout  one CTA: column-stream chunk offsets.
//   D4 d_cols        column stream (u16, 0xFFFF + u32 escapes), same scheme in
//                    2-byte units; truncation / trailing-byte checks.
//   D5 d_assemble    rows = segmented sum of row gaps; cols = sum segmented at
//                    new rows (index_coding.hpp:141-153); flat = row*cols+col
//                    (patch.hpp:251) + range checks.
//   D6 d_scatter     W[flat] = value for every entry if no check failed.
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"

namespace pulse {
namespace dev {

namespace {

enum Totals : int {
    kTotEntries = 0,   // sum of counts
    kTotRowChunks = 1, // row-grammar chunks
    kTotColChunks = 2, // col-grammar chunks
    kTicket0 = 8,      // tickets 8..12
};

constexpr uint32_t kParseChunksPerTile = kThreads;  // one 16-byte chunk per thread
constexpr uint32_t kNoPayload = 0xFF;  // d_layout "representation" for int64-index applies

__device__ __forceinline__ uint64_t take_ticket(uint64_t* totals, int which) {
    return atomicAdd(reinterpret_cast<unsigned long long*>(totals + kTicket0 + which), 1ull);
}

// Entry walk for decode: calls f(i, e, o) for entries [i0, i1) where e is the
// patch entry and o the ordinal inside it.
template <class F>
__device__ __forceinline__ void walk(const uint64_t* es, uint32_t n_e, uint64_t i0, uint64_t i1, F&& f) {
    if (i0 >= i1) return;
    uint32_t e = upper_index<uint64_t>(es, 0, n_e, i0);
    for (uint64_t i = i0; i < i1; ++i) {
        while (es[e + 1] <= i) ++e;
        f(i, e, i - es[e]);
    }
}

}  // namespace

// =============================================================================================
// D0: layout
// =============================================================================================
constexpr int kLT = 1024;

__global__ void __launch_bounds__(kLT, 1)
d_layout(const pulse_patch_entry* __restrict__ entries, uint32_t n_e, const uint64_t* __restrict__ numel,
         const uint64_t* __restrict__ cols, uint32_t repr, EntryLayout* __restrict__ el,
         uint64_t* __restrict__ es, uint64_t* __restrict__ ck, uint64_t* __restrict__ totals,
         uint64_t* __restrict__ err, uint32_t* __restrict__ flags, uint64_t cap,
         const pulse_result* __restrict__ patch_result) {
    __shared__ uint64_t s_tmp[33 * 3];
    // per-call state (totals and tickets, flags, first-error key), zeroed here rather
    // than by three memset nodes ahead of this 1-CTA kernel
    if (threadIdx.x < 16) totals[threadIdx.x] = 0;
    if (threadIdx.x < 4) flags[threadIdx.x] = 0;
    if (threadIdx.x == 0) *err = kNoError;
    __syncthreads();
    // With `patch_result` (the encode's device result) the entry count comes from
    // the device and a failed encode applies nothing: entries past the count are
    // empty, and the encode's own first error becomes this call's error.
    uint32_t n_live = n_e;
    if (patch_result) {
        const pulse_result pr = *patch_result;
        n_live = pr.status != 0 ? 0u : min(pr.n_entries, n_e);
        if (pr.status != 0 && threadIdx.x == 0)
            report(err, error_key(uint32_t(pr.err_tensor), pr.err_stage, pr.err_elem,
                                  pr.err_check ? pr.err_check : uint32_t(kCapacity)));
    }
    uint64_t base_e = 0, base_c = 0, base_f = 0;
    for (uint32_t e0 = 0; e0 < n_e; e0 += kLT) {
        const uint32_t e = e0 + threadIdx.x;
        const bool v = e < n_live;
        pulse_patch_entry pe{};
        if (v) pe = entries[e];
        const uint64_t ne = v ? numel[pe.tensor] : 0;
        const uint64_t nchunks = v ? (pe.idx_nbytes + kParseBytes - 1) / kParseBytes : 0;
        uint64_t sc[3] = {v ? pe.count : 0, nchunks, ne}, tot[3];
        cta_exclusive_scan<3, kLT, AllSum>(sc, tot, s_tmp);
        const uint64_t xe = sc[0], xc = sc[1], xf = sc[2];
        const uint64_t te = tot[0], tc = tot[1], tf = tot[2];
        if (!v && e < n_e) {  // empty entry (past the device-side count)
            EntryLayout L{};
            L.es = base_e + xe;
            L.ck = base_c + xc;
            el[e] = L;
            es[e] = L.es;
            ck[e] = L.ck;
        }
        if (v) {
            EntryLayout L;
            L.tensor = pe.tensor;
            L.count = pe.count;
            L.idx_off = pe.idx_off;
            L.idx_nbytes = pe.idx_nbytes;
            L.val_off = pe.val_off;
            L.es = base_e + xe;
            L.ck = base_c + xc;
            L.numel = ne;
            L.cols = cols[pe.tensor];
            L.flat_base = base_f + xf;
            L.col_start = pe.idx_nbytes;  // D2 overwrites once it finds the row stream's end
            L.cu = 0;
            el[e] = L;
            es[e] = L.es;
            ck[e] = L.ck;
            // fixed-layout fast path (apply_fast.cu) only if no entry needs escapes
            if (repr <= PULSE_FLAT_INT32 &&
                pe.idx_nbytes != (repr == PULSE_COO_DOWNSCALED ? 3 : 4) * pe.count)
                atomicExch(flags, 1u);
            if (repr > PULSE_FLAT_INT32) {
                // caller-provided int64 indices: no payload to check
            } else if (repr != PULSE_COO_DOWNSCALED) {
                // patch.hpp:193,217: require_int32_indexable; then u32 reads of `count`
                // entries (truncation) and the trailing-bytes check.
                if (ne >= (1ull << 31)) report(err, error_key(e, kStageTensor, 0, kDimInt32));
                if (pe.idx_nbytes < 4 * pe.count)
                    report(err, error_key(e, kStageRows, pe.idx_nbytes / 4, kTrunc));
                else if (pe.idx_nbytes > 4 * pe.count)
                    report(err, error_key(e, kStageTrailing, 0, kTrailing));
            } else if (pe.count > 0 && pe.idx_nbytes == 0) {
                report(err, error_key(e, kStageRows, 0, kTrunc));
            }
        }
        base_e += te;
        base_c += tc;
        base_f += tf;
    }
    if (threadIdx.x == 0) {
        es[n_e] = base_e;
        ck[n_e] = base_c;
        totals[kTotEntries] = base_e;
        totals[kTotRowChunks] = base_c;
        if (base_e > cap) {  // more entries than the plan's scratch holds: decode nothing
            report(err, error_key(0, kStageTensor, 0, kCapacity));
            totals[kTotEntries] = 0;
            totals[kTotRowChunks] = 0;
            atomicExch(flags, 1u);
        }
    }
}

// =============================================================================================
// D1: fixed-width payloads (COO_INT32, FLAT_INT32)
// =============================================================================================
template <bool kFlat>
__global__ void __launch_bounds__(kThreads)
d_fixed(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ es, uint32_t n_e,
        const uint8_t* __restrict__ body, const pulse_flat_carry* __restrict__ carry,
        uint64_t* __restrict__ status, uint64_t* __restrict__ totals, uint64_t* __restrict__ out,
        uint64_t* __restrict__ err, const uint32_t* __restrict__ flags) {
    if (*(volatile const uint32_t*)flags == 0) return;  // fixed-layout fast path handled it
    using Op = typename std::conditional<kFlat, SumOp, SegSumOp>::type;
    constexpr uint64_t H = SegSumOp::kHead;
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_tile, s_excl;
    const uint64_t n = totals[kTotEntries];
    const uint64_t n_tiles = (n + kChunkEntries - 1) / kChunkEntries;
    const bool has_prev = carry && carry->has_prev;
    const uint64_t gap_base = has_prev ? carry->gap_base : 0;
    while (true) {
        if (threadIdx.x == 0) s_tile = take_ticket(totals, 0);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= n_tiles) break;
        const uint64_t i0 = tile * kChunkEntries + uint64_t(threadIdx.x) * kEntriesPerThread;
        const uint64_t i1 = min(i0 + kEntriesPerThread, n);
        uint32_t g[kEntriesPerThread];
        uint64_t agg = 0;
        int k = 0;
        walk(es, n_e, i0, i1, [&](uint64_t, uint32_t e, uint64_t o) {
            const EntryLayout& L = el[e];
            const uint32_t gap = 4 * o + 4 <= L.idx_nbytes ? rd_u32(body + L.idx_off + 4 * o) : 0;
            g[k++] = gap;
            agg = Op::op(agg, (!kFlat && o == 0) ? (H | gap) : uint64_t(gap));
        });
        uint64_t tot;
        const uint64_t bex = block_exclusive<Op>(agg, s_warp, tot);
        if (threadIdx.x < 32) {
            const uint64_t x = lookback<Op>(status, tile, tot);
            if (threadIdx.x == 0) s_excl = x;
        }
        __syncthreads();
        uint64_t acc = Op::op(s_excl, bex);
        k = 0;
        walk(es, n_e, i0, i1, [&](uint64_t i, uint32_t e, uint64_t o) {
            const EntryLayout& L = el[e];
            const uint32_t gap = g[k++];
            acc = Op::op(acc, (!kFlat && o == 0) ? (H | gap) : uint64_t(gap));
            if (4 * o + 4 > L.idx_nbytes) return;  // truncated: reported by d_layout
            const uint64_t S = acc & (H - 1);
            if (kFlat) {
                // patch.hpp:219-237: global = prev + entry (first of stream absolute)
                if (gap == 0 && (i > 0 || has_prev)) { report(err, error_key(e, kStageRows, o, kZeroGap)); return; }
                const int64_t local = int64_t(S) - int64_t(gap_base) - int64_t(L.flat_base);
                if (local < 0 || uint64_t(local) >= L.numel) { report(err, error_key(e, kStageRows, o, kIdxRange)); return; }
                out[i] = uint64_t(local);
            } else {
                // patch.hpp:195-210
                if (o > 0 && gap == 0) { report(err, error_key(e, kStageRows, o, kZeroGap)); return; }
                if (S >= L.numel) { report(err, error_key(e, kStageRows, o, kIdxRange)); return; }
                out[i] = S;
            }
        });
        __syncthreads();
    }
}

// =============================================================================================
// D2: COO_DOWNSCALED row stream
// =============================================================================================
__device__ __forceinline__ uint64_t row_sync_start(const uint8_t* blob, uint64_t a) {
    // walk back to a position with no 0xFF among the 4 preceding bytes
    uint64_t p = a;
    while (p > 0) {
        bool ff = false;
        const uint64_t lo = p >= 4 ? p - 4 : 0;
        for (uint64_t q = lo; q < p; ++q) ff |= blob[q] == 0xFF;
        if (!ff) break;
        --p;
    }
    // parse forward to the first entry boundary >= a
    while (p < a) p += blob[p] == 0xFF ? 5 : 1;
    return p;
}

__global__ void __launch_bounds__(kThreads)
d_rows(EntryLayout* __restrict__ el, const uint64_t* __restrict__ ck, uint32_t n_e,
       const uint8_t* __restrict__ body, uint64_t* __restrict__ status, uint64_t* __restrict__ totals,
       uint32_t* __restrict__ rowgap, uint64_t* __restrict__ err, const uint32_t* __restrict__ flags) {
    if (*(volatile const uint32_t*)flags == 0) return;  // fixed-layout fast path handled it
    constexpr uint64_t H = SegSumOp::kHead;
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_tile, s_excl;
    const uint64_t n_chunks = totals[kTotRowChunks];
    const uint64_t n_tiles = (n_chunks + kParseChunksPerTile - 1) / kParseChunksPerTile;
    while (true) {
        if (threadIdx.x == 0) s_tile = take_ticket(totals, 1);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= n_tiles) break;
        const uint64_t c = tile * kParseChunksPerTile + threadIdx.x;
        uint32_t e = 0;
        uint64_t a = 0, b = 0, nb = 0, first = 0;
        const uint8_t* blob = body;
        uint64_t item = 0;
        if (c < n_chunks) {
            e = upper_index<uint64_t>(ck, 0, n_e, c);
            const uint64_t q = c - ck[e];
            nb = el[e].idx_nbytes;
            blob = body + el[e].idx_off;
            a = q * kParseBytes;
            b = min(a + kParseBytes, nb);
            first = row_sync_start(blob, a);
            uint64_t cnt = 0;
            for (uint64_t p = first; p < b; p += blob[p] == 0xFF ? 5 : 1) ++cnt;
            item = (q == 0 ? H : 0) | cnt;
        }
        uint64_t tot;
        const uint64_t bex = block_exclusive<SegSumOp>(item, s_warp, tot);
        if (threadIdx.x < 32) {
            const uint64_t x = lookback<SegSumOp>(status, tile, tot);
            if (threadIdx.x == 0) s_excl = x;
        }
        __syncthreads();
        if (c < n_chunks) {
            uint64_t o = (item & H) ? 0 : (SegSumOp::op(s_excl, bex) & (H - 1));
            const EntryLayout& L = el[e];
            for (uint64_t p = first; p < b; ++o) {
                const bool esc = blob[p] == 0xFF;
                const uint64_t len = esc ? 5 : 1;
                if (o < L.count) {
                    if (p + len > nb) {
                        report(err, error_key(e, kStageRows, o, kTrunc));
                    } else {
                        rowgap[L.es + o] = esc ? rd_u32(blob + p + 1) : blob[p];
                        if (p + len == nb && o + 1 < L.count)  // stream ends before `count` rows
                            report(err, error_key(e, kStageRows, o + 1, kTrunc));
                    }
                } else if (o == L.count) {
                    el[e].col_start = p;
                }
                p += len;
            }
        }
        __syncthreads();
    }
}

// =============================================================================================
// D3: column-stream chunk layout
// =============================================================================================
__global__ void __launch_bounds__(kLT, 1)
d_col_layout(EntryLayout* __restrict__ el, uint32_t n_e, uint64_t* __restrict__ cu,
             uint64_t* __restrict__ totals, uint64_t* __restrict__ err,
             const uint32_t* __restrict__ flags) {
    if (*(volatile const uint32_t*)flags == 0) return;
    __shared__ uint64_t s_tmp[33];
    uint64_t base = 0;
    for (uint32_t e0 = 0; e0 < n_e; e0 += kLT) {
        const uint32_t e = e0 + threadIdx.x;
        uint64_t chunks = 0;
        if (e < n_e) {
            const EntryLayout L = el[e];
            const uint64_t len = L.idx_nbytes - L.col_start;
            chunks = (len + kParseBytes - 1) / kParseBytes;
            if (len == 0 && L.count > 0) report(err, error_key(e, kStageCols, 0, kTrunc));
        }
        uint64_t xs[1] = {chunks}, ts[1];
        cta_exclusive_scan<1, kLT, AllSum>(xs, ts, s_tmp);
        const uint64_t x = xs[0], t = ts[0];
        if (e < n_e) {
            el[e].cu = base + x;
            cu[e] = base + x;
        }
        base += t;
    }
    if (threadIdx.x == 0) {
        cu[n_e] = base;
        totals[kTotColChunks] = base;
    }
}

// =============================================================================================
// D4: COO_DOWNSCALED column stream (2-byte units)
// =============================================================================================
__device__ __forceinline__ bool col_marker(const uint8_t* s, uint64_t p, uint64_t len) {
    return p + 2 <= len && s[p] == 0xFF && s[p + 1] == 0xFF;
}

__device__ __forceinline__ uint64_t col_sync_start(const uint8_t* s, uint64_t a, uint64_t len) {
    uint64_t p = a;  // even
    while (p > 0) {
        const bool m = col_marker(s, p - 2, len) || (p >= 4 && col_marker(s, p - 4, len));
        if (!m) break;
        p -= 2;
    }
    while (p < a) p += col_marker(s, p, len) ? 6 : 2;
    return p;
}

__global__ void __launch_bounds__(kThreads)
d_cols(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ cu, uint32_t n_e,
       const uint8_t* __restrict__ body, uint64_t* __restrict__ status, uint64_t* __restrict__ totals,
       uint32_t* __restrict__ colent, uint64_t* __restrict__ err, const uint32_t* __restrict__ flags) {
    if (*(volatile const uint32_t*)flags == 0) return;  // fixed-layout fast path handled it
    constexpr uint64_t H = SegSumOp::kHead;
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_tile, s_excl;
    const uint64_t n_chunks = totals[kTotColChunks];
    const uint64_t n_tiles = (n_chunks + kParseChunksPerTile - 1) / kParseChunksPerTile;
    while (true) {
        if (threadIdx.x == 0) s_tile = take_ticket(totals, 2);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= n_tiles) break;
        const uint64_t c = tile * kParseChunksPerTile + threadIdx.x;
        uint32_t e = 0;
        uint64_t b = 0, len = 0, first = 0;
        const uint8_t* s = body;
        uint64_t item = 0;
        if (c < n_chunks) {
            e = upper_index<uint64_t>(cu, 0, n_e, c);
            const uint64_t q = c - cu[e];
            const EntryLayout& L = el[e];
            s = body + L.idx_off + L.col_start;
            len = L.idx_nbytes - L.col_start;
            const uint64_t a = q * kParseBytes;
            b = min(a + kParseBytes, len);
            first = col_sync_start(s, a, len);
            uint64_t cnt = 0;
            for (uint64_t p = first; p < b; p += col_marker(s, p, len) ? 6 : 2) ++cnt;
            item = (q == 0 ? H : 0) | cnt;
        }
        uint64_t tot;
        const uint64_t bex = block_exclusive<SegSumOp>(item, s_warp, tot);
        if (threadIdx.x < 32) {
            const uint64_t x = lookback<SegSumOp>(status, tile, tot);
            if (threadIdx.x == 0) s_excl = x;
        }
        __syncthreads();
        if (c < n_chunks) {
            uint64_t o = (item & H) ? 0 : (SegSumOp::op(s_excl, bex) & (H - 1));
            const EntryLayout& L = el[e];
            for (uint64_t p = first; p < b; ++o) {
                const bool esc = col_marker(s, p, len);
                const uint64_t elen = esc ? 6 : 2;
                if (o < L.count) {
                    if (p + elen > len) {
                        report(err, error_key(e, kStageCols, o, kTrunc));
                    } else {
                        colent[L.es + o] = esc ? rd_u32(s + p + 2) : rd_u16(s + p);
                        if (p + elen == len && o + 1 < L.count)
                            report(err, error_key(e, kStageCols, o + 1, kTrunc));
                    }
                } else if (o == L.count) {
                    report(err, error_key(e, kStageTrailing, 0, kTrailing));  // index_coding.hpp:154-156
                }
                p += elen;
            }
        }
        __syncthreads();
    }
}

// =============================================================================================
// D5: COO_DOWNSCALED assemble
// =============================================================================================
__global__ void __launch_bounds__(kThreads)
d_assemble(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ es, uint32_t n_e,
           const uint32_t* __restrict__ rowgap, const uint32_t* __restrict__ colent,
           uint64_t* __restrict__ st_rows, uint64_t* __restrict__ st_cols, uint64_t* __restrict__ totals,
           uint64_t* __restrict__ out, uint64_t* __restrict__ err, const uint32_t* __restrict__ flags,
           int64_t* __restrict__ raw_rows = nullptr, int64_t* __restrict__ raw_cols = nullptr) {
    if (*(volatile const uint32_t*)flags == 0) return;  // fixed-layout fast path handled it
    constexpr uint64_t H = SegSumOp::kHead;
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_tile, s_xr, s_xc;
    const uint64_t n = totals[kTotEntries];
    const uint64_t n_tiles = (n + kChunkEntries - 1) / kChunkEntries;
    while (true) {
        if (threadIdx.x == 0) s_tile = take_ticket(totals, 3);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= n_tiles) break;
        const uint64_t i0 = tile * kChunkEntries + uint64_t(threadIdx.x) * kEntriesPerThread;
        const uint64_t i1 = min(i0 + kEntriesPerThread, n);
        uint32_t rg[kEntriesPerThread], cv[kEntriesPerThread];
        uint64_t ar = 0, ac = 0;
        int k = 0;
        walk(es, n_e, i0, i1, [&](uint64_t i, uint32_t, uint64_t o) {
            rg[k] = rowgap[i];
            cv[k] = colent[i];
            const bool new_row = o == 0 || rg[k] != 0;
            ar = SegSumOp::op(ar, (o == 0 ? H : 0) | rg[k]);
            ac = SegSumOp::op(ac, (new_row ? H : 0) | cv[k]);
            ++k;
        });
        uint64_t tr, tc;
        const uint64_t xr = block_exclusive<SegSumOp>(ar, s_warp, tr);
        const uint64_t xc = block_exclusive<SegSumOp>(ac, s_warp, tc);
        if (threadIdx.x < 32) {
            const uint64_t a = lookback<SegSumOp>(st_rows, tile, tr);
            const uint64_t b = lookback<SegSumOp>(st_cols, tile, tc);
            if (threadIdx.x == 0) { s_xr = a; s_xc = b; }
        }
        __syncthreads();
        uint64_t row = SegSumOp::op(s_xr, xr), col = SegSumOp::op(s_xc, xc);
        k = 0;
        walk(es, n_e, i0, i1, [&](uint64_t i, uint32_t e, uint64_t o) {
            const bool new_row = o == 0 || rg[k] != 0;
            row = SegSumOp::op(row, (o == 0 ? H : 0) | rg[k]);
            col = SegSumOp::op(col, (new_row ? H : 0) | cv[k]);
            const uint32_t entry = cv[k];
            ++k;
            const EntryLayout& L = el[e];
            if (!new_row && entry == 0) { report(err, error_key(e, kStageCols, o, kZeroColGap)); return; }
            const uint64_t r = row & (H - 1), cc = col & (H - 1);
            if (raw_rows) {  // upscale_coo: the coordinates themselves, no tensor range checks
                raw_rows[i] = int64_t(r);
                raw_cols[i] = int64_t(cc);
                return;
            }
            if (cc >= L.cols) { report(err, error_key(e, kStageRange, o, kColRange)); return; }
            const uint64_t flat = r * L.cols + cc;
            if (flat >= L.numel) { report(err, error_key(e, kStageRange, o, kIdxRange)); return; }
            out[i] = flat;
        });
        __syncthreads();
    }
}

// =============================================================================================
// D6: scatter (validate-then-scatter: nothing is written if any check failed)
// =============================================================================================
__global__ void __launch_bounds__(kThreads)
d_scatter(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ es, uint32_t n_e,
          const uint8_t* __restrict__ body, const uint16_t* __restrict__ vals,
          const uint64_t* __restrict__ flat, const int64_t* __restrict__ flat64,
          uint16_t* const* __restrict__ weights, const uint64_t* __restrict__ totals,
          const uint64_t* __restrict__ err, const uint32_t* __restrict__ flags) {
    if (*err != kNoError) return;
    if (flags && *(volatile const uint32_t*)flags == 0) return;  // fixed-layout fast path scattered
    const uint64_t n = totals[kTotEntries];
    const uint64_t stride = uint64_t(gridDim.x) * kThreads * kEntriesPerThread;
    for (uint64_t i0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) * kEntriesPerThread; i0 < n; i0 += stride) {
        walk(es, n_e, i0, min(i0 + kEntriesPerThread, n), [&](uint64_t i, uint32_t e, uint64_t o) {
            const EntryLayout& L = el[e];
            const uint16_t v = vals ? vals[i] : uint16_t(rd_u16(body + L.val_off + 2 * o));
            const uint64_t f = flat64 ? uint64_t(flat64[i]) : flat[i];
            weights[L.tensor][f] = v;
        });
    }
}

// Validation of caller-provided int64 indices (patch.hpp:325-336).
__global__ void __launch_bounds__(kThreads)
d_validate_idx64(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ es, uint32_t n_e,
                 const int64_t* __restrict__ idx, const uint64_t* __restrict__ totals,
                 uint64_t* __restrict__ err) {
    const uint64_t n = totals[kTotEntries];
    const uint64_t stride = uint64_t(gridDim.x) * kThreads * kEntriesPerThread;
    for (uint64_t i0 = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) * kEntriesPerThread; i0 < n; i0 += stride) {
        walk(es, n_e, i0, min(i0 + kEntriesPerThread, n), [&](uint64_t i, uint32_t e, uint64_t o) {
            const int64_t last = o == 0 ? -1 : idx[i - 1];
            if (idx[i] <= last) { report(err, error_key(e, kStageRows, o, kApplyOrder)); return; }
            if (uint64_t(idx[i]) >= el[e].numel) report(err, error_key(e, kStageRows, o, kApplyRange));
        });
    }
}

__global__ void d_finalize(const uint64_t* __restrict__ totals, uint32_t n_e, const uint64_t* __restrict__ err,
                           pulse_result* __restrict__ result) {
    if (threadIdx.x) return;
    pulse_result r{};
    r.n_changes = totals[kTotEntries];
    r.n_entries = n_e;
    const uint64_t k = *err;
    if (k != kNoError) {
        r.status = check_status(key_check(k));
        r.err_check = key_check(k);
        r.err_stage = key_stage(k);
        r.err_tensor = key_tensor(k);
        r.err_elem = key_elem(k);
    }
    *result = r;
}

// =============================================================================================
// launchers
// =============================================================================================
static unsigned persistent_grid() { return unsigned(sm_count() * 8); }

static void decode_prologue(const PlanDev& p, const pulse_patch_entry* entries, uint32_t n_entries,
                            uint32_t repr, cudaStream_t s, const pulse_result* patch_result = nullptr) {
    d_layout<<<1, kLT, 0, s>>>(entries, n_entries, p.numel, p.cols, repr, p.elay, p.d_es, p.d_ck,
                              p.d_totals, p.err, p.d_flags, p.cap, patch_result);
    PULSE_LAUNCHED("d_layout", s);
}

// Look-back status words only matter on the general path; clear them there.
__global__ void d_clear_status(uint64_t* __restrict__ st, uint64_t n, const uint32_t* __restrict__ flags) {
    if (*(volatile const uint32_t*)flags == 0) return;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        st[i] = 0;
}

void launch_decode(const PlanDev& p, uint32_t repr, const uint8_t* body,
                   const pulse_patch_entry* entries, uint32_t n_entries,
                   const pulse_flat_carry* carry, int weights_slot, int64_t* out_indices,
                   pulse_result* result, cudaStream_t s, const pulse_result* patch_result) {
    decode_prologue(p, entries, n_entries, repr, s, patch_result);
    uint64_t* out = out_indices ? reinterpret_cast<uint64_t*>(out_indices) : p.flat;
    const unsigned g = persistent_grid();
    uint64_t* st0 = p.d_status;
    uint64_t* st1 = p.d_status + p.d_status_len;
    uint64_t* st2 = p.d_status + 2 * p.d_status_len;
    uint64_t* st3 = p.d_status + 3 * p.d_status_len;
    if (n_entries > 0) {
        // common case: fixed-layout payloads (no escapes) -- apply_fast.cu
        launch_apply_fast(p, repr, body, n_entries, carry, weights_slot, out_indices, p.d_flags, s);
        // general path (escapes, malformed sizes): runs only if d_layout / F1 raised flags[0]
        launch_gated(s, p.d_flags, [&](cudaStream_t gs) {
            d_clear_status<<<g, kThreads, 0, gs>>>(p.d_status, 4 * p.d_status_len, p.d_flags);
            PULSE_LAUNCHED("d_clear_status", gs);
            if (repr == PULSE_COO_INT32) {
                d_fixed<false><<<g, kThreads, 0, gs>>>(p.elay, p.d_es, n_entries, body, nullptr, st0, p.d_totals, out, p.err, p.d_flags);
                PULSE_LAUNCHED("d_fixed<false>", gs);
            } else if (repr == PULSE_FLAT_INT32) {
                d_fixed<true><<<g, kThreads, 0, gs>>>(p.elay, p.d_es, n_entries, body, carry, st0, p.d_totals, out, p.err, p.d_flags);
                PULSE_LAUNCHED("d_fixed<true>", gs);
            } else {
                d_rows<<<g, kThreads, 0, gs>>>(p.elay, p.d_ck, n_entries, body, st2, p.d_totals, p.rowgap, p.err, p.d_flags);
                PULSE_LAUNCHED("d_rows", gs);
                d_col_layout<<<1, kLT, 0, gs>>>(p.elay, n_entries, p.d_cu, p.d_totals, p.err, p.d_flags);
                PULSE_LAUNCHED("d_col_layout", gs);
                d_cols<<<g, kThreads, 0, gs>>>(p.elay, p.d_cu, n_entries, body, st3, p.d_totals, p.colent, p.err, p.d_flags);
                PULSE_LAUNCHED("d_cols", gs);
                d_assemble<<<g, kThreads, 0, gs>>>(p.elay, p.d_es, n_entries, p.rowgap, p.colent, st0, st1, p.d_totals, out, p.err, p.d_flags);
                PULSE_LAUNCHED("d_assemble", gs);
            }
            if (weights_slot >= 0)
                {
                d_scatter<<<g, kThreads, 0, gs>>>(p.elay, p.d_es, n_entries, body, nullptr, out, nullptr,
                                                 p.slot[weights_slot], p.d_totals, p.err, p.d_flags);
                PULSE_LAUNCHED("d_scatter", gs);
                }
        });
    }
    d_finalize<<<1, 32, 0, s>>>(p.d_totals, n_entries, p.err, result);
    PULSE_LAUNCHED("d_finalize", s);
}

void launch_apply_idx64(const PlanDev& p, const int64_t* idx64, const uint16_t* vals,
                        const pulse_patch_entry* entries, uint32_t n_entries, int weights_slot,
                        pulse_result* result, cudaStream_t s) {
    decode_prologue(p, entries, n_entries, kNoPayload, s);
    const unsigned g = persistent_grid();
    if (n_entries > 0) {
        d_validate_idx64<<<g, kThreads, 0, s>>>(p.elay, p.d_es, n_entries, idx64, p.d_totals, p.err);
        PULSE_LAUNCHED("d_validate_idx64", s);
        if (weights_slot >= 0)
            {
            d_scatter<<<g, kThreads, 0, s>>>(p.elay, p.d_es, n_entries, nullptr, vals, nullptr, idx64,
                                             p.slot[weights_slot], p.d_totals, p.err, nullptr);
            PULSE_LAUNCHED("d_scatter", s);
            }
    }
    d_finalize<<<1, 32, 0, s>>>(p.d_totals, n_entries, p.err, result);
    PULSE_LAUNCHED("d_finalize", s);
}

// upscale_coo (index_coding.hpp:130-158) of one payload, in parallel: the general decoder's
// row and column stream parses (sync-point rule) for a one-entry table, then the segmented
// sums written as (row, column) pairs.  The caller's plan has one tensor; its geometry is
// not checked (no range checks in raw mode).
__global__ void d_force_general(uint32_t* __restrict__ flags) { flags[0] = 1u; }

void launch_coo_unpack_par(const PlanDev& p, const uint8_t* body, const pulse_patch_entry* entry,
                           int64_t* rows, int64_t* cols, pulse_result* result, cudaStream_t s) {
    decode_prologue(p, entry, 1, PULSE_COO_DOWNSCALED, s);
    d_force_general<<<1, 1, 0, s>>>(p.d_flags);
    PULSE_LAUNCHED("d_force_general", s);
    const unsigned g = persistent_grid();
    uint64_t* st0 = p.d_status;
    uint64_t* st1 = p.d_status + p.d_status_len;
    uint64_t* st2 = p.d_status + 2 * p.d_status_len;
    uint64_t* st3 = p.d_status + 3 * p.d_status_len;
    d_clear_status<<<g, kThreads, 0, s>>>(p.d_status, 4 * p.d_status_len, p.d_flags);
    PULSE_LAUNCHED("d_clear_status", s);
    d_rows<<<g, kThreads, 0, s>>>(p.elay, p.d_ck, 1, body, st2, p.d_totals, p.rowgap, p.err, p.d_flags);
    PULSE_LAUNCHED("d_rows", s);
    d_col_layout<<<1, kLT, 0, s>>>(p.elay, 1, p.d_cu, p.d_totals, p.err, p.d_flags);
    PULSE_LAUNCHED("d_col_layout", s);
    d_cols<<<g, kThreads, 0, s>>>(p.elay, p.d_cu, 1, body, st3, p.d_totals, p.colent, p.err, p.d_flags);
    PULSE_LAUNCHED("d_cols", s);
    d_assemble<<<g, kThreads, 0, s>>>(p.elay, p.d_es, 1, p.rowgap, p.colent, st0, st1, p.d_totals, nullptr, p.err,
                                      p.d_flags, rows, cols);
    PULSE_LAUNCHED("d_assemble", s);
    d_finalize<<<1, 32, 0, s>>>(p.d_totals, 1, p.err, result);
    PULSE_LAUNCHED("d_finalize", s);
}

// Small device-to-peers store (pulse_store_to_peers): thread t copies byte t % nbytes to
// destination t / nbytes (NVLink stores when the destinations are peer-mapped).
__global__ void k_store_to_peers(const uint8_t* __restrict__ src, PeerPtrs dst, uint32_t n_dst, uint32_t nbytes) {
    for (uint32_t t = threadIdx.x; t < n_dst * nbytes; t += blockDim.x)
        static_cast<uint8_t*>(dst.p[t / nbytes])[t % nbytes] = src[t % nbytes];
}

void launch_store_to_peers(const void* src, const PeerPtrs& dst, uint32_t n_dst, uint32_t nbytes, cudaStream_t s) {
    k_store_to_peers<<<1, 256, 0, s>>>(static_cast<const uint8_t*>(src), dst, n_dst, nbytes);
    PULSE_LAUNCHED("k_store_to_peers", s);
}

// All-gather of small per-rank records over peer memory, inside a stream (or a graph):
// every rank's table holds 2 x world slots of kSlotBytes (record, then a u64 epoch tag at
// +kSlotTag), double-buffered by epoch parity so a rank one step ahead never overwrites a
// slot its peers have not read.  Post: epoch += 1, the record to this rank's slot in every
// table, a system fence, then the tag.  Wait: spin until every rank's slot carries the
// epoch, fence, copy the records out contiguously.
constexpr uint32_t kSlotBytes = 64, kSlotTag = 48;

__global__ void k_peer_post(const uint8_t* __restrict__ src, PeerPtrs tables, uint32_t world, uint32_t rank,
                            uint32_t nbytes, unsigned long long* __restrict__ epoch) {
    __shared__ unsigned long long s_e;
    if (threadIdx.x == 0) s_e = ++*epoch;
    __syncthreads();
    const unsigned long long e = s_e;
    const uint32_t slot = uint32_t((e & 1) * world + rank) * kSlotBytes;
    for (uint32_t t = threadIdx.x; t < world * nbytes; t += blockDim.x)
        static_cast<uint8_t*>(tables.p[t / nbytes])[slot + t % nbytes] = src[t % nbytes];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < world)
        *reinterpret_cast<volatile unsigned long long*>(static_cast<uint8_t*>(tables.p[threadIdx.x]) + slot + kSlotTag) = e;
}

__global__ void k_peer_wait(const uint8_t* __restrict__ table, uint32_t world, uint32_t nbytes,
                            const unsigned long long* __restrict__ epoch, uint8_t* __restrict__ out) {
    const unsigned long long e = *epoch;
    const uint8_t* base = table + (e & 1) * world * kSlotBytes;
    if (threadIdx.x < world) {
        const volatile unsigned long long* tag =
            reinterpret_cast<const volatile unsigned long long*>(base + threadIdx.x * kSlotBytes + kSlotTag);
        uint64_t spins = 0;
        while (*tag != e) {
            __nanosleep(64);
            if (++spins > 64 * kSpinLimit) {  // seconds: a rank that never posts -- fail loudly
                watchdog_fire(4, threadIdx.x, e, *tag);
                __trap();
            }
        }
    }
    __threadfence_system();
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < world * nbytes; t += blockDim.x)
        out[t] = reinterpret_cast<const volatile uint8_t*>(base)[(t / nbytes) * kSlotBytes + t % nbytes];
}

void launch_peer_allgather(const void* src, const PeerPtrs& tables, const void* my_table, uint32_t world,
                           uint32_t rank, uint32_t nbytes, unsigned long long* epoch, void* out, cudaStream_t s) {
    k_peer_post<<<1, 256, 0, s>>>(static_cast<const uint8_t*>(src), tables, world, rank, nbytes, epoch);
    PULSE_LAUNCHED("k_peer_post", s);
    k_peer_wait<<<1, 256, 0, s>>>(static_cast<const uint8_t*>(my_table), world, nbytes, epoch,
                                  static_cast<uint8_t*>(out));
    PULSE_LAUNCHED("k_peer_wait", s);
}

// FLAT_INT32 carry of shard `rank` from all ranks' scan summaries (device side
// of shard.flat_carry): the nearest earlier rank that emitted an index.
__global__ void k_flat_carry(const pulse_scan_summary* __restrict__ gathered, uint32_t rank,
                             pulse_flat_carry* __restrict__ out) {
    if (threadIdx.x) return;
    pulse_flat_carry c{0, 0};
    for (int q = int(rank) - 1; q >= 0; --q) {
        if (gathered[q].has_change) {
            c.has_prev = 1;
            c.gap_base = gathered[q].last_gap_base;
            break;
        }
    }
    *out = c;
}

void launch_flat_carry(const pulse_scan_summary* gathered, uint32_t rank, pulse_flat_carry* out, cudaStream_t s) {
    k_flat_carry<<<1, 32, 0, s>>>(gathered, rank, out);
    PULSE_LAUNCHED("k_flat_carry", s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_decode)

}  // namespace dev
}  // namespace pulse
