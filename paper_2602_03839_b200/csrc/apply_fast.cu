// PULSE apply, fixed-layout fast path (sm_100a).
//
// When no entry of a patch needs an escape -- COO_DOWNSCALED payloads with
// idx_nbytes == 3 * count and no 0xFF row byte / 0xFFFF column unit, or any
// COO_INT32 / FLAT_INT32 payload (always 4 bytes per entry) -- entry o of a
// tensor has its row gap at byte o, its column entry at byte count + 2o (or its
// u32 gap at byte 4o) of the index payload (index_coding.hpp:104-127,
// patch.hpp:120-156).  Decoding is then a pair of segmented prefix sums over
// the entries, read straight from the body.  The pipeline (launch_all):
//
//   F1s f_stream<agg>  per warp range (4096 entries; 1024 under 16 M changes): segmented-sum aggregates
//                      (rows restart at each tensor; columns at each new row,
//                      index_coding.hpp:141-153), escape markers, the range's
//                      patch entry, and every reference check that needs no
//                      carry (see "Checks without the carry" below); lists the
//                      chunks of non-plain ranges for F3.
//   F2 f_range_scan    exclusive scan of the range aggregates (decoupled
//                      look-back over blocks) + F1s's deferred column check.
//   F3 f_pass<validate> the exact reference checks on F1s's listed chunks (on
//                      every range if anything looked wrong); a second pass,
//                      behind a conditional graph node, re-checks everything
//                      only if a check failed, so the reported error is the
//                      reference's first failing entry.
//   F5 f_stream<scatter> decode + write, only if nothing failed: a bad patch
//                      never half-applies (the reference validates on a copy,
//                      patch.hpp:311), and no backup of the old values is needed.
//   (decode-only callers -- int64 indices out -- use f_pass<scatter> last.)
//   PULSE_APPLY_MODE=1|2 selects the earlier pipelines (F1 f_pass<agg>, then a
//   checked scatter with backup + restore, or exact validation of every range)
//   for A/B measurements.
//
// Data movement.  f_stream stages the next chunk (rows / columns / u32 gaps /
// values) with cp.async while the current one decodes, and removes the
// payload's byte misalignment on the shared-memory read (funnel shifts); each
// lane decodes 16 or 32 CONSECUTIVE entries serially (one warp segmented scan
// per chunk).  F5 transposes the decoded indices back to entry order through
// shared memory so each warp store instruction covers 32 consecutive changes
// (a few sectors for clustered updates) rather than 32 scattered ones.  Chunks
// never straddle two patch entries; only tensors with >= 2^32 elements take the
// per-round walker path.
//
// If d_layout or F1s finds anything the fixed layout cannot express (escapes,
// short/long payloads, marker bytes), `flags[0]` routes the patch to the
// general parser in decode.cu instead; every kernel checks it on entry.
#include <cstdlib>

#include "device.cuh"
#include "internal.hpp"
#include "stage.cuh"

namespace pulse {
namespace dev {

namespace {

// Entries per warp range (aggregate granularity), the same rule in every apply kernel of a call:
// 4096 for large patches, 1024 under PULSE_APPLY_RANGE_SPLIT (16 M) changes so small patches keep
// enough warps busy (C1, 168 K changes: 41 ranges of 4096 left most of the GPU idle in F1s / F5).
#ifndef PULSE_F3_CTAS_PER_SM
#define PULSE_F3_CTAS_PER_SM 64  // no cap
#endif
#ifndef PULSE_F5_NATURAL
#define PULSE_F5_NATURAL 0  // F5 scatter in entry order (1) or as interleaved pairs (0)
#endif
#ifndef PULSE_APPLY_RANGE_MIN
#define PULSE_APPLY_RANGE_MIN 1024
#endif
#ifndef PULSE_APPLY_RANGE_SPLIT
#define PULSE_APPLY_RANGE_SPLIT (uint64_t(1) << 24)
#endif
#ifndef PULSE_APPLY_RANGE_MAX
#define PULSE_APPLY_RANGE_MAX 4096
#endif
constexpr uint32_t kRangeMin = PULSE_APPLY_RANGE_MIN;
__device__ __forceinline__ uint32_t apply_range(uint64_t n) {
    return n < uint64_t(PULSE_APPLY_RANGE_SPLIT) ? kRangeMin : uint32_t(PULSE_APPLY_RANGE_MAX);
}
constexpr uint32_t kChunk = 1024;  // entries staged per warp step
constexpr uint32_t kPer = kChunk / 32;  // consecutive entries per lane
constexpr uint64_t H = SegSumOp::kHead;

enum Repr : int { kCoo = 0, kI32 = 1, kFlat = 2 };
enum Pass : int { kAgg = 0, kValidate = 1, kScatter = 2, kApply = 3, kRestore = 4 };
__host__ __device__ constexpr bool checks(int pass) { return pass == kValidate || pass == kApply || pass == kRestore; }
__host__ __device__ constexpr bool reports(int pass) { return pass == kValidate || pass == kApply; }
constexpr uint32_t kInvalid = 0xFFFFFFFFu;  // decoded-index marker of an entry that failed a check

// Per-warp staging area (bytes).  a: COO rows (1 KiB used) or u32 gaps (4 KiB);
// b: COO column units; v: values; x: decoded tensor-local indices.
constexpr uint32_t kABytes = kChunk * 4, kBBytes = kChunk * 2, kVBytes = kChunk * 2, kXBytes = kChunk * 4;
__host__ __device__ constexpr uint32_t warp_smem(int pass) { return kABytes + kBBytes + (pass >= kScatter ? kVBytes + kXBytes : 0); }

__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// Inclusive SegSum scan over lanes of a (rows, cols) pair.
__device__ __forceinline__ void warp_segscan2(uint64_t& r, uint64_t& c) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t pr = __shfl_up_sync(0xffffffffu, r, off);
        const uint64_t pc = __shfl_up_sync(0xffffffffu, c, off);
        if (lane >= off) {
            r = SegSumOp::op(pr, r);
            c = SegSumOp::op(pc, c);
        }
    }
}

// The same on 32-bit words, segment head in bit 31 (values below 2^31).
__device__ __forceinline__ void warp_segscan2_32(uint32_t& r, uint32_t& c) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t pr = __shfl_up_sync(0xffffffffu, r, off);
        const uint32_t pc = __shfl_up_sync(0xffffffffu, c, off);
        if (lane >= off) {
            r = (r & 0x80000000u) ? r : ((pr + r) | (pr & 0x80000000u));
            c = (c & 0x80000000u) ? c : ((pc + c) | (pc & 0x80000000u));
        }
    }
}

// ---- per-round walker (fallback for chunks that straddle patch entries) -------------------
struct ECtx {
    uint32_t e;
    uint64_t lo, hi;  // entries [lo, hi) belong to e
    EntryLayout L;
};

__device__ __forceinline__ ECtx load_ectx(const EntryLayout* el, const uint64_t* es, uint32_t e) {
    ECtx c;
    c.e = e;
    c.lo = es[e];
    c.hi = es[e + 1];
    c.L = el[e];
    return c;
}

struct Fields {
    bool valid;
    uint32_t e;
    uint64_t o;
    uint32_t a;  // COO: row gap byte; int32: the u32 gap
    uint32_t b;  // COO: column entry (u16)
    uint32_t tensor;
    uint64_t val_off, numel, cols, flat_base;
};

struct EWalker {
    const EntryLayout* el;
    const uint64_t* es;
    uint32_t n_e;
    uint64_t base, end;
    ECtx ctx;

    __device__ EWalker(const EntryLayout* el_, const uint64_t* es_, uint32_t n_e_, uint64_t first, uint64_t last)
        : el(el_), es(es_), n_e(n_e_), base(first), end(last) {
        ctx = load_ectx(el, es, upper_index<uint64_t>(es, 0, n_e, first));
    }

    __device__ __forceinline__ Fields next(const uint8_t* __restrict__ body, bool coo) {
        const int lane = threadIdx.x & 31;
        Fields f;
        const uint64_t i = base + lane;
        f.valid = i < end;
        uint32_t e = ctx.e;
        uint64_t lo = ctx.lo, idx_off = ctx.L.idx_off, count = ctx.L.count;
        f.tensor = uint32_t(ctx.L.tensor);
        f.val_off = ctx.L.val_off;
        f.numel = ctx.L.numel;
        f.cols = ctx.L.cols;
        f.flat_base = ctx.L.flat_base;
        const bool crosses = base + 32 > ctx.hi;  // warp-uniform
        if (crosses && f.valid && i >= ctx.hi) {
            while (es[e + 1] <= i) ++e;
            const EntryLayout& L = el[e];
            lo = es[e];
            idx_off = L.idx_off;
            count = L.count;
            f.tensor = uint32_t(L.tensor);
            f.val_off = L.val_off;
            f.numel = L.numel;
            f.cols = L.cols;
            f.flat_base = L.flat_base;
        }
        f.e = e;
        f.o = i - lo;
        f.a = f.b = 0;
        if (f.valid) {
            const uint8_t* p = body + idx_off;
            if (coo) {
                f.a = p[f.o];
                f.b = rd_u16(p + count + 2 * f.o);
            } else {
                f.a = rd_u32(p + 4 * f.o);
            }
        }
        if (crosses) {
            const uint32_t last_e = __shfl_sync(0xffffffffu, e, 31);
            if (last_e != ctx.e) ctx = load_ectx(el, es, last_e);
        }
        base += 32;
        return f;
    }
};

__device__ __forceinline__ uint64_t seg_round_agg(bool head, uint64_t v) {
    const uint32_t hm = __ballot_sync(0xffffffffu, head);
    const int lane = threadIdx.x & 31;
    const int last = hm ? 31 - __clz(hm) : 0;
    uint64_t x = (hm == 0 || lane >= last) ? v : 0;
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x | (hm ? H : 0);
}

__device__ __forceinline__ uint64_t seg_round_scan(bool head, uint64_t v, uint64_t& carry) {
    const int lane = threadIdx.x & 31;
    uint64_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
    }
    const uint32_t hm = __ballot_sync(0xffffffffu, head) & lanemask_le();
    const int h = hm ? 31 - __clz(hm) : -1;
    const uint64_t ex_at_h = __shfl_sync(0xffffffffu, inc - v, h < 0 ? 0 : h);
    const uint64_t r = h < 0 ? carry + inc : inc - ex_at_h;
    carry = __shfl_sync(0xffffffffu, r, 31);
    return r;
}

// Error reporting stays out of line: the unrolled per-entry loops then keep a
// small instruction footprint (the checks almost never fire).
__device__ __noinline__ void report_cold(uint64_t* err, uint64_t key) { report(err, key); }

__device__ __forceinline__ bool fast_blocked(const uint32_t* flags) { return *(volatile const uint32_t*)flags != 0; }

struct ApplyArgs {
    const EntryLayout* el;
    const uint64_t* es;
    uint32_t n_e;
    const uint8_t* body;
    const pulse_flat_carry* carry;
    const uint64_t* totals;
    ulonglong2* agg;  // F1 out / F2 in-out / F3-F4 in
    uint32_t* flags;
    uint64_t* err;
    uint16_t* const* weights;
    int64_t* out_idx;
    uint16_t* backup;  // [entries]: pre-apply value of every written element (kApply / kRestore)
    uint64_t* scan_status;               // F2 look-back words (2 per block, zeroed per call)
    unsigned long long* scan_ticket;     // F2 block ticket (zeroed per call)
    uint32_t scan_blocks;                // F2 grid: blocks for the plan's capacity
    uint32_t* range_e;                   // [ranges] F1s out: patch entry holding each range's first entry
    bool checked;                        // the F1s-F5 pipeline (F1s checks, F3 on listed pieces)
    struct Piece {                       // F1s out: one chunk of a non-plain range, for F3
        uint64_t c0, rg, ar, ac;         // first entry, range, in-range aggregate at c0
        uint32_t len, e;                 // entries, patch entry
    }* pieces;
    unsigned long long* n_pieces;        // pieces appended (zeroed by decode_prologue)
    uint64_t piece_cap;                  // beyond it F1s falls back to checking every range exactly
    uint64_t* slack;                     // [ranges] F1s out: cols - 1 - first row segment's local end column
    int vmode;                           // F3 validate: 0 = non-plain ranges (all if suspect), 1 = all if any failure
};

// Walker path over entries [first, last) for one pass.  (ar, ac): aggregates
// (kAgg) or running values (validate / scatter); returned advanced with the
// marker flag.  Everything by value, not by reference: an address-taken
// ApplyArgs / ar / ac / marker would live in local memory across the caller's
// whole streaming loop (the same fix took K2 emit's LDL/STL count 294 -> 53).
struct SpanState {
    uint64_t ar, ac;
    bool marker;
};

template <int kRepr, int kPass>
__device__ __noinline__ SpanState slow_span(const ApplyArgs A, uint64_t first, uint64_t last, uint64_t ar,
                                            uint64_t ac, bool marker, bool has_prev, uint64_t gap_base) {
    constexpr bool coo = kRepr == kCoo;
    EWalker w(A.el, A.es, A.n_e, first, last);
    while (w.base < w.end) {
        const uint64_t i = w.base + (threadIdx.x & 31);
        const Fields f = w.next(A.body, coo);
        if (kPass == kAgg) {
            if (coo) {
                marker |= f.valid && (f.a == 0xFF || f.b == 0xFFFF);
                const bool hr = f.valid && f.o == 0;
                const bool hc = f.valid && (f.o == 0 || f.a != 0);
                ar = SegSumOp::op(ar, seg_round_agg(hr, f.a));
                ac = SegSumOp::op(ac, seg_round_agg(hc, f.b));
            } else {
                const bool hr = kRepr == kI32 && f.valid && f.o == 0;
                ar = SegSumOp::op(ar, seg_round_agg(hr, f.a));
            }
            continue;
        }
        // per entry: (valid, flat index); `valid` false once a check failed
        bool ok = f.valid;
        uint64_t flat = 0;
        if (coo) {
            const bool hr = f.valid && f.o == 0;
            const bool nr = f.valid && (f.o == 0 || f.a != 0);
            const uint64_t row = seg_round_scan(hr, f.a, ar);
            const uint64_t col = seg_round_scan(nr, f.b, ac);
            if (ok && checks(kPass)) {
                uint64_t key = kNoError;
                if (!nr && f.b == 0) key = error_key(f.e, kStageCols, f.o, kZeroColGap);
                else if (col >= f.cols) key = error_key(f.e, kStageRange, f.o, kColRange);
                else if (row * f.cols + col >= f.numel) key = error_key(f.e, kStageRange, f.o, kIdxRange);
                if (key != kNoError) {
                    ok = false;
                    if (reports(kPass)) report(A.err, key);
                }
            }
            flat = row * f.cols + col;
        } else if (kRepr == kI32) {
            const bool hr = f.valid && f.o == 0;
            const uint64_t idx = seg_round_scan(hr, f.a, ar);
            if (ok && checks(kPass)) {
                uint64_t key = kNoError;
                if (f.o > 0 && f.a == 0) key = error_key(f.e, kStageRows, f.o, kZeroGap);
                else if (idx >= f.numel) key = error_key(f.e, kStageRows, f.o, kIdxRange);
                if (key != kNoError) {
                    ok = false;
                    if (reports(kPass)) report(A.err, key);
                }
            }
            flat = idx;
        } else {  // FLAT_INT32: one running global sum (patch.hpp:219-237)
            const uint64_t S = seg_round_scan(false, f.a, ar);
            const int64_t local = int64_t(S) - int64_t(gap_base) - int64_t(f.flat_base);
            if (ok && checks(kPass)) {
                uint64_t key = kNoError;
                if (f.a == 0 && (i > 0 || has_prev)) key = error_key(f.e, kStageRows, f.o, kZeroGap);
                else if (local < 0 || uint64_t(local) >= f.numel) key = error_key(f.e, kStageRows, f.o, kIdxRange);
                if (key != kNoError) {
                    ok = false;
                    if (reports(kPass)) report(A.err, key);
                }
            }
            flat = uint64_t(local);
        }
        if (!ok || kPass == kValidate) continue;
        if (kPass == kScatter) {
            if (A.out_idx) A.out_idx[i] = int64_t(flat);
            else A.weights[f.tensor][flat] = uint16_t(rd_u16(A.body + f.val_off + 2 * f.o));
        } else if (kPass == kApply) {
            uint16_t* w = A.weights[f.tensor] + flat;
            A.backup[i] = *w;
            *w = uint16_t(rd_u16(A.body + f.val_off + 2 * f.o));
        } else if (kPass == kRestore) {
            A.weights[f.tensor][flat] = A.backup[i];
        }
    }
    return SpanState{ar, ac, marker};
}

}  // namespace

// =============================================================================================
// F1 / F3 / F4: one kernel body, three passes
// =============================================================================================
template <int kRepr, int kPass>
__global__ void __launch_bounds__(kThreads, kPass >= kScatter ? 2 : 4)
f_pass(ApplyArgs A) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (fast_blocked(A.flags)) return;
    if (kPass == kScatter && *(volatile const uint64_t*)A.err != kNoError) return;
    if (kPass == kRestore && *(volatile const uint64_t*)A.err == kNoError) return;  // nothing failed: keep
    constexpr bool coo = kRepr == kCoo;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* ws = smem + warp * warp_smem(kPass);
    uint4* sa = reinterpret_cast<uint4*>(ws);
    uint4* sb = reinterpret_cast<uint4*>(ws + kABytes);
    uint16_t* sv = reinterpret_cast<uint16_t*>(ws + kABytes + kBBytes);
    uint4* sx = reinterpret_cast<uint4*>(ws + kABytes + kBBytes + kVBytes);

    const uint64_t n = A.totals[0];
    const uint32_t kRange = apply_range(n);
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
    const bool has_prev = A.carry && A.carry->has_prev;
    const uint64_t gap_base = has_prev ? A.carry->gap_base : 0;
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;

    // F3 validate after F1s: exact checks where F1s could not decide (see f_stream).
    // Filtered: the non-plain ranges F1s listed, one 1024-entry chunk per warp, each
    // the pieces F1s listed (one entry-aligned chunk of a non-plain range each, with its
    // in-range carry), one per warp.
    bool filter = false;
    uint64_t n_items = n_ranges;
    if (kPass == kValidate && A.checked) {
        const bool suspect = *(volatile const uint32_t*)(A.flags + 1) != 0;
        if (A.vmode == 0) {
            filter = !suspect;
            if (filter) n_items = min(uint64_t(*(volatile const unsigned long long*)A.n_pieces), A.piece_cap);
        } else {  // second launch: re-check everything only if the filtered pass found a failure
            if (suspect || *(volatile const uint64_t*)A.err == kNoError) return;
        }
    }
    for (uint64_t it = uint64_t(blockIdx.x) * kWarps + warp; it < n_items; it += stride) {
        ApplyArgs::Piece pc{};
        if (filter) pc = A.pieces[it];
        const uint64_t rg = filter ? pc.rg : it;
        const uint64_t r0 = rg * kRange;
        const uint64_t c_first = filter ? pc.c0 : r0;
        // r1 as c_first + a 32-bit span: the form `filter ? pc.c0 + pc.len : min(r0 + kRange, n)`
        // with a run-time kRange made ptxas 12.9 guard the spill of r1 with the carry-out of its
        // own predicated add (tools/sass_pred_check.py), leaving a stale r1 in local memory
        const uint32_t span = filter ? pc.len : uint32_t(min(uint64_t(kRange), n > r0 ? n - r0 : 0));
        const uint64_t r1 = c_first + span;
        if (c_first >= r1) continue;
        uint64_t ar = 0, ac = 0;  // kAgg: aggregates; else running (row, col) / sums
        if (kPass != kAgg) {
            const ulonglong2 p = A.agg[rg];
            ar = p.x;
            ac = p.y;
            if (filter) {
                ar = SegSumOp::op(ar, pc.ar) & (H - 1);
                ac = SegSumOp::op(ac, pc.ac) & (H - 1);
            }
        }
        bool marker = false;
        // the chunk's entry from F1s (new pipeline) instead of a binary search over the entries
        uint32_t e = filter ? pc.e
                   : kPass != kAgg && A.checked ? A.range_e[rg] : upper_index<uint64_t>(A.es, 0, A.n_e, c_first);
        if (kPass == kAgg && lane == 0) A.range_e[rg] = e;
        // chunks end at the next 1024-aligned entry, the range end or the patch entry's end:
        // a chunk never straddles two entries, so only tensors >= 2^32 take the walker
        for (uint64_t c0 = c_first, c_end = 0; c0 < r1; c0 = c_end) {
            while (A.es[e + 1] <= c0) ++e;
            const uint64_t lo = A.es[e], hi = A.es[e + 1];
            c_end = min(min(r1, (c0 / kChunk + 1) * kChunk), hi);
            const uint32_t len = uint32_t(c_end - c0);
            const EntryLayout L = A.el[e];
            if (L.numel >= (1ull << 32)) {
                const SpanState st = slow_span<kRepr, kPass>(A, c0, c0 + len, ar, ac, marker, has_prev, gap_base);
                ar = st.ar;
                ac = st.ac;
                marker = st.marker;
                continue;
            }
            const uint64_t o0 = c0 - lo;
            // ---- stage ----
            if (coo) {
                stage<2>(sa, A.body + L.idx_off + o0, len);
                stage<4>(sb, A.body + L.idx_off + L.count + 2 * o0, 2 * len);
            } else {
                stage<8>(sa, A.body + L.idx_off + 4 * o0, 4 * len);
            }
            if ((kPass == kScatter && !A.out_idx) || kPass == kApply)
                stage<1>(reinterpret_cast<uint4*>(sv), A.body + L.val_off + 2 * o0, 2 * len);
            __syncwarp();
            // ---- this lane's kPer consecutive entries, straight from shared memory ----
            const int nv = max(0, min(int(kPer), int(len) - lane * int(kPer)));
            // packed fields: COO rows 4 per word, columns 2 per word; int32 one per word
            constexpr int kAW = coo ? 8 : 32, kBW = coo ? 16 : 1;
            uint32_t aw[kAW], bw[kBW];
            if (coo) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const uint4 q = lane_vec<2>(sa, i);
                    aw[4 * i] = q.x; aw[4 * i + 1] = q.y; aw[4 * i + 2] = q.z; aw[4 * i + 3] = q.w;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint4 q = lane_vec<4>(sb, i);
                    bw[4 * i] = q.x; bw[4 * i + 1] = q.y; bw[4 * i + 2] = q.z; bw[4 * i + 3] = q.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint4 q = lane_vec<8>(sa, i);
                    aw[4 * i] = q.x; aw[4 * i + 1] = q.y; aw[4 * i + 2] = q.z; aw[4 * i + 3] = q.w;
                }
                bw[0] = 0;
            }
#define PULSE_AV(j) (coo ? (aw[(j) >> 2] >> (8 * ((j) & 3))) & 0xFFu : aw[(j) % kAW])
#define PULSE_BV(j) (coo ? (bw[((j) >> 1) % kBW] >> (16 * ((j) & 1))) & 0xFFFFu : 0u)
            const uint64_t ol = o0 + uint64_t(lane) * kPer;
            const uint64_t nrows = L.numel / (coo && L.cols ? L.cols : 1);  // COO row extent
            const bool lane_first = ol == 0;  // this lane holds the entry's first index (ordinal 0)
            const bool lane_gfirst = c0 + uint64_t(lane) * kPer == 0;  // ... the patch's first entry
            // lane aggregates
            uint64_t lr = 0, lc = 0;
            bool lmark = false;
#pragma unroll
            for (int j = 0; j < int(kPer); ++j) {
                if (j < nv) {
                    const uint32_t a = PULSE_AV(j), b = PULSE_BV(j);
                    const bool first = j == 0 && lane_first;
                    const bool hr = kRepr != kFlat && first;
                    if (coo) {
                        const bool hc = first || a != 0;
                        lmark |= a == 0xFF || b == 0xFFFF;
                        lc = hc ? (H | b) : lc + b;
                    }
                    lr = hr ? (H | a) : lr + a;
                }
            }
            uint64_t ir = lr, ic = lc;
            warp_segscan2(ir, ic);
            const uint64_t tr = __shfl_sync(0xffffffffu, ir, 31), tc = __shfl_sync(0xffffffffu, ic, 31);
            if (kPass == kAgg) {
                marker |= lmark;
                ar = SegSumOp::op(ar, tr);
                ac = SegSumOp::op(ac, tc);
                continue;
            }
            uint64_t er = __shfl_up_sync(0xffffffffu, ir, 1), ec = __shfl_up_sync(0xffffffffu, ic, 1);
            if (lane == 0) er = ec = 0;
            uint64_t row = SegSumOp::op(ar, er) & (H - 1), col = SegSumOp::op(ac, ec) & (H - 1);
            ar = SegSumOp::op(ar, tr) & (H - 1);
            ac = SegSumOp::op(ac, tc) & (H - 1);
#pragma unroll
            for (int i = 0; i < int(kPer) / 4; ++i) {
                uint32_t xv[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int j = 4 * i + c;
                    xv[c] = kInvalid;
                    if (j >= nv) continue;
                    const uint32_t a = PULSE_AV(j), b = PULSE_BV(j);
                    const bool first = j == 0 && lane_first;
#define PULSE_ORD (ol + uint64_t(j))  /* entry ordinal, only for error keys */
                    uint64_t key = kNoError;
                    if (coo) {
                        const bool nr = first || a != 0;
                        row = first ? a : row + a;
                        col = nr ? b : col + b;
                        if (checks(kPass)) {
                            // patch.hpp:247-254; with col < cols, flat >= numel <=> row >= numel / cols
                            if (!nr && b == 0) key = error_key(e, kStageCols, PULSE_ORD, kZeroColGap);
                            else if (col >= L.cols) key = error_key(e, kStageRange, PULSE_ORD, kColRange);
                            else if (row >= nrows) key = error_key(e, kStageRange, PULSE_ORD, kIdxRange);
                        }
                        if (key == kNoError) xv[c] = uint32_t(row) * uint32_t(L.cols) + uint32_t(col);
                    } else if (kRepr == kI32) {
                        row = first ? a : row + a;
                        if (checks(kPass)) {
                            if (!first && a == 0) key = error_key(e, kStageRows, PULSE_ORD, kZeroGap);
                            else if (row >= L.numel) key = error_key(e, kStageRows, PULSE_ORD, kIdxRange);
                        }
                        if (key == kNoError) xv[c] = uint32_t(row);
                    } else {
                        row += a;
                        const int64_t local = int64_t(row) - int64_t(gap_base) - int64_t(L.flat_base);
                        if (checks(kPass)) {
                            // the patch's very first gap may be 0 only without a previous shard
                            const bool gfirst = j == 0 && lane_gfirst;
                            if (a == 0 && (!gfirst || has_prev)) key = error_key(e, kStageRows, PULSE_ORD, kZeroGap);
                            else if (local < 0 || uint64_t(local) >= L.numel) key = error_key(e, kStageRows, PULSE_ORD, kIdxRange);
                        }
                        if (key == kNoError) xv[c] = uint32_t(local);
                    }
#undef PULSE_ORD
                    if (reports(kPass) && key != kNoError) report_cold(A.err, key);
                }
                if (kPass >= kScatter) sx[swz<8>(uint32_t(lane * 8 + i))] = make_uint4(xv[0], xv[1], xv[2], xv[3]);
            }
#undef PULSE_AV
#undef PULSE_BV
            if (kPass < kScatter) continue;
            // ---- indices are in shared memory in entry order: coalesced writes ----
            __syncwarp();
            const uint32_t* xs = reinterpret_cast<const uint32_t*>(sx);
            if (kPass == kScatter && A.out_idx) {
                for (uint32_t k = lane; k < len; k += 32) {
                    const uint32_t q = k >> 2;
                    A.out_idx[c0 + k] = int64_t(xs[swz<8>(q) * 4 + (k & 3)]);
                }
            } else if (kPass == kScatter) {
                uint16_t* W = A.weights[L.tensor];
#pragma unroll 4
                for (uint32_t k = lane; k < len; k += 32) {
                    const uint32_t q = k >> 2;
                    W[xs[swz<8>(q) * 4 + (k & 3)]] = sv[k];
                }
            } else if (kPass == kApply) {
                // all of this lane's backup reads in flight at once, then the writes
                uint16_t* W = A.weights[L.tensor];
                uint16_t* bk = A.backup + c0;
                uint32_t xk[kPer];
                uint16_t old[kPer];
#pragma unroll
                for (int t = 0; t < int(kPer); ++t) {
                    const uint32_t k = uint32_t(lane) + 32u * t;
                    xk[t] = k < len ? xs[swz<8>(k >> 2) * 4 + (k & 3)] : kInvalid;
                    old[t] = xk[t] != kInvalid ? W[xk[t]] : uint16_t(0);
                }
#pragma unroll
                for (int t = 0; t < int(kPer); ++t) {
                    const uint32_t k = uint32_t(lane) + 32u * t;
                    if (xk[t] != kInvalid) {
                        bk[k] = old[t];
                        W[xk[t]] = sv[k];
                    }
                }
            } else {  // kRestore
                uint16_t* W = A.weights[L.tensor];
                const uint16_t* bk = A.backup + c0;
                for (uint32_t k = lane; k < len; k += 32) {
                    const uint32_t x = xs[swz<8>(k >> 2) * 4 + (k & 3)];
                    if (x != kInvalid) W[x] = bk[k];
                }
            }
            __syncwarp();
        }
        if (kPass == kAgg) {
            if (__any_sync(0xffffffffu, marker) && lane == 0) atomicExch(A.flags, 1u);
            if (lane == 0) A.agg[rg] = make_ulonglong2(ar, ac);
        }
    }
}

// =============================================================================================
// Streaming passes over fixed-layout payloads: F1s f_stream<agg> and F5 f_stream<scatter>
// =============================================================================================
// F1s (aggregates + checks) and F5 (the in-place scatter of a patch that has
// passed every check) share one skeleton, leaner and latency-hidden next to F1/F3:
//  * 512-entry chunks, 16 consecutive entries per lane; three CTAs per SM;
//  * the next chunk's rows / columns / u32 gaps (/ values) are in flight
//    (cp.async of the 16-byte blocks covering them, double-buffered) while the
//    current one decodes; the payload's byte alignment is removed on the
//    shared-memory read (funnel shifts), not through registers;
//  * per-lane running values in 32 bits where they fit (COO rows / columns);
//  * each range's patch entry: a warp search in F1s (two dependent loads for a
//    few hundred entries), recorded for F3 / F5 (one load per range).
//
// Checks without the carry.  Inside a range that holds no patch-entry start or
// end ("plain" range) every reference check but one is local or monotone:
//   zero gaps (patch.hpp:201-203, 225-227; index_coding.hpp:147-149) -- local;
//   rows / int32 indices / FLAT positions (patch.hpp:206-208, 231-233, 252-254)
//     -- non-decreasing within an entry, so bounded by the entry's first and
//     last entries, which lie in non-plain ranges;
//   COO columns (patch.hpp:247-250) -- increasing within a row: a column is
//     known exactly once a row starts inside the range (checked here); the
//     range's first row segment ends at carry + P, checked by F2 once the
//     carry is known (`slack` = cols - 1 - P).
// Non-plain ranges (and every range, once anything looked wrong) go through the
// exact F3 checks (f_pass<validate>), which also pin the reference's first
// failing entry; F5 runs only if nothing failed.
constexpr uint64_t kNoSlack = ~0ull;

// Per-warp staging of F1s (1024-entry chunks: more bytes in flight per warp for
// a pass that only reads) and F5 (512-entry chunks, values and decoded indices
// too).  Lane l reads its fields as slots [P*l, P*l + P] of a buffer swizzled
// with V = P (P = 16-byte slots per lane).
template <int kRepr, bool kAgg_>
struct SLay {
    static constexpr bool coo = kRepr == kCoo;
    static constexpr uint32_t ch = kAgg_ ? 1024 : 512;                        // entries per chunk
    static constexpr uint32_t per = ch / 32;                                  // entries per lane
    static constexpr uint32_t va = coo ? per / 16 : per / 4;                  // rows | u32 gaps
    static constexpr uint32_t vb = per / 8;                                   // columns
    static constexpr uint32_t a_slots = 32 * va + 1;
    static constexpr uint32_t b_slots = coo ? 32 * vb + 1 : 0;
    static constexpr uint32_t v_slots = kAgg_ ? 0 : 2 * ch / 16 + 1;          // values (V=2)
    static constexpr uint32_t buf = 16 * (a_slots + b_slots + v_slots);
    static constexpr uint32_t warp = 2 * buf + (kAgg_ ? 0 : 8 * ch);          // 2 buffers (+ (index, value) pairs)
};


// Queues the 16-byte blocks covering [g, g+len) into dst (swizzle V); returns g & 15.
template <int V>
__device__ __forceinline__ uint32_t stage_cover(uint4* dst, const uint8_t* g, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uintptr_t ga = reinterpret_cast<uintptr_t>(g);
    const uint32_t s = uint32_t(ga & 15);
    const uint8_t* base = reinterpret_cast<const uint8_t*>(ga - s);
    const uint32_t nslots = len ? (s + len + 15) >> 4 : 0;
    const uint32_t sdst = smem_u32(dst);
    for (uint32_t q = lane; q < nslots; q += 32) cp_async16_s(sdst + 16 * swz<V>(q), base + 16 * q);
    return s;
}

// 16 payload bytes starting at byte s + 16*k of a staged buffer (slots k, k+1).
template <int V>
__device__ __forceinline__ uint4 staged16(const uint4* buf, uint32_t k, uint32_t s) {
    const uint4 lo = lds128(buf + swz<V>(k));
    if (s == 0) return lo;
    const uint4 hi = lds128(buf + swz<V>(k + 1));
    return funnel16(lo, hi, s >> 2, (s & 3) * 8);
}

struct SCtx {
    uint32_t e;
    uint32_t tensor;
    uint64_t lo, hi;  // entries [lo, hi) belong to patch entry e
    const uint8_t* rows;  // body + idx_off: COO row bytes / u32 gaps
    const uint8_t* colp;  // COO column units (body + idx_off + count)
    const uint8_t* vals;  // body + val_off
    uint64_t numel, cols, flat_base;
};

__device__ __forceinline__ void load_sctx(SCtx& c, const ApplyArgs& A, uint32_t e) {
    c.e = e;
    c.lo = A.es[e];
    c.hi = A.es[e + 1];
    const EntryLayout& L = A.el[e];
    c.tensor = uint32_t(L.tensor);
    c.rows = A.body + L.idx_off;
    c.colp = A.body + L.idx_off + L.count;
    c.vals = A.body + L.val_off;
    c.numel = L.numel;
    c.cols = L.cols;
    c.flat_base = L.flat_base;
}


// One staged fast chunk of f_stream: lane aggregates + warp scan, then either
// the carry-free checks (F1s) or the decode + scatter (F5).  Branch-free per
// entry; kFull (every chunk but a range's last) drops the tail guards.
template <int kRepr, bool kAgg_, bool kFull>
__device__ __forceinline__ void chunk_body(const ApplyArgs& A, const SCtx& cur, uint64_t c0, uint32_t len, uint64_t r0,
                                           const uint8_t* bb, uint32_t* sx, const uint32_t* sh, bool has_prev,
                                           uint64_t gap_base, uint64_t& ar, uint64_t& ac, bool& suspect,
                                           bool& marker, uint64_t& slack) {
    using Y = SLay<kRepr, kAgg_>;
    constexpr bool coo = kRepr == kCoo;
    constexpr int kPer = int(Y::per);
    const int lane = threadIdx.x & 31;
    const uint4* sa = reinterpret_cast<const uint4*>(bb);
    const uint4* sb = reinterpret_cast<const uint4*>(bb + 16 * Y::a_slots);
    const uint64_t o0 = c0 - cur.lo;
    const int nv = kFull ? kPer : max(0, min(kPer, int(len) - lane * kPer));
    const uint64_t i0 = c0 + uint64_t(lane) * kPer;  // global ordinal of the lane's first entry
    const bool lane_first = o0 + uint64_t(lane) * kPer == 0;
    // this lane's fields: COO rows (4 per word) + columns (2 per word); int32: u32 gaps
    constexpr int kAW = coo ? kPer / 4 : kPer, kBW = coo ? kPer / 2 : 1;
    uint32_t aw[kAW], bw[kBW];
#pragma unroll
    for (int i = 0; i < int(Y::va); ++i) {
        const uint4 q = staged16<Y::va>(sa, uint32_t(Y::va * lane + i), sh[0]);
        aw[4 * i] = q.x; aw[4 * i + 1] = q.y; aw[4 * i + 2] = q.z; aw[4 * i + 3] = q.w;
    }
    if (coo) {
#pragma unroll
        for (int i = 0; i < int(Y::vb); ++i) {
            const uint4 q = staged16<Y::vb>(sb, uint32_t(Y::vb * lane + i), sh[1]);
            bw[(4 * i) % kBW] = q.x; bw[(4 * i + 1) % kBW] = q.y; bw[(4 * i + 2) % kBW] = q.z; bw[(4 * i + 3) % kBW] = q.w;
        }
    } else {
        bw[0] = 0;
    }
    if (!kFull) {  // entries past the chunk read as (0, 0) and are never heads
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (j >= nv) {
                if (coo) {
                    aw[(j >> 2) % kAW] &= ~(0xFFu << (8 * (j & 3)));
                    bw[(j >> 1) % kBW] &= ~(0xFFFFu << (16 * (j & 1)));
                } else {
                    aw[j % kAW] = 0;
                }
            }
        }
    }
#define PULSE_SA(j) (coo ? (aw[((j) >> 2) % kAW] >> (8 * ((j) & 3))) & 0xFFu : aw[(j) % kAW])
#define PULSE_SB(j) (coo ? (bw[((j) >> 1) % kBW] >> (16 * ((j) & 1))) & 0xFFFFu : 0u)
    // ---- lane aggregates (+ the carry-free checks of F1s) ----
    uint64_t lr, lc = 0;
    bool bad = false, mk = false, head0 = lane_first;
    uint32_t P = 0;  // COO: column sum of the lane's entries before its first row start
    bool hc = false;
    if (coo) {
        uint32_t rs = 0;
#pragma unroll
        for (int w = 0; w < kAW; ++w) {
            rs = __dp4a(aw[w], 0x01010101u, rs);
            if (kAgg_) mk |= ((~aw[w] - 0x01010101u) & aw[w] & 0x80808080u) != 0;  // a 0xFF row byte
        }
        if (kAgg_) {
#pragma unroll
            for (int w = 0; w < kBW; ++w) mk |= ((~bw[w] - 0x00010001u) & bw[w] & 0x80008000u) != 0;  // 0xFFFF
        }
        uint32_t c = 0, cmax = 0;
        bool zero = false;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t a = PULSE_SA(j), bv = PULSE_SB(j);
            const bool nr = a != 0 || (j == 0 && lane_first);
            if (j == 0) head0 = nr;
            if (kAgg_) {
                zero |= !nr && bv == 0 && (kFull || j < nv);  // zero column gap within a row
                if (nr && !hc) P = c;  // the lane's first row start: P = the column sum before it
            }
            c = nr ? bv : c + bv;
            hc |= nr;
            if (kAgg_ && hc) cmax = max(cmax, c);  // rows that start in this lane: columns known
        }
        if (kAgg_) bad |= zero || cmax >= uint32_t(cur.cols);
        lr = uint64_t(rs) | (lane_first ? H : 0);
        lc = uint64_t(c) | (hc ? H : 0);
    } else {
        uint64_t r = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t a = PULSE_SA(j);
            r += a;
            if (kAgg_) {
                if (kRepr == kI32) bad |= a == 0 && !(j == 0 && lane_first) && (kFull || j < nv);
                else bad |= a == 0 && (i0 + j > 0 || has_prev) && (kFull || j < nv);
            }
        }
        lr = r | (kRepr == kI32 && lane_first ? H : 0);
    }
    uint64_t tr, tc, er, ec;
    if (coo) {
        // COO lane aggregates fit 31 bits (<= 32 row bytes, <= 32 u16 columns per lane; <= 32 lanes):
        // the warp scan runs on 32-bit words with the segment head in bit 31
        uint32_t r = uint32_t(lr) | (lr & H ? 0x80000000u : 0u), cc = uint32_t(lc) | (lc & H ? 0x80000000u : 0u);
        warp_segscan2_32(r, cc);
        const uint32_t t_r = __shfl_sync(0xffffffffu, r, 31), t_c = __shfl_sync(0xffffffffu, cc, 31);
        uint32_t e_r = __shfl_up_sync(0xffffffffu, r, 1), e_c = __shfl_up_sync(0xffffffffu, cc, 1);
        if (lane == 0) e_r = e_c = 0;
        auto widen = [](uint32_t x) { return uint64_t(x & 0x7FFFFFFFu) | (x >> 31 ? H : 0); };
        tr = widen(t_r);
        tc = widen(t_c);
        er = widen(e_r);
        ec = widen(e_c);
    } else {
        uint64_t ir = lr, ic = lc;
        warp_segscan2(ir, ic);
        tr = __shfl_sync(0xffffffffu, ir, 31);
        tc = __shfl_sync(0xffffffffu, ic, 31);
        er = __shfl_up_sync(0xffffffffu, ir, 1);
        ec = __shfl_up_sync(0xffffffffu, ic, 1);
        if (lane == 0) er = ec = 0;
    }
    if (kAgg_) {
        uint64_t pend = kNoSlack;
        if (coo && hc && !lane_first) {
            // the lane's first row segment ends in this lane, at column (state at lane start) + P
            // (not when the lane starts a patch entry: the segment before is the previous
            // entry's, whose end lies in this non-plain range and gets the exact checks)
            const uint64_t cs = SegSumOp::op(ac, ec);
            const uint64_t end = (cs & (H - 1)) + P;
            if (cs & H) bad |= end >= cur.cols;              // a row started earlier in the range: exact
            else if (i0 > r0 || !head0) pend = end;           // the range's first row segment: carry needed
        }
        suspect |= __any_sync(0xffffffffu, bad);
        marker |= __any_sync(0xffffffffu, mk);
        if (coo) {
            const uint32_t who = __ballot_sync(0xffffffffu, pend != kNoSlack);
            if (who) {  // at most one lane per range: the first row start after its first entry
                const uint64_t p = __shfl_sync(0xffffffffu, pend, __ffs(who) - 1);
                if (p >= cur.cols) suspect = true;
                else slack = cur.cols - 1 - p;
            }
        }
        ar = SegSumOp::op(ar, tr);
        ac = SegSumOp::op(ac, tc);
        return;
    }
    // ---- F5: decode into shared memory (lane-consecutive, swizzled), then scatter ----
    uint64_t row = SegSumOp::op(ar, er) & (H - 1);
    const uint64_t col = SegSumOp::op(ac, ec) & (H - 1);
    ar = SegSumOp::op(ar, tr) & (H - 1);
    ac = SegSumOp::op(ac, tc) & (H - 1);
    const uint32_t cols32 = uint32_t(cur.cols);
    uint32_t r32 = uint32_t(row), c32 = uint32_t(col);
    const uint64_t flat_off = gap_base + cur.flat_base;
    // this lane's 16 values: two funnel-aligned 16-byte reads of the staged value blob
    const uint4* svb = reinterpret_cast<const uint4*>(bb + 16 * (Y::a_slots + Y::b_slots));
    const uint4 v0 = staged16<2>(svb, uint32_t(2 * lane), sh[2]);
    const uint4 v1 = staged16<2>(svb, uint32_t(2 * lane + 1), sh[2]);
    const uint32_t vw[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint32_t xv[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t a = PULSE_SA(j), bv = PULSE_SB(j);
        const bool first = j == 0 && lane_first;
        if (coo) {
            r32 = first ? a : r32 + a;
            c32 = (first || a != 0) ? bv : c32 + bv;
            xv[j] = r32 * cols32 + c32;
        } else if (kRepr == kI32) {
            r32 = first ? a : r32 + a;
            xv[j] = r32;
        } else {
            row += a;
            xv[j] = uint32_t(row - flat_off);
        }
    }
    // (index, value) pairs, lane-consecutive, two per 16-byte slot (swizzled: conflict-free both ways)
    uint4* sp = reinterpret_cast<uint4*>(sx);
#pragma unroll
    for (int i = 0; i < kPer / 2; ++i)
        sp[swz<8>(uint32_t(lane * (kPer / 2) + i))] =
            make_uint4(xv[2 * i], vw[i] & 0xFFFFu, xv[2 * i + 1], vw[i] >> 16);
#undef PULSE_SA
#undef PULSE_SB
    __syncwarp();
    uint16_t* W = A.weights[cur.tensor];
#if PULSE_F5_NATURAL
    // scatter in entry order: each store instruction covers 32 consecutive changes
    const uint2* sp2 = reinterpret_cast<const uint2*>(sp);
#pragma unroll 4
    for (uint32_t k = lane; k < len; k += 32) {
        const uint2 q = sp2[2 * swz<8>(k >> 1) + (k & 1)];
        W[q.x] = uint16_t(q.y);
    }
#else
    // scatter: each store instruction covers 32 of 64 consecutive changes (a few sectors)
    const uint32_t npairs = (len + 1) / 2;
#pragma unroll 4
    for (uint32_t k2 = lane; k2 < npairs; k2 += 32) {
        const uint4 q = lds128(sp + swz<8>(k2));
        W[q.x] = uint16_t(q.y);
        if (2 * k2 + 1 < len) W[q.z] = uint16_t(q.w);
    }
#endif
}

// F5 resident CTAs per SM (the COO scatter spills ~170 B at 3; 2 measured ~0.5% faster at 7B)
#ifndef PULSE_F5_MINB
#define PULSE_F5_MINB 3
#endif

#ifndef PULSE_F1_MINB
#define PULSE_F1_MINB 3
#endif
template <int kRepr, bool kAgg_>
__global__ void __launch_bounds__(kThreads, kAgg_ ? PULSE_F1_MINB : PULSE_F5_MINB) f_stream(ApplyArgs A) {
    extern __shared__ __align__(16) uint8_t smem[];
    using Y = SLay<kRepr, kAgg_>;
    constexpr bool coo = kRepr == kCoo;
    constexpr bool agg = kAgg_;
    constexpr uint32_t kSChunk = Y::ch;
    if (fast_blocked(A.flags)) return;
    if (!agg && *(volatile const uint64_t*)A.err != kNoError) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* ws = smem + warp * Y::warp;
    uint32_t* sx = reinterpret_cast<uint32_t*>(ws + 2 * Y::buf);

    const uint64_t n = A.totals[0];
    const uint32_t kRange = apply_range(n);
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
    const bool has_prev = A.carry && A.carry->has_prev;
    const uint64_t gap_base = has_prev ? A.carry->gap_base : 0;
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;

    if (agg) {  // F2's look-back words start cleared (no memset node ahead of F2)
        for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < 2ull * A.scan_blocks;
             i += uint64_t(gridDim.x) * blockDim.x)
            A.scan_status[i] = 0;
    }
    // F1s finds each range's patch entry (a warp search) and records it for F3 / F5
    auto range_entry = [&](uint64_t r) -> uint32_t {
        if (!agg) return A.range_e[r];
        const uint32_t e = warp_upper_index(A.es, A.n_e, r * kRange);
        if ((threadIdx.x & 31) == 0) A.range_e[r] = e;
        return e;
    };
    uint64_t rg = uint64_t(blockIdx.x) * kWarps + warp;
    if (rg >= n_ranges) return;
    uint64_t c0 = rg * kRange;
    SCtx cur;
    load_sctx(cur, A, range_entry(rg));
    auto range_end = [&](uint64_t r) { return min(r * kRange + kRange, n); };
    // chunks end at the next kSChunk-aligned entry, the range end or the patch entry's
    // end: a chunk never straddles two entries, so only tensors >= 2^32 take the walker
    auto chunk_len = [&](uint64_t r, uint64_t c, const SCtx& cx) {
        return uint32_t(min(min(range_end(r), (c / kSChunk + 1) * kSChunk), cx.hi) - c);
    };
    auto is_fast = [&](const SCtx& c, uint64_t cc, uint32_t len) {
        return c.hi >= cc + len && c.numel < (1ull << 32);
    };
    // always commits one cp.async group (possibly empty): the wait<1> below then
    // always means "everything but the chunk after this one"
    auto prefetch = [&](bool any, const SCtx& c, uint64_t cc, uint32_t len, uint32_t b, uint32_t* sh) {
        if (any && is_fast(c, cc, len)) {
            uint8_t* bb = ws + b * Y::buf;
            const uint64_t o0 = cc - c.lo;
            if (coo) {
                sh[0] = stage_cover<Y::va>(reinterpret_cast<uint4*>(bb), c.rows + o0, len);
                sh[1] = stage_cover<Y::vb>(reinterpret_cast<uint4*>(bb + 16 * Y::a_slots), c.colp + 2 * o0, 2 * len);
            } else {
                sh[0] = stage_cover<Y::va>(reinterpret_cast<uint4*>(bb), c.rows + 4 * o0, 4 * len);
            }
            if (!agg)
                sh[2] = stage_cover<2>(reinterpret_cast<uint4*>(bb + 16 * (Y::a_slots + Y::b_slots)), c.vals + 2 * o0,
                                       2 * len);
        }
        cp_async_commit();
    };
    // range state (F1s): plain range?, first-row-segment slack, anything wrong, escape markers
    bool plain = false, suspect = false, marker = false;
    uint64_t slack = kNoSlack;
    auto range_begin = [&](uint64_t r, const SCtx& c) {
        plain = c.lo < r * kRange && c.hi > range_end(r) && c.numel < (1ull << 32);
        slack = kNoSlack;
    };
    uint32_t len = chunk_len(rg, c0, cur);
    uint32_t sh_cur[3] = {0, 0, 0}, sh_nx[3] = {0, 0, 0};
    uint32_t b = 0;
    prefetch(true, cur, c0, len, 0, sh_cur);
    uint64_t ar = 0, ac = 0;
    if (agg) {
        range_begin(rg, cur);
    } else {
        const ulonglong2 p = A.agg[rg];
        ar = p.x;
        ac = p.y;
    }
    while (true) {
        // ---- the next chunk: position and entry context (loads overlap the wait below) ----
        uint64_t rg_nx = rg, c_nx = c0 + len;
        if (c_nx >= range_end(rg)) {
            rg_nx = rg + stride;
            c_nx = rg_nx * kRange;
        }
        const bool has_nx = rg_nx < n_ranges;
        SCtx nx = cur;
        uint32_t len_nx = 0;
        ulonglong2 carry_nx = make_ulonglong2(0, 0);
        if (has_nx) {
            if (rg_nx != rg) {
                if (!agg) carry_nx = A.agg[rg_nx];
                load_sctx(nx, A, range_entry(rg_nx));
            } else if (c_nx >= cur.hi) {
                uint32_t e = cur.e + 1;
                while (A.es[e + 1] <= c_nx) ++e;
                load_sctx(nx, A, e);
            }
            len_nx = chunk_len(rg_nx, c_nx, nx);
        }
        if (agg && !plain) {  // this chunk gets F3's exact checks: list it with its in-range carry
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(A.n_pieces, 1ull);
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if (slot < A.piece_cap) {
                if (lane == 0) A.pieces[slot] = ApplyArgs::Piece{c0, rg, ar, ac, len, cur.e};
            } else {
                suspect = true;  // list full: every range gets the exact checks
            }
        }
        if (!is_fast(cur, c0, len)) {
            // straddles patch entries or a tensor >= 2^32 elements: per-round walker (never plain)
            const SpanState st =
                slow_span<kRepr, agg ? kAgg : kScatter>(A, c0, c0 + len, ar, ac, marker, has_prev, gap_base);
            ar = st.ar;
            ac = st.ac;
            marker = st.marker;
            prefetch(has_nx, nx, c_nx, len_nx, b ^ 1, sh_nx);
        } else {
            prefetch(has_nx, nx, c_nx, len_nx, b ^ 1, sh_nx);
            cp_async_wait<1>();
            __syncwarp();
            const uint8_t* bb = ws + b * Y::buf;
            if (len == kSChunk)
                chunk_body<kRepr, agg, true>(A, cur, c0, len, rg * kRange, bb, sx, sh_cur, has_prev, gap_base, ar, ac,
                                             suspect, marker, slack);
            else
                chunk_body<kRepr, agg, false>(A, cur, c0, len, rg * kRange, bb, sx, sh_cur, has_prev, gap_base, ar,
                                              ac, suspect, marker, slack);
            __syncwarp();
        }
        const bool range_done = !has_nx || rg_nx != rg;
        if (agg && range_done) {
            if (lane == 0) {
                A.agg[rg] = make_ulonglong2(ar, ac);
                A.slack[rg] = plain ? slack : kNoSlack;
            }
            if (marker && lane == 0) atomicExch(A.flags, 1u);
            if (suspect && lane == 0) atomicExch(A.flags + 1, 1u);
            marker = suspect = false;
        }
        if (!has_nx) break;
        if (rg_nx != rg) {
            if (agg) {
                ar = ac = 0;
                range_begin(rg_nx, nx);
            } else {
                ar = carry_nx.x;
                ac = carry_nx.y;
            }
        }
        rg = rg_nx;
        c0 = c_nx;
        len = len_nx;
        cur = nx;
        sh_cur[0] = sh_nx[0];
        sh_cur[1] = sh_nx[1];
        sh_cur[2] = sh_nx[2];
        b ^= 1;
    }
    cp_async_wait<0>();
}

// =============================================================================================
// F2: exclusive SegSum scan of the range aggregates (one CTA of 1024)
// =============================================================================================
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 4;  // items per thread

// One 1024-thread CTA per block of 4096 range aggregates, blocks taken in ticket
// order and chained by a decoupled look-back (one status word per block and
// stream) -- the scan is spread over several SMs instead of serialising ~18K
// 64-bit segmented adds on one.
constexpr uint64_t kScanBlock = uint64_t(kScanThreads) * kScanPer;

__global__ void __launch_bounds__(kScanThreads, 1)
f_range_scan(const uint64_t* __restrict__ totals, ulonglong2* __restrict__ agg, uint32_t* __restrict__ flags,
             uint64_t* __restrict__ status, unsigned long long* __restrict__ ticket,
             const uint64_t* __restrict__ slack) {
    __shared__ uint64_t s_scan[33 * 2];
    __shared__ uint64_t s_blk, s_pre[2];
    if (fast_blocked(flags)) return;
    const uint64_t n = totals[0];
    const uint64_t n_ranges = (n + apply_range(n) - 1) / apply_range(n);
    const uint64_t n_blocks = (n_ranges + kScanBlock - 1) / kScanBlock;
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1ull);
    __syncthreads();
    const uint64_t blk = s_blk;
    if (blk >= n_blocks) return;
    const uint64_t q0 = blk * kScanBlock + uint64_t(threadIdx.x) * kScanPer;
    ulonglong2 v[kScanPer];
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) v[j] = q0 + j < n_ranges ? agg[q0 + j] : make_ulonglong2(0, 0);
    uint64_t ar = 0, ac = 0;  // this thread's aggregate
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {
        ar = SegSumOp::op(ar, v[j].x);
        ac = SegSumOp::op(ac, v[j].y);
    }
    uint64_t ex[2] = {ar, ac}, tot[2];
    cta_exclusive_scan<2, kScanThreads, AllSegSum>(ex, tot, s_scan);  // -> exclusive within the block
    const uint64_t er = ex[0], ec = ex[1];
    if (threadIdx.x < 32) {  // warp 0: the block's exclusive prefix for both streams
        const uint64_t pr = lookback<SegSumOp>(status, blk, tot[0]);
        const uint64_t pc = lookback<SegSumOp>(status + n_blocks, blk, tot[1]);
        if (threadIdx.x == 0) {
            s_pre[0] = pr;
            s_pre[1] = pc;
        }
    }
    __syncthreads();
    uint64_t sr = SegSumOp::op(s_pre[0], er), sc = SegSumOp::op(s_pre[1], ec);
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {  // in place: aggregate -> exclusive prefix
        if (q0 + j < n_ranges) {
            agg[q0 + j] = make_ulonglong2(sr & (H - 1), sc & (H - 1));
            // F1s deferred check: the range's first row segment ends at carry + P < cols
            if (slack && (sc & (H - 1)) > slack[q0 + j]) atomicExch(flags + 1, 1u);
        }
        sr = SegSumOp::op(sr, v[j].x);
        sc = SegSumOp::op(sc, v[j].y);
    }
}

// =============================================================================================
// launcher (called from launch_decode after d_layout)
// =============================================================================================
namespace {
template <int kRepr, int kPass>
void launch_pass(const ApplyArgs& a, cudaStream_t s) {
    const uint32_t smem = kWarps * warp_smem(kPass);
    static PerDeviceInt occ;  // per instantiation and device: resident CTAs per SM (persistent grid)
    int& per_sm = occ.here();
    if (!per_sm) {
        cudaFuncSetAttribute(f_pass<kRepr, kPass>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int v = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, f_pass<kRepr, kPass>, kThreads, smem);
        per_sm = v > 0 ? v : 1;
    }
    // F3 (validate) walks a short list of pieces (or, rarely, every range): PULSE_F3_CTAS_PER_SM
    // caps its grid below full occupancy (fewer idle CTAs to schedule for small patches)
    const int cap = kPass == kValidate ? PULSE_F3_CTAS_PER_SM : per_sm;
    f_pass<kRepr, kPass><<<unsigned(sm_count() * (per_sm < cap ? per_sm : cap)), kThreads, smem, s>>>(a);
    PULSE_LAUNCHED("f_pass", s);
}

template <int kRepr, bool kAgg_>
void launch_stream(const ApplyArgs& a, cudaStream_t s) {
    const uint32_t smem = kWarps * SLay<kRepr, kAgg_>::warp;
    static PerDeviceInt occ;
    int& per_sm = occ.here();
    if (!per_sm) {
        cudaFuncSetAttribute(f_stream<kRepr, kAgg_>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int v = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, f_stream<kRepr, kAgg_>, kThreads, smem);
        per_sm = v > 0 ? v : 1;
    }
    f_stream<kRepr, kAgg_><<<unsigned(sm_count() * per_sm), kThreads, smem, s>>>(a);
    PULSE_LAUNCHED(kAgg_ ? "f_stream<agg>" : "f_stream<scatter>", s);
}

void launch_range_scan(const ApplyArgs& a, const uint64_t* slack, cudaStream_t s) {
    cudaMemsetAsync(a.scan_status, 0, 2 * sizeof(uint64_t) * a.scan_blocks, s);
    f_range_scan<<<a.scan_blocks, kScanThreads, 0, s>>>(a.totals, a.agg, a.flags, a.scan_status, a.scan_ticket,
                                                        slack);
    PULSE_LAUNCHED("f_range_scan", s);
}

template <int kRepr>
void launch_all(const ApplyArgs& a, bool scatter, cudaStream_t s) {
    // PULSE_APPLY_MODE (A/B experiments): 1 = F1 + checked scatter with backup and restore;
    // 2 = F1 + exact validation of every range + F3 scatter; default: the pipeline below
    static const int mode = getenv("PULSE_APPLY_MODE") ? atoi(getenv("PULSE_APPLY_MODE")) : 0;
    if (mode == 1 || mode == 2) {
        ApplyArgs b = a;
        b.checked = false;
        launch_pass<kRepr, kAgg>(b, s);
        launch_range_scan(b, nullptr, s);
        if (b.weights && mode == 1) {
            launch_pass<kRepr, kApply>(b, s);
            launch_pass<kRepr, kRestore>(b, s);
        } else {
            launch_pass<kRepr, kValidate>(b, s);
            if (scatter) launch_pass<kRepr, kScatter>(b, s);
        }
        return;
    }
    // F1s aggregates + carry-free checks + range entries -> F2 scan (+ deferred column
    // check) -> F3 exact checks where F1s could not decide (twice: the second only re-checks
    // everything if the first found a failure, to report the reference's first one) -> F5 scatter
    launch_stream<kRepr, true>(a, s);  // F1s (F0 folded in; it also clears F2's look-back words)
    f_range_scan<<<a.scan_blocks, kScanThreads, 0, s>>>(a.totals, a.agg, a.flags, a.scan_status, a.scan_ticket,
                                                        a.slack);
    PULSE_LAUNCHED("f_range_scan", s);
    ApplyArgs v = a;
    v.vmode = 0;
    launch_pass<kRepr, kValidate>(v, s);
    v.vmode = 1;
    launch_gated_on_error(s, a.err, [&](cudaStream_t gs) { launch_pass<kRepr, kValidate>(v, gs); });
    if (scatter && a.weights) launch_stream<kRepr, false>(a, s);
    else if (scatter) launch_pass<kRepr, kScatter>(a, s);
}
}  // namespace

void launch_apply_fast(const PlanDev& p, uint32_t repr, const uint8_t* body, uint32_t n_entries,
                       const pulse_flat_carry* carry, int weights_slot, int64_t* out_indices, uint32_t* flags,
                       cudaStream_t s) {
    ApplyArgs a;
    a.el = p.elay;
    a.es = p.d_es;
    a.n_e = n_entries;
    a.body = body;
    a.carry = carry;
    a.totals = p.d_totals;
    a.agg = reinterpret_cast<ulonglong2*>(p.flat);  // flat scratch is free on this path
    a.flags = flags;
    a.err = p.err;
    a.weights = weights_slot >= 0 ? p.slot[weights_slot] : nullptr;
    a.out_idx = out_indices;
    a.backup = reinterpret_cast<uint16_t*>(p.rowgap);  // general-decoder scratch, idle on this path
    a.scan_status = p.d_status;  // general-decoder look-back words, idle on this path
    a.scan_ticket = reinterpret_cast<unsigned long long*>(p.d_totals + 15);  // zeroed by decode_prologue
    a.scan_blocks = uint32_t((p.cap / kRangeMin + 2 + kScanBlock - 1) / kScanBlock);
    // general-decoder scratch, idle on this path: colent [cap] u32 >= 2 x ranges, rowgap
    // [cap] u32 >= 2 x ranges u64 (the legacy backup of PULSE_APPLY_MODE=1 uses rowgap instead)
    const uint64_t n_rg = p.cap / kRangeMin + 2;
    a.range_e = p.colent;
    a.checked = true;
    // flat scratch [cap] u64: range aggregates, then the piece list
    a.pieces = reinterpret_cast<ApplyArgs::Piece*>(a.agg + n_rg);
    a.piece_cap = (8 * p.cap - 16 * n_rg) / sizeof(ApplyArgs::Piece);
    a.n_pieces = reinterpret_cast<unsigned long long*>(p.d_totals + 13);  // zeroed by decode_prologue
    a.slack = reinterpret_cast<uint64_t*>(p.rowgap);
    a.vmode = 0;
    if (out_indices) a.weights = nullptr;
    const bool scatter = weights_slot >= 0 || out_indices;
    if (repr == PULSE_COO_DOWNSCALED) launch_all<kCoo>(a, scatter, s);
    else if (repr == PULSE_COO_INT32) launch_all<kI32>(a, scatter, s);
    else launch_all<kFlat>(a, scatter, s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_apply)

}  // namespace dev
}  // namespace pulse
