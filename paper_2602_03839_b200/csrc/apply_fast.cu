// PULSE apply, fixed-layout fast path (sm_100a).
//
// When no entry of a patch needs an escape -- COO_DOWNSCALED payloads with
// idx_nbytes == 3 * count and no 0xFF row byte / 0xFFFF column unit, or any
// COO_INT32 / FLAT_INT32 payload (always 4 bytes per entry) -- entry o of a
// tensor has its row gap at byte o, its column entry at byte count + 2o (or its
// u32 gap at byte 4o) of the index payload (index_coding.hpp:104-127,
// patch.hpp:120-156).  Decoding is then a pair of segmented prefix sums over
// the entries, read straight from the body:
//
//   F1 f_agg<0>      per warp range of 4096 entries: segmented-sum aggregates
//                    (rows: restart at each tensor; columns: restart at each new
//                    row, index_coding.hpp:141-153); flags escape markers.
//   F2 f_range_scan  one CTA: exclusive scan of the range aggregates.
//   F3 f_pass<apply> recompute every (row, col) / index, apply the reference
//                    checks (zero gap, column range, index range) and, for each
//                    entry that passes, save W[flat] to a backup and write the
//                    value -- an entry that fails is never written.
//   F4 f_pass<restore> only if some check failed anywhere: recompute and put the
//                    backed-up values back, so a bad patch never half-applies
//                    (the reference validates on a copy, patch.hpp:311).
//   (decode-only callers -- int64 indices out -- run validate, then scatter.)
//
// Data movement.  A warp works on 1024-entry chunks.  It stages a chunk's row
// bytes / column units / u32 gaps (and, for F4, its values) from the body into
// its own shared memory with coalesced 16-byte loads, funnel-shifting the
// arbitrary byte alignment of the payload away; each lane then decodes 32
// CONSECUTIVE entries serially from shared memory (one warp segmented scan per
// chunk, not per 32 entries).  Shared-memory vectors are XOR-swizzled so both
// the staging stores and the per-lane 16-byte reads are bank-conflict free.
// F4 transposes the decoded indices back to entry order through shared memory
// so each warp store instruction covers 32 consecutive changes (a few sectors
// for clustered updates) rather than 32 scattered ones.
//
// A chunk that straddles two patch entries (at most one per changed tensor) or
// a tensor with >= 2^32 elements takes the per-round walker path instead.
//
// If d_layout or F1 finds anything the fixed layout cannot express (escapes,
// short/long payloads, marker bytes), `flags[0]` routes the patch to the
// general parser in decode.cu instead; every kernel checks it on entry.
#include <cstdlib>

#include "device.cuh"
#include "internal.hpp"
#include "stage.cuh"

namespace pulse {
namespace dev {

namespace {

constexpr uint32_t kRange = 4096;  // entries per warp range (aggregate granularity)
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
};

// Walker path over entries [first, last) for one pass.  (ar, ac): aggregates
// (kAgg) or running values (validate / scatter); updated in place.
template <int kRepr, int kPass>
__device__ __noinline__ void slow_span(const ApplyArgs& A, uint64_t first, uint64_t last, uint64_t& ar, uint64_t& ac,
                                       bool& marker, bool has_prev, uint64_t gap_base) {
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
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
    const bool has_prev = A.carry && A.carry->has_prev;
    const uint64_t gap_base = has_prev ? A.carry->gap_base : 0;
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;

    for (uint64_t rg = uint64_t(blockIdx.x) * kWarps + warp; rg < n_ranges; rg += stride) {
        const uint64_t r0 = rg * kRange, r1 = min(r0 + kRange, n);
        uint64_t ar = 0, ac = 0;  // kAgg: aggregates; else running (row, col) / sums
        if (kPass != kAgg) {
            const ulonglong2 p = A.agg[rg];
            ar = p.x;
            ac = p.y;
        }
        bool marker = false;
        uint32_t e = upper_index<uint64_t>(A.es, 0, A.n_e, r0);
        for (uint64_t c0 = r0; c0 < r1; c0 += kChunk) {
            const uint32_t len = uint32_t(r1 - c0 < kChunk ? r1 - c0 : kChunk);
            while (A.es[e + 1] <= c0) ++e;
            const uint64_t lo = A.es[e], hi = A.es[e + 1];
            const EntryLayout L = A.el[e];
            if (hi < c0 + len || L.numel >= (1ull << 32)) {
                slow_span<kRepr, kPass>(A, c0, c0 + len, ar, ac, marker, has_prev, gap_base);
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
// F2: exclusive SegSum scan of the range aggregates (one CTA of 1024)
// =============================================================================================
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 4;  // items per thread

__device__ __forceinline__ void cta_seg_exclusive(uint64_t& vr, uint64_t& vc, uint64_t* s_r, uint64_t* s_c) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t ir = vr, ic = vc;
    warp_segscan2(ir, ic);
    if (lane == 31) {
        s_r[warp] = ir;
        s_c[warp] = ic;
    }
    __syncthreads();
    uint64_t br = 0, bc = 0;
    for (int w = 0; w < warp; ++w) {
        br = SegSumOp::op(br, s_r[w]);
        bc = SegSumOp::op(bc, s_c[w]);
    }
    uint64_t er = __shfl_up_sync(0xffffffffu, ir, 1), ec = __shfl_up_sync(0xffffffffu, ic, 1);
    if (lane == 0) {
        er = 0;
        ec = 0;
    }
    vr = SegSumOp::op(br, er);
    vc = SegSumOp::op(bc, ec);
    __syncthreads();
}

// One 1024-thread CTA per block of 4096 range aggregates, blocks taken in ticket
// order and chained by a decoupled look-back (one status word per block and
// stream) -- the scan is spread over several SMs instead of serialising ~18K
// 64-bit segmented adds on one.
constexpr uint64_t kScanBlock = uint64_t(kScanThreads) * kScanPer;

__global__ void __launch_bounds__(kScanThreads, 1)
f_range_scan(const uint64_t* __restrict__ totals, ulonglong2* __restrict__ agg, const uint32_t* __restrict__ flags,
             uint64_t* __restrict__ status, unsigned long long* __restrict__ ticket) {
    __shared__ uint64_t s_r[32], s_c[32];
    __shared__ uint64_t s_blk, s_tot[2], s_pre[2];
    if (fast_blocked(flags)) return;
    const uint64_t n = totals[0];
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
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
    uint64_t er = ar, ec = ac;
    cta_seg_exclusive(er, ec, s_r, s_c);  // -> exclusive within the block
    if (threadIdx.x == kScanThreads - 1) {
        s_tot[0] = SegSumOp::op(er, ar);
        s_tot[1] = SegSumOp::op(ec, ac);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: the block's exclusive prefix for both streams
        const uint64_t pr = lookback<SegSumOp>(status, blk, s_tot[0]);
        const uint64_t pc = lookback<SegSumOp>(status + n_blocks, blk, s_tot[1]);
        if (threadIdx.x == 0) {
            s_pre[0] = pr;
            s_pre[1] = pc;
        }
    }
    __syncthreads();
    uint64_t sr = SegSumOp::op(s_pre[0], er), sc = SegSumOp::op(s_pre[1], ec);
#pragma unroll
    for (int j = 0; j < kScanPer; ++j) {  // in place: aggregate -> exclusive prefix
        if (q0 + j < n_ranges) agg[q0 + j] = make_ulonglong2(sr & (H - 1), sc & (H - 1));
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
    f_pass<kRepr, kPass><<<unsigned(sm_count() * per_sm), kThreads, smem, s>>>(a);
    PULSE_LAUNCHED("f_pass", s);
}

template <int kRepr>
void launch_all(const ApplyArgs& a, bool scatter, cudaStream_t s) {
    launch_pass<kRepr, kAgg>(a, s);
    cudaMemsetAsync(a.scan_status, 0, 2 * sizeof(uint64_t) * a.scan_blocks, s);
    f_range_scan<<<a.scan_blocks, kScanThreads, 0, s>>>(a.totals, a.agg, a.flags, a.scan_status, a.scan_ticket);
    PULSE_LAUNCHED("f_range_scan", s);
    static const int mode = getenv("PULSE_APPLY_MODE") ? atoi(getenv("PULSE_APPLY_MODE")) : 0;
    if (a.weights && mode == 0) {  // in place: checked writes with backup, restore if anything failed
        launch_pass<kRepr, kApply>(a, s);
        launch_pass<kRepr, kRestore>(a, s);
    } else {          // indices only (or PULSE_APPLY_MODE=1 in place): validate, then write them
        launch_pass<kRepr, kValidate>(a, s);
        if (scatter) launch_pass<kRepr, kScatter>(a, s);
    }
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
    a.scan_blocks = uint32_t((p.cap / kRange + 2 + kScanBlock - 1) / kScanBlock);
    if (out_indices) a.weights = nullptr;
    const bool scatter = weights_slot >= 0 || out_indices;
    if (repr == PULSE_COO_DOWNSCALED) launch_all<kCoo>(a, scatter, s);
    else if (repr == PULSE_COO_INT32) launch_all<kI32>(a, scatter, s);
    else launch_all<kFlat>(a, scatter, s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_apply)

}  // namespace dev
}  // namespace pulse
