// PULSE index coding on sm_100a (K2): the raw index payloads of
// encode_index_payloads (patch.hpp:116-174) and the value payloads, written
// straight into the identity-codec PULP body (patch_file.hpp:76-82).
//
//   K2a k2_scan_escapes  COO_DOWNSCALED: per warp range (k2_range_entries: 1,024 entries under
//                        16 M changes, 8,192 above), the number of row / column entries that
//                        need the 0xFF / 0xFFFF escape (index_coding.hpp:68-90), plus the
//                        argument checks the reference applies to caller-provided indices.
//   K2L k2_layout        one CTA: exclusive scan of the range escape counts, per-tensor payload
//                        sizes and body offsets, FLAT_INT32 cross-tensor gap bases
//                        (patch.hpp:131-156), the entry table and the result record.
//   K2b k2_emit          single pass: every row/column entry (or u32 gap) and every value, at
//                        its final byte offset.
// COO_DOWNSCALED first runs optimistically (layout + emit assuming no escapes); K2a and the
// exact layout + emit run only if the emit saw an escape (a conditional graph node).
//
// Fast path: a warp stages a 1,024-entry chunk of one segment in shared memory (cp.async, the
// next chunk in flight) and each lane codes 32 consecutive entries serially, its predecessor
// coming from the previous lane; the packed rows / columns / values leave through shared memory
// as aligned 16-byte stores.  Segment boundaries, caller int64 indices and chunks with escapes
// take the per-round walker: 32 entries per round, lane l -> entry round*32 + l, the previous
// entry (delta coding) from a shuffle, the segment / tensor context warp-uniform.
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"
#include "stage.cuh"

namespace pulse {
namespace dev {

// ---- entry sources -------------------------------------------------------------------------
// Compacted K1 output (segment-relative u32) or caller int64 indices
// (encode_index_payloads over an in-memory SparsePatch; segments == tensors).
struct EntryMap {
    const SegDesc* segs;
    const uint32_t* seg_first;
    const uint64_t* seg_start;  // [n_segs + 1] entry offsets
    uint32_t n_segs;
    const uint32_t* idx32;
    const int64_t* idx64;
    const ColDiv* coldiv;       // per tensor
    const uint64_t* numel;      // per tensor
    const TensorLayout* tlay;   // per tensor (emit only; may be null)
    uint64_t cap;               // entries the idx32/val16 arrays hold (mode A); ~0 for mode B
};

// Entries K2 may touch: on overflow K1 counted more changes than it stored, and
// k2_layout reports PULSE_E_CAPACITY -- the kernels must not read past `cap`.
__device__ __forceinline__ uint64_t k2_entries(const EntryMap& em) {
    const uint64_t n = em.seg_start[em.n_segs];
    return n < em.cap ? n : em.cap;
}

// Division of a local index by the tensor's column extent (patch.hpp:165-166):
// 32-bit magic multiply when both fit, 64-bit division otherwise.
__device__ __forceinline__ void coo_split(int64_t L, const ColDiv& cd, int64_t& row, int64_t& col) {
    if (!cd.wide && L >= 0 && L < (int64_t(1) << 32)) {
        const uint32_t n = uint32_t(L);
        const uint32_t q = uint32_t((uint64_t(__umulhi(n, cd.magic)) + n) >> cd.shift);
        row = q;
        col = int64_t(n - q * cd.cols32);
    } else {
        const int64_t c = int64_t(cd.cols);
        row = L / c;
        col = L % c;
    }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-uniform context of the segment a round starts in.
struct SegCtx {
    uint32_t sg, t;
    uint64_t hi;        // first entry after the segment
    uint64_t ts;        // first entry of the tensor
    uint64_t elem_off;  // segment offset inside the tensor
    bool fast;          // 32-bit fast path allowed: tensor < 2^32 elements, compacted input
    uint32_t cols32, magic, shift;
    TensorLayout tl;    // emit only
};

__device__ __forceinline__ SegCtx load_ctx(const EntryMap& em, uint32_t sg) {
    SegCtx c;
    c.sg = sg;
    c.hi = em.seg_start[sg + 1];
    const SegDesc d = em.segs[sg];
    c.t = d.tensor;
    c.elem_off = d.elem_off;
    c.ts = em.seg_start[em.seg_first[d.tensor]];
    const ColDiv cd = em.coldiv[d.tensor];
    c.cols32 = cd.cols32;
    c.magic = cd.magic;
    c.shift = cd.shift;
    c.fast = !em.idx64 && !cd.wide && em.numel[d.tensor] < (1ull << 32);
    if (em.tlay) c.tl = em.tlay[d.tensor];
    return c;
}

__device__ __forceinline__ uint32_t div_magic(uint32_t n, uint32_t magic, uint32_t shift) {
    return uint32_t((uint64_t(__umulhi(n, magic)) + n) >> shift);
}

// One entry of a round, with its predecessor in the same tensor.
struct Ent {
    bool valid;
    uint32_t t;
    uint64_t i, j;      // global entry, ordinal inside the tensor
    int64_t L, Lp;      // local index; previous local index (-1 when j == 0)
};

// Entries per K2 warp range, the same rule in every K2 kernel of a call: eight staged chunks for
// large patches (fewer per-range look-ups), one for patches under 16 M changes, so small
// patches with escapes (walker path) still keep thousands of warps busy (7B / 99.99%: K2
// 0.33 -> 0.14 ms; 99%: 0.333 ms with 1024, 0.310 with 4096, 0.290 with 8192 and 0.296 with
// 16384 entries; 90%: 2.34 -> 2.24 ms from 4096 to 8192, profiles/r2d_ab_variants.txt).
#ifndef PULSE_K2_RANGE_SPLIT
#define PULSE_K2_RANGE_SPLIT (uint64_t(1) << 24)
#endif
#ifndef PULSE_K2_RANGE_MUL
#define PULSE_K2_RANGE_MUL 8
#endif
__device__ __forceinline__ uint32_t k2_range_entries(uint64_t n) {
    return n < uint64_t(PULSE_K2_RANGE_SPLIT) ? kK2RangeEntries : PULSE_K2_RANGE_MUL * kK2RangeEntries;
}

struct Walker {
    const EntryMap& em;
    uint64_t n, base, end;
    SegCtx ctx;
    int64_t carry_L;   // previous round's lane-31 L (same tensor when j > 0)
    uint32_t cur[8];   // this lane's compacted indices for the current batch of 8 rounds
    uint32_t nxt[8];   // ... and the next batch (prefetched)

    __device__ __forceinline__ void fetch(uint32_t (&dst)[8], uint64_t b) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint64_t i = b + uint64_t(r) * 32 + lane;
            dst[r] = i < end ? em.idx32[i] : 0;
        }
    }

    __device__ Walker(const EntryMap& e, uint64_t n_, uint64_t first, uint64_t last)
        : em(e), n(n_), base(first), end(min(last, n_)) {
        if (!em.idx64) {
            fetch(cur, first);
            fetch(nxt, first + 256);
        }
        const uint64_t f = first < n ? first : (n ? n - 1 : 0);
        ctx = load_ctx(em, em.n_segs ? upper_index<uint64_t>(em.seg_start, 0, em.n_segs, f) : 0);
        carry_L = -1;
        if (first > 0 && first < n) {
            const uint32_t sp = upper_index<uint64_t>(em.seg_start, 0, em.n_segs, first - 1);
            carry_L = em.idx64 ? em.idx64[first - 1] : int64_t(em.segs[sp].elem_off + em.idx32[first - 1]);
        }
    }

    __device__ __forceinline__ bool done() const { return base >= end; }

    // Warp-uniform: the whole round lies in the current segment and the 32-bit
    // fast path applies.
    __device__ __forceinline__ bool fast_round() const { return ctx.fast && base + 32 <= ctx.hi; }

    // Fast-path round: this lane's ordinal j, local index L, predecessor Lp
    // (shuffled; lane 0 from the previous round).  Advances the walker.
    __device__ __forceinline__ void fast_step(int rr, uint32_t& j, uint32_t& L, uint32_t& Lp, bool& valid) {
        const int lane = threadIdx.x & 31;
        valid = base + lane < end;
        j = uint32_t(base - ctx.ts) + lane;
        L = uint32_t(ctx.elem_off) + cur[rr];
        uint32_t up = __shfl_up_sync(0xffffffffu, L, 1);
        if (lane == 0) up = uint32_t(carry_L);
        Lp = up;
        carry_L = int64_t(__shfl_sync(0xffffffffu, L, 31));
        base += 32;
    }

    // Round `rr` (0..7) of the current batch; call with a compile-time rr
    // (unrolled loop) so the batch arrays stay in registers, then rotate().
    __device__ __forceinline__ Ent next(int rr) {
        const int lane = threadIdx.x & 31;
        Ent r;
        r.i = base + lane;
        r.valid = r.i < end;
        uint32_t t = ctx.t;
        uint64_t ts = ctx.ts, eoff = ctx.elem_off;
        uint32_t sg = ctx.sg;
        const bool crosses = base + 32 > ctx.hi && ctx.hi < end;  // warp-uniform
        if (crosses && r.valid && r.i >= ctx.hi) {  // rare: walk to this lane's segment
            while (em.seg_start[sg + 1] <= r.i) ++sg;
            const SegDesc d = em.segs[sg];
            t = d.tensor;
            eoff = d.elem_off;
            ts = em.seg_start[em.seg_first[t]];
        }
        r.t = t;
        r.j = r.i - ts;
        r.L = !r.valid ? 0 : em.idx64 ? em.idx64[r.i] : int64_t(eoff + cur[rr]);
        int64_t up = __shfl_up_sync(0xffffffffu, r.L, 1);
        if (lane == 0) up = carry_L;
        r.Lp = (r.valid && r.j > 0) ? up : -1;
        carry_L = __shfl_sync(0xffffffffu, r.L, 31);
        if (crosses) {
            const uint32_t last_sg = __shfl_sync(0xffffffffu, sg, 31);
            if (last_sg != ctx.sg) ctx = load_ctx(em, last_sg);
        }
        base += 32;
        return r;
    }

    __device__ __forceinline__ void rotate() {  // next batch becomes current; prefetch the one after
        if (!em.idx64) {
#pragma unroll
            for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
            fetch(nxt, base + 256);
        }
    }
};

// COO_DOWNSCALED fields of an entry: row gap (first: absolute row) and column
// entry (absolute on a new row, else within-row gap), index_coding.hpp:117-126.
// The predecessor's (row, col) comes from the neighbouring lane.
struct Coo {
    int64_t rg, cv;
};

struct CooWalker {
    int64_t carry_row = 0, carry_col = 0;
    __device__ __forceinline__ Coo fields(const Ent& r, const ColDiv& cd) {
        const int lane = threadIdx.x & 31;
        int64_t row = 0, col = 0;
        if (r.valid) coo_split(r.L, cd, row, col);
        int64_t prow = __shfl_up_sync(0xffffffffu, row, 1), pcol = __shfl_up_sync(0xffffffffu, col, 1);
        if (lane == 0) {
            prow = carry_row;
            pcol = carry_col;
        }
        carry_row = __shfl_sync(0xffffffffu, row, 31);
        carry_col = __shfl_sync(0xffffffffu, col, 31);
        Coo f;
        const bool new_row = r.j == 0 || row != prow;
        f.rg = r.j == 0 ? row : row - prow;
        f.cv = new_row ? col : col - pcol;
        return f;
    }
};

// =============================================================================================
// Staged fast path shared by K2a / K2b.  A warp takes 1024-entry chunks that lie
// inside one segment of a tensor with < 2^32 elements (compacted K1 input):
// the chunk's u32 indices are staged into shared memory with coalesced 16-byte
// loads and each lane derives 32 CONSECUTIVE entries serially -- the
// predecessor of its first entry is the previous lane's last one (shared
// memory; the global entry before the chunk for lane 0).  Everything else
// (segment boundaries, caller int64 indices, and in K2b chunks with escapes)
// takes the per-round walker path.
// =============================================================================================
constexpr uint32_t kChunkE = 1024;                 // entries per staged chunk
constexpr uint32_t kLaneE = kChunkE / 32;          // consecutive entries per lane
constexpr uint32_t kSIdx = kChunkE * 4, kSVal = kChunkE * 2;
// double-buffered (cp.async prefetch of the next chunk): K2a idx; K2b idx + values
// (K2b's packed row/column output reuses the chunk's own idx buffer)
constexpr uint32_t kScanWarpSmem = 2 * kSIdx;
constexpr uint32_t kEmitWarpSmem = 2 * (kSIdx + kSVal);

// A warp's work: ranges rg, rg + stride, ...; each cut into kChunkE chunks.
struct ChunkIt {
    bool ok;
    uint64_t rg, c0, r1;
    uint32_t len;
    bool start;  // the range's first chunk
    __device__ __forceinline__ bool range_start() const { return start; }
    __device__ __forceinline__ bool range_end() const { return c0 + len >= r1; }
};
__device__ __forceinline__ ChunkIt chunk_at(uint64_t rg, uint64_t n_ranges, uint64_t n) {
    const uint32_t re = k2_range_entries(n);
    ChunkIt it;
    it.ok = rg < n_ranges;
    it.rg = rg;
    it.c0 = rg * re;
    it.r1 = min(it.c0 + re, n);
    it.start = true;
    it.len = it.ok ? uint32_t(it.r1 - it.c0 < kChunkE ? it.r1 - it.c0 : kChunkE) : 0;
    return it;
}
__device__ __forceinline__ ChunkIt chunk_next(const ChunkIt& it, uint64_t stride, uint64_t n_ranges, uint64_t n) {
    if (it.c0 + kChunkE < it.r1) {
        ChunkIt nx = it;
        nx.start = false;
        nx.c0 += kChunkE;
        nx.len = uint32_t(nx.r1 - nx.c0 < kChunkE ? nx.r1 - nx.c0 : kChunkE);
        return nx;
    }
    return chunk_at(it.rg + stride, n_ranges, n);
}

struct FastCtx {
    bool fast;
    uint32_t t;
    uint64_t ts;        // first entry of the tensor
    uint32_t elem_off;  // segment offset inside the tensor (< 2^32 on the fast path)
    uint32_t cols32, magic, shift;
};

// Segment of chunk [c0, c0+len) (sg walks forward monotonically) and whether
// the staged path applies.
__device__ __forceinline__ FastCtx fast_ctx(const EntryMap& em, uint64_t c0, uint32_t len, uint32_t& sg) {
    FastCtx c;
    while (em.seg_start[sg + 1] <= c0) ++sg;
    const SegDesc d = em.segs[sg];
    const ColDiv cd = em.coldiv[d.tensor];
    c.t = d.tensor;
    c.ts = em.seg_start[em.seg_first[d.tensor]];
    c.elem_off = uint32_t(d.elem_off);
    c.cols32 = cd.cols32;
    c.magic = cd.magic;
    c.shift = cd.shift;
    c.fast = !em.idx64 && em.seg_start[sg + 1] >= c0 + len && !cd.wide && em.numel[d.tensor] < (1ull << 32);
    return c;
}

// Local index of the predecessor of this lane's first entry (meaningful when
// that entry is not the tensor's first): the previous lane's last staged index,
// or for lane 0 the global entry before the chunk (same tensor, maybe the
// previous segment).
__device__ __forceinline__ uint32_t lane_pred(const EntryMap& em, const uint4* sidx, uint64_t c0, const FastCtx& c,
                                              uint32_t sg) {
    const int lane = threadIdx.x & 31;
    if (lane > 0) return c.elem_off + smem_word<8>(sidx, uint32_t(lane) * kLaneE - 1);
    if (c0 > c.ts) {
        const uint32_t sp = c0 - 1 >= em.seg_start[sg] ? sg : sg - 1;  // same tensor: this or the previous segment
        return uint32_t(em.segs[sp].elem_off + em.idx32[c0 - 1]);
    }
    return 0;
}

// Local index of staged entry 4*i + k of this lane (compile-time i, k).
#define PULSE_LANE_L(q, k) (c.elem_off + ((k) == 0 ? (q).x : (k) == 1 ? (q).y : (k) == 2 ? (q).z : (q).w))

__device__ __forceinline__ void st_u16_any(uint8_t* p, uint32_t v) {
    if ((reinterpret_cast<uintptr_t>(p) & 1) == 0) *reinterpret_cast<uint16_t*>(p) = uint16_t(v);
    else wr_u16(p, v);
}
__device__ __forceinline__ void st_u32_any(uint8_t* p, uint32_t v) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    if ((a & 3) == 0) {
        *reinterpret_cast<uint32_t*>(p) = v;
    } else if ((a & 1) == 0) {
        reinterpret_cast<uint16_t*>(p)[0] = uint16_t(v);
        reinterpret_cast<uint16_t*>(p)[1] = uint16_t(v >> 16);
    } else {
        wr_u32(p, v);
    }
}

// Per-round walker path of K2a over entries [first, last); (re, ce) returned
// advanced (by value, like k2b_span: no address-taken state in the caller's loop).
__device__ __noinline__ uint2 k2a_span(const EntryMap em, uint32_t repr, uint64_t n, uint64_t first, uint64_t last,
                                       uint32_t* __restrict__ t_resc, uint32_t* __restrict__ t_cesc,
                                       uint64_t* __restrict__ err, uint32_t re, uint32_t ce) {
    const bool coo = repr == PULSE_COO_DOWNSCALED;
    const int lane = threadIdx.x & 31;
    Walker w(em, n, first, last);
    CooWalker cw;
    bool seeded = false;
    while (!w.done()) {
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        if (seeded && w.fast_round()) {
            if (coo) {
                uint32_t j, L, Lp;
                bool valid;
                w.fast_step(rr, j, L, Lp, valid);
                const uint32_t row = div_magic(L, w.ctx.magic, w.ctx.shift);
                const uint32_t col = L - row * w.ctx.cols32;
                uint32_t prow = __shfl_up_sync(0xffffffffu, row, 1), pcol = __shfl_up_sync(0xffffffffu, col, 1);
                if (lane == 0) {
                    prow = uint32_t(cw.carry_row);
                    pcol = uint32_t(cw.carry_col);
                }
                cw.carry_row = __shfl_sync(0xffffffffu, row, 31);
                cw.carry_col = __shfl_sync(0xffffffffu, col, 31);
                const bool nr = j == 0 || row != prow;
                const uint32_t rgap = j == 0 ? row : row - prow;
                const uint32_t cval = nr ? col : col - pcol;
                const bool rf = valid && rgap >= 0xFF, cf = valid && cval >= 0xFFFF;
                if (rf) atomicAdd(t_resc + w.ctx.t, 1u);
                if (cf) atomicAdd(t_cesc + w.ctx.t, 1u);
                re += __popc(__ballot_sync(0xffffffffu, rf));
                ce += __popc(__ballot_sync(0xffffffffu, cf));
            } else {
                uint32_t j, L, Lp;
                bool valid;
                w.fast_step(rr, j, L, Lp, valid);
            }
            continue;
        }
        const Ent r = w.next(rr);
        const ColDiv cd = em.coldiv[r.t];
        if (!seeded) {  // predecessor (row, col) of the span's first entry
            seeded = true;
            const int64_t Lp0 = __shfl_sync(0xffffffffu, r.Lp, 0);
            const uint32_t t0 = __shfl_sync(0xffffffffu, r.t, 0);
            if (coo && Lp0 >= 0) coo_split(Lp0, em.coldiv[t0], cw.carry_row, cw.carry_col);
        }
        bool rf = false, cf = false;
        if (em.idx64 && r.valid) {  // argument checks, in the reference's order
            if (repr == PULSE_COO_INT32) {  // delta_encode_indices, index_coding.hpp:18-25
                if (r.L < 0) report(err, error_key(r.t, kStageRows, r.j, kArgNegative));
                else if (r.j > 0 && r.L <= r.Lp) report(err, error_key(r.t, kStageRows, r.j, kArgOrder));
            } else if (repr == PULSE_FLAT_INT32) {  // patch.hpp:139-147 (first entry: k2_layout)
                if (r.j > 0 && r.L <= r.Lp) report(err, error_key(r.t, kStageRows, r.j, kArgOrder));
                else if (r.j > 0 && r.L - r.Lp > 0xFFFFFFFFll)
                    report(err, error_key(r.t, kStageRows, r.j, kDimFlatGap));
            }
        }
        if (coo) {
            const Coo f = cw.fields(r, cd);
            if (r.valid) {
                if (em.idx64) {  // downscale_coo, index_coding.hpp:117-121
                    int64_t row, col;
                    coo_split(r.L, cd, row, col);
                    if (row < 0 || col < 0) report(err, error_key(r.t, kStageRows, r.j, kArgNegative));
                    else if (r.j > 0 && r.L <= r.Lp) report(err, error_key(r.t, kStageRows, r.j, kArgOrder));
                }
                if (f.rg > 0xFFFFFFFFll) report(err, error_key(r.t, kStageRows, r.j, kDimRow));
                if (f.cv > 0xFFFFFFFFll) report(err, error_key(r.t, kStageCols, r.j, kDimCol));
                rf = f.rg >= 0xFF;
                cf = f.cv >= 0xFFFF;
                if (rf) atomicAdd(t_resc + r.t, 1u);
                if (cf) atomicAdd(t_cesc + r.t, 1u);
            }
        }
        re += __popc(__ballot_sync(0xffffffffu, rf));
        ce += __popc(__ballot_sync(0xffffffffu, cf));
      }
      w.rotate();
    }
    return make_uint2(re, ce);
}

// =============================================================================================
// K2a
// =============================================================================================
__global__ void __launch_bounds__(kThreads, 3)
k2_scan_escapes(EntryMap em, uint32_t repr, uint64_t* __restrict__ range_cnt, uint32_t* __restrict__ t_resc,
                uint32_t* __restrict__ t_cesc, uint64_t* __restrict__ err, const uint32_t* __restrict__ run_if) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (run_if && *(volatile const uint32_t*)run_if == 0) return;
    const uint64_t n = k2_entries(em);
    const uint64_t n_ranges = (n + k2_range_entries(n) - 1) / k2_range_entries(n);
    const bool coo = repr == PULSE_COO_DOWNSCALED;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4* bufs = reinterpret_cast<uint4*>(smem + warp * kScanWarpSmem);
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;
    const bool staged = coo && !em.idx64;
    ChunkIt cur = chunk_at(uint64_t(blockIdx.x) * kWarps + warp, n_ranges, n);
    if (staged && cur.ok) stage_async<8>(bufs, reinterpret_cast<const uint8_t*>(em.idx32 + cur.c0), 4 * cur.len);
    cp_async_commit();
    uint32_t re = 0, ce = 0, sg = 0, b = 0;
    while (cur.ok) {
        const ChunkIt nx = chunk_next(cur, stride, n_ranges, n);
        if (staged && nx.ok)  // prefetch the next chunk while this one is decoded
            stage_async<8>(bufs + (b ^ 1) * (kSIdx / 16), reinterpret_cast<const uint8_t*>(em.idx32 + nx.c0), 4 * nx.len);
        cp_async_commit();
        if (cur.range_start()) {
            re = ce = 0;
            sg = em.n_segs ? upper_index<uint64_t>(em.seg_start, 0, em.n_segs, cur.c0) : 0;
        }
        const uint64_t c0 = cur.c0;
        const uint32_t len = cur.len;
        const FastCtx c = fast_ctx(em, c0, len, sg);
        if (!staged || !c.fast) {
            const uint2 rc = k2a_span(em, repr, n, c0, c0 + len, t_resc, t_cesc, err, re, ce);
            re = rc.x;
            ce = rc.y;
        } else {
            const uint4* sidx = bufs + b * (kSIdx / 16);
            cp_async_wait<1>();
            __syncwarp();
            const uint32_t Lp = lane_pred(em, sidx, c0, c, sg);
            const int nv = max(0, min(int(kLaneE), int(len) - lane * int(kLaneE)));
            const bool lane_first = c0 - c.ts + uint64_t(lane) * kLaneE == 0;  // lane holds the tensor's first entry
            uint32_t prow = div_magic(Lp, c.magic, c.shift), pcol = Lp - prow * c.cols32;
            uint32_t lre = 0, lce = 0;
#pragma unroll
            for (int i = 0; i < int(kLaneE / 4); ++i) {
                const uint4 q = lane_vec<8>(sidx, i);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = 4 * i + k;
                    if (j < nv) {
                        const uint32_t Lj = PULSE_LANE_L(q, k);
                        const uint32_t row = div_magic(Lj, c.magic, c.shift), col = Lj - row * c.cols32;
                        const bool first = j == 0 && lane_first;
                        const bool nr = first || row != prow;
                        const uint32_t rgap = first ? row : row - prow;
                        const uint32_t cval = nr ? col : col - pcol;
                        lre += rgap >= 0xFF;
                        lce += cval >= 0xFFFF;
                        prow = row;
                        pcol = col;
                    }
                }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                lre += __shfl_xor_sync(0xffffffffu, lre, off);
                lce += __shfl_xor_sync(0xffffffffu, lce, off);
            }
            if (lane == 0) {
                if (lre) atomicAdd(t_resc + c.t, lre);
                if (lce) atomicAdd(t_cesc + c.t, lce);
            }
            re += lre;
            ce += lce;
            __syncwarp();
        }
        if (cur.range_end() && coo && lane == 0) range_cnt[cur.rg] = uint64_t(re) | (uint64_t(ce) << 32);
        cur = nx;
        b ^= 1;
    }
    cp_async_wait<0>();
}

// =============================================================================================
// K2L: layout (one CTA of 1024 threads)
// =============================================================================================
constexpr int kLayoutThreads = 1024;

// k2_layout's fused scan: four sums and one max (slot 4).
struct LayoutOps {
    static __device__ __forceinline__ uint64_t op(int k, uint64_t a, uint64_t b) {
        return k == 4 ? (a > b ? a : b) : a + b;
    }
};

struct LayoutArgs {
    const uint64_t* range_cnt;   // COO: packed (row | col << 32) escapes per warp range (k2_range_entries)
    ulonglong2* range_pre;       // COO: global escapes before each range
    EntryMap em;
    uint32_t n_tensors;
    const uint64_t* numel;
    uint32_t repr;
    const uint32_t* t_resc;
    const uint32_t* t_cesc;
    TensorLayout* tlay;
    const pulse_scan_summary* gathered;  // may be null
    uint32_t n_ranks, rank;
    uint64_t body_cap;
    pulse_patch_entry* entries;
    pulse_result* result;
    uint64_t* err;
    uint64_t cap;  // K1 capacity (mode A); ~0 for mode B
    const uint32_t* run_if;  // run only if *run_if != 0 (exact re-run after an optimistic pass)
    bool optimistic;         // COO: lay out assuming no escapes (the optimistic emit reads no range_pre)
    uint32_t* zero_u32[3];   // optimistic: per-call state this kernel clears first (t_resc, t_cesc, esc flag)
};

__device__ __forceinline__ int64_t entry_local(const EntryMap& em, uint64_t i) {
    const uint32_t sg = upper_index<uint64_t>(em.seg_start, 0, em.n_segs, i);
    return em.idx64 ? em.idx64[i] : int64_t(em.segs[sg].elem_off + em.idx32[i]);
}

__global__ void __launch_bounds__(kLayoutThreads, 1) k2_layout(LayoutArgs a) {
    if (a.run_if && *(volatile const uint32_t*)a.run_if == 0) return;
    __shared__ uint64_t s_tmp[33 * 5];
    const int tid = threadIdx.x;
    const EntryMap& em = a.em;
    const uint64_t n = em.seg_start[em.n_segs];
    const bool coo = a.repr == PULSE_COO_DOWNSCALED;
    const bool overflow = n > a.cap;
    if (a.optimistic) {  // per-call state, cleared here instead of by memset nodes ahead of K2
        for (uint32_t i = tid; i < a.n_tensors; i += kLayoutThreads) {
            a.zero_u32[0][i] = 0;
            a.zero_u32[1][i] = 0;
        }
        if (tid == 0) {
            *a.zero_u32[2] = 0;
            *a.err = kNoError;
        }
        __syncthreads();
    }

    // (1) COO_DOWNSCALED: exclusive scan of the per-range escape counts (each
    // thread sums a contiguous block, one CTA scan, then writes its block)
    if (coo && !overflow && !a.optimistic) {
        const uint64_t n_ranges = (n + k2_range_entries(n) - 1) / k2_range_entries(n);
        const uint64_t per = (n_ranges + kLayoutThreads - 1) / kLayoutThreads;
        const uint64_t q0 = min(n_ranges, per * tid), q1 = min(n_ranges, q0 + per);
        uint64_t sr = 0, sc = 0;
        for (uint64_t q = q0; q < q1; ++q) {
            const uint64_t v = a.range_cnt[q];
            sr += v & 0xFFFFFFFFull;
            sc += v >> 32;
        }
        uint64_t x2[2] = {sr, sc}, t2[2];
        cta_exclusive_scan<2, kLayoutThreads, AllSum>(x2, t2, s_tmp);
        uint64_t er = x2[0], ec = x2[1];
        for (uint64_t q = q0; q < q1; ++q) {
            const uint64_t v = a.range_cnt[q];
            a.range_pre[q] = make_ulonglong2(er, ec);
            er += v & 0xFFFFFFFFull;
            ec += v >> 32;
        }
    }

    // FLAT carry from earlier shards
    uint64_t carry_has = 0, carry_gap = 0;
    if (a.gathered) {
        for (int q = int(a.rank) - 1; q >= 0; --q) {
            if (a.gathered[q].has_change) {
                carry_has = 1;
                carry_gap = a.gathered[q].last_gap_base;
                break;
            }
        }
    }

    uint64_t body_base = 0, rts_base = 0, cts_base = 0, entry_base = 0;
    int64_t prev_changed = -1;  // last changed tensor of earlier rounds
    for (uint32_t t0 = 0; t0 < a.n_tensors; t0 += kLayoutThreads) {
        const uint32_t t = t0 + tid;
        const bool valid = t < a.n_tensors;
        uint64_t count = 0, resc = 0, cesc = 0, idx_nb = 0;
        if (valid) {
            count = em.seg_start[em.seg_first[t + 1]] - em.seg_start[em.seg_first[t]];
            if (coo) {
                resc = a.t_resc[t];
                cesc = a.t_cesc[t];
                idx_nb = 3 * count + 4 * (resc + cesc);
            } else {
                idx_nb = 4 * count;
            }
        }
        const bool changed = count > 0 && !overflow;
        // one fused scan: body bytes, row / column escapes, entries (sums) and the last changed
        // tensor before t (max of t + 1; 0 = none)
        uint64_t x5[5] = {changed ? idx_nb + 2 * count : 0, resc, cesc, changed ? 1ull : 0ull,
                          changed ? uint64_t(t) + 1 : 0ull},
                 t5[5];
        cta_exclusive_scan<5, kLayoutThreads, LayoutOps>(x5, t5, s_tmp);
        const uint64_t eb = x5[0], er = x5[1], ec = x5[2], ee = x5[3];
        const uint64_t tb = t5[0], tr = t5[1], tc = t5[2], te = t5[3];
        const int64_t mx = int64_t(t5[4]) - 1;
        const int64_t pc = max(prev_changed, int64_t(x5[4]) - 1);  // previous changed tensor before t
        if (valid) {
            TensorLayout L;
            L.idx_off = body_base + eb;
            L.val_off = L.idx_off + idx_nb;
            L.row_bytes = count + 4 * resc;
            L.rts = rts_base + er;
            L.cts = cts_base + ec;
            L.count_nz = changed;
            L.has_prev = 0;
            L.gap_base = 0;
            if (a.repr == PULSE_FLAT_INT32) {
                if (pc >= 0) {
                    const uint64_t last_i = em.seg_start[em.seg_first[pc + 1]] - 1;
                    L.has_prev = 1;
                    L.gap_base = a.numel[pc] - uint64_t(entry_local(em, last_i));
                } else if (carry_has) {
                    L.has_prev = 1;
                    L.gap_base = carry_gap;
                }
            }
            a.tlay[t] = L;
            if (changed) {
                if (a.repr != PULSE_COO_DOWNSCALED && a.numel[t] >= (1ull << 31))
                    report(a.err, error_key(t, kStageTensor, 0, kDimInt32));
                if (a.repr == PULSE_FLAT_INT32) {
                    // patch.hpp:141-147 for the tensor's first entry
                    const int64_t first = entry_local(em, em.seg_start[em.seg_first[t]]);
                    const int64_t entry = first + int64_t(L.has_prev ? L.gap_base : 0);
                    if (entry < 0 || (L.has_prev && entry == 0))
                        report(a.err, error_key(t, kStageRows, 0, kArgOrder));
                    else if (entry > 0xFFFFFFFFll)
                        report(a.err, error_key(t, kStageRows, 0, kDimFlatGap));
                }
                pulse_patch_entry e;
                e.tensor = t;
                e.reserved = 0;
                e.count = count;
                e.idx_off = L.idx_off;
                e.idx_nbytes = idx_nb;
                e.val_off = L.idx_off + idx_nb;
                a.entries[entry_base + ee] = e;
            }
        }
        body_base += tb;
        rts_base += tr;
        cts_base += tc;
        entry_base += te;
        prev_changed = max(prev_changed, mx);
        __syncthreads();
    }

    if (tid == 0) {
        pulse_result r{};
        r.n_changes = n;
        r.body_bytes = body_base;
        r.n_entries = uint32_t(entry_base);
        if (prev_changed >= 0) {  // FLAT continuation for the next shard
            r.carry_out.has_prev = 1;
            r.carry_out.gap_base = a.numel[prev_changed] - uint64_t(entry_local(em, n - 1));
        } else {
            r.carry_out.has_prev = carry_has;
            r.carry_out.gap_base = carry_gap;
        }
        const uint64_t k = *a.err;
        if (overflow) {
            r.status = PULSE_E_CAPACITY;
            r.err_check = kCapacity;
            r.required = n;
        } else if (k != kNoError) {
            r.status = check_status(key_check(k));
            r.err_check = key_check(k);
            r.err_stage = key_stage(k);
            r.err_tensor = key_tensor(k);
            r.err_elem = key_elem(k);
        } else if (body_base > a.body_cap) {
            r.status = PULSE_E_CAPACITY;
            r.err_check = kCapacity;
            r.required = body_base;
            // the optimistic layout assumed no escapes: have the exact pipeline (gated on the
            // escape flag) re-run so `required` is the exact body size
            if (a.optimistic) *a.zero_u32[2] = 1;
        }
        *a.result = r;
    }
}

// =============================================================================================
// K2b: emit
// =============================================================================================
// Per-round walker path of K2b over entries [first, last); (R, Cc): global row /
// column escapes before `first` (COO_DOWNSCALED), returned advanced.  Everything
// by value, not by reference: an address-taken R/Cc/EntryMap lived in local
// memory across K2b's whole chunk loop (its reloads were the top long-scoreboard
// stalls in the r1f ncu capture; k2_emit's LDL/STL count 294 -> 53).
__device__ __noinline__ ulonglong2 k2b_span(const EntryMap em, uint32_t repr, uint64_t n, uint64_t first,
                                            uint64_t last, const TensorLayout* __restrict__ tlay,
                                            const uint16_t* __restrict__ vals, uint8_t* __restrict__ body, uint64_t R,
                                            uint64_t Cc) {
    const int lane = threadIdx.x & 31;
    const bool coo = repr == PULSE_COO_DOWNSCALED;
    Walker w(em, n, first, last);
    CooWalker cw;
    bool seeded = false;
    while (!w.done()) {
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        if (seeded && w.fast_round()) {
            const TensorLayout& tl = w.ctx.tl;
            const uint64_t i = w.base + lane;
            uint32_t j, L, Lp;
            bool valid;
            w.fast_step(rr, j, L, Lp, valid);
            if (coo) {
                const uint32_t row = div_magic(L, w.ctx.magic, w.ctx.shift);
                const uint32_t col = L - row * w.ctx.cols32;
                uint32_t prow = __shfl_up_sync(0xffffffffu, row, 1), pcol = __shfl_up_sync(0xffffffffu, col, 1);
                if (lane == 0) {
                    prow = uint32_t(cw.carry_row);
                    pcol = uint32_t(cw.carry_col);
                }
                cw.carry_row = __shfl_sync(0xffffffffu, row, 31);
                cw.carry_col = __shfl_sync(0xffffffffu, col, 31);
                const bool nr = j == 0 || row != prow;
                const uint32_t rgap = j == 0 ? row : row - prow;
                const uint32_t cval = nr ? col : col - pcol;
                const bool rf = valid && rgap >= 0xFF, cf = valid && cval >= 0xFFFF;
                const uint32_t br = __ballot_sync(0xffffffffu, rf), bc = __ballot_sync(0xffffffffu, cf);
                if (valid) {
                    const uint64_t Ri = R + __popc(br & lanemask_lt());
                    const uint64_t Ci = Cc + __popc(bc & lanemask_lt());
                    uint8_t* rp = body + tl.idx_off + j + 4 * (Ri - tl.rts);
                    if (rf) {
                        rp[0] = 0xFF;
                        wr_u32(rp + 1, rgap);
                    } else {
                        rp[0] = uint8_t(rgap);
                    }
                    uint8_t* cq = body + tl.idx_off + tl.row_bytes + 2ull * j + 4 * (Ci - tl.cts);
                    if (cf) {
                        wr_u16(cq, 0xFFFF);
                        wr_u32(cq + 2, cval);
                    } else {
                        st_u16_any(cq, cval);
                    }
                    st_u16_any(body + tl.val_off + 2ull * j, vals[i]);
                }
                R += __popc(br);
                Cc += __popc(bc);
            } else if (valid) {
                uint64_t g;
                if (j > 0) g = L - Lp;
                else g = uint64_t(L) + (repr == PULSE_FLAT_INT32 && tl.has_prev ? tl.gap_base : 0);
                st_u32_any(body + tl.idx_off + 4ull * j, uint32_t(g));
                st_u16_any(body + tl.val_off + 2ull * j, vals[i]);
            }
            continue;
        }
        const Ent r = w.next(rr);
        const TensorLayout& tl = tlay[r.t];
        if (coo) {
            const ColDiv cd = em.coldiv[r.t];
            if (!seeded) {
                const int64_t Lp0 = __shfl_sync(0xffffffffu, r.Lp, 0);
                const uint32_t t0 = __shfl_sync(0xffffffffu, r.t, 0);
                if (Lp0 >= 0) coo_split(Lp0, em.coldiv[t0], cw.carry_row, cw.carry_col);
            }
            const Coo f = cw.fields(r, cd);
            const bool rf = r.valid && f.rg >= 0xFF, cf = r.valid && f.cv >= 0xFFFF;
            const uint32_t br = __ballot_sync(0xffffffffu, rf), bc = __ballot_sync(0xffffffffu, cf);
            if (r.valid) {
                const uint64_t Ri = R + __popc(br & lanemask_lt());
                const uint64_t Ci = Cc + __popc(bc & lanemask_lt());
                uint8_t* rp = body + tl.idx_off + r.j + 4 * (Ri - tl.rts);
                if (rf) {
                    rp[0] = 0xFF;
                    wr_u32(rp + 1, uint32_t(f.rg));
                } else {
                    rp[0] = uint8_t(f.rg);
                }
                uint8_t* cq = body + tl.idx_off + tl.row_bytes + 2 * r.j + 4 * (Ci - tl.cts);
                if (cf) {
                    wr_u16(cq, 0xFFFF);
                    wr_u32(cq + 2, uint32_t(f.cv));
                } else {
                    st_u16_any(cq, uint32_t(f.cv));
                }
                st_u16_any(body + tl.val_off + 2 * r.j, vals[r.i]);
            }
            R += __popc(br);
            Cc += __popc(bc);
        } else if (r.valid) {
            uint64_t g;
            if (r.j > 0) g = uint64_t(r.L - r.Lp);
            else g = uint64_t(r.L) + (repr == PULSE_FLAT_INT32 && tl.has_prev ? tl.gap_base : 0);
            st_u32_any(body + tl.idx_off + 4 * r.j, uint32_t(g));
            st_u16_any(body + tl.val_off + 2 * r.j, vals[r.i]);
        }
        seeded = true;
      }
      w.rotate();
    }
    return make_ulonglong2(R, Cc);
}

// One staged fast chunk of K2b: COO_DOWNSCALED row/column entries or int32 gaps,
// then the value blob.  Returns false (nothing written) if a COO entry needs an
// escape -- the caller then re-emits the chunk with the walker.  kFull (every
// chunk but a range's last) drops the per-entry tail guards.
template <bool kFull>
__device__ __forceinline__ bool k2b_chunk(const EntryMap& em, uint32_t repr, const FastCtx& c, const TensorLayout& tl,
                                          uint64_t c0, uint32_t len, uint32_t sg, uint64_t R, uint64_t Cc,
                                          uint4* sidx, const uint4* sval, uint8_t* __restrict__ body) {
    const int lane = threadIdx.x & 31;
    const uint32_t Lp = lane_pred(em, sidx, c0, c, sg);
    const int nv = kFull ? int(kLaneE) : max(0, min(int(kLaneE), int(len) - lane * int(kLaneE)));
    const uint64_t j0 = c0 - c.ts;                                     // ordinal of the chunk's first entry
    const bool lane_first = j0 + uint64_t(lane) * kLaneE == 0;         // lane holds the tensor's first entry
    if (repr == PULSE_COO_DOWNSCALED) {
        uint32_t prow = div_magic(Lp, c.magic, c.shift), pcol = Lp - prow * c.cols32;
        uint32_t rw[kLaneE / 4], cw2[kLaneE / 2];
        bool esc = false;
#pragma unroll
        for (int i = 0; i < int(kLaneE / 4); ++i) {
            const uint4 q = lane_vec<8>(sidx, i);
            uint32_t rr = 0, c0w = 0, c1w = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = 4 * i + k;
                const bool v = kFull || j < nv;
                const uint32_t Lj = PULSE_LANE_L(q, k);
                const uint32_t row = div_magic(Lj, c.magic, c.shift), col = Lj - row * c.cols32;
                const bool first = j == 0 && lane_first;
                const bool nr = first || row != prow;
                const uint32_t rgap = first ? row : row - prow;
                const uint32_t cval = nr ? col : col - pcol;
                esc |= v && (rgap >= 0xFF || cval >= 0xFFFF);
                rr |= (v ? rgap & 0xFF : 0u) << (8 * k);
                const uint32_t cpart = (v ? cval & 0xFFFF : 0u) << (16 * (k & 1));
                if (k < 2) c0w |= cpart;
                else c1w |= cpart;
                prow = row;
                pcol = col;
            }
            rw[i] = rr;
            cw2[2 * i] = c0w;
            cw2[2 * i + 1] = c1w;
        }
        if (__any_sync(0xffffffffu, esc)) return false;  // escapes: variable-size entries
        // packed rows (1 KiB, V=2) and columns (2 KiB, V=4) replace the chunk's indices
        uint4* srow = sidx;
        uint4* scol = sidx + kChunkE / 16;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 2; ++i)
            srow[swz<2>(uint32_t(lane * 2 + i))] = make_uint4(rw[4 * i], rw[4 * i + 1], rw[4 * i + 2], rw[4 * i + 3]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
            scol[swz<4>(uint32_t(lane * 4 + i))] = make_uint4(cw2[4 * i], cw2[4 * i + 1], cw2[4 * i + 2], cw2[4 * i + 3]);
        __syncwarp();
        unstage<2>(body + tl.idx_off + j0 + 4 * (R - tl.rts), srow, len);
        unstage<4>(body + tl.idx_off + tl.row_bytes + 2 * j0 + 4 * (Cc - tl.cts), scol, 2 * len);
    } else {
        const uint64_t first_add = repr == PULSE_FLAT_INT32 && tl.has_prev ? tl.gap_base : 0;
        uint32_t prev = Lp;
        __syncwarp();  // every lane has read its predecessor before gaps overwrite indices
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // in place: each lane rewrites only its own slots
            const uint32_t slot = swz<8>(uint32_t(lane * 8 + i));
            const uint4 q = lds128(sidx + slot);
            uint32_t g[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t Lj = PULSE_LANE_L(q, k);
                g[k] = (i == 0 && k == 0 && lane_first) ? uint32_t(uint64_t(Lj) + first_add) : Lj - prev;
                prev = Lj;
            }
            sidx[slot] = make_uint4(g[0], g[1], g[2], g[3]);
        }
        __syncwarp();
        unstage<8>(body + tl.idx_off + 4 * j0, sidx, 4 * len);
    }
    unstage<1>(body + tl.val_off + 2 * j0, sval, 2 * len);
    return true;
}

__global__ void __launch_bounds__(kThreads, 2)
k2_emit(EntryMap em, uint32_t repr, const TensorLayout* __restrict__ tlay,
        const ulonglong2* __restrict__ range_pre, const uint16_t* __restrict__ vals,
        const pulse_result* __restrict__ result, uint8_t* __restrict__ body,
        const uint32_t* __restrict__ run_if, uint32_t* __restrict__ esc_flag) {
    extern __shared__ __align__(16) uint8_t smem[];
    if (run_if && *(volatile const uint32_t*)run_if == 0) return;
    if (result->status != 0) return;
    const uint64_t n = k2_entries(em);
    const uint64_t n_ranges = (n + k2_range_entries(n) - 1) / k2_range_entries(n);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool coo = repr == PULSE_COO_DOWNSCALED;
    uint8_t* ws = smem + warp * kEmitWarpSmem;  // [idx0 | idx1 | val0 | val1]
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;
    const bool staged = !em.idx64;
    auto prefetch = [&](const ChunkIt& it, uint32_t bb) {
        if (staged && it.ok) {
            stage_async<8>(reinterpret_cast<uint4*>(ws + bb * kSIdx), reinterpret_cast<const uint8_t*>(em.idx32 + it.c0),
                           4 * it.len);
            stage_async<1>(reinterpret_cast<uint4*>(ws + 2 * kSIdx + bb * kSVal),
                           reinterpret_cast<const uint8_t*>(vals + it.c0), 2 * it.len);
        }
        cp_async_commit();
    };
    ChunkIt cur = chunk_at(uint64_t(blockIdx.x) * kWarps + warp, n_ranges, n);
    prefetch(cur, 0);
    uint64_t R = 0, Cc = 0;
    uint32_t sg = 0, b = 0;
    // segment context, cached while consecutive chunks stay in one segment
    FastCtx c{};
    TensorLayout tl{};
    uint32_t ctx_sg = ~0u;
    uint64_t ctx_hi = 0;
    bool ctx_ok = false;  // 32-bit fast path allowed for the cached segment's tensor
    while (cur.ok) {
        const ChunkIt nx = chunk_next(cur, stride, n_ranges, n);
        prefetch(nx, b ^ 1);
        if (cur.range_start()) {
            R = Cc = 0;
            if (coo && !esc_flag) {  // exact pass: escapes before the range (the optimistic pass assumes none)
                const ulonglong2 p = range_pre[cur.rg];
                R = p.x;
                Cc = p.y;
            }
            sg = em.n_segs ? warp_upper_index(em.seg_start, em.n_segs, cur.c0) : 0;
        }
        const uint64_t c0 = cur.c0;
        const uint32_t len = cur.len;
        if (sg != ctx_sg || c0 >= ctx_hi) {
            c = fast_ctx(em, c0, len, sg);
            tl = tlay[c.t];
            ctx_sg = sg;
            ctx_hi = em.seg_start[sg + 1];
            ctx_ok = !em.idx64 && !em.coldiv[c.t].wide && em.numel[c.t] < (1ull << 32);
        }
        c.fast = ctx_ok && ctx_hi >= c0 + len;
        uint4* sidx = reinterpret_cast<uint4*>(ws + b * kSIdx);
        const uint4* sval = reinterpret_cast<const uint4*>(ws + 2 * kSIdx + b * kSVal);
        bool done = false;
        if (staged && c.fast) {
            cp_async_wait<1>();
            __syncwarp();
            done = len == kChunkE ? k2b_chunk<true>(em, repr, c, tl, c0, len, sg, R, Cc, sidx, sval, body)
                                  : k2b_chunk<false>(em, repr, c, tl, c0, len, sg, R, Cc, sidx, sval, body);
            __syncwarp();
        }
        if (!done) {  // segment boundary, caller int64 indices, or escapes: per-round walker
            cp_async_wait<1>();  // this chunk's staging lands before its buffer is reused
            const ulonglong2 rc = k2b_span(em, repr, n, c0, c0 + len, tlay, vals, body, R, Cc);
            R = rc.x;
            Cc = rc.y;
            __syncwarp();
        }
        if (esc_flag && (R | Cc) && lane == 0) atomicExch(esc_flag, 1u);  // optimistic pass: escapes seen
        cur = nx;
        b ^= 1;
    }
    cp_async_wait<0>();
}

// =============================================================================================
// launchers
// =============================================================================================
static void emit_common(const PlanDev& p, const EntryMap& em, uint32_t repr, bool validate_args,
                        const pulse_scan_summary* gathered, uint32_t n_ranks, uint32_t rank,
                        const uint16_t* vals, uint8_t* body, uint64_t body_cap, pulse_patch_entry* entries,
                        pulse_result* result, uint64_t cap, cudaStream_t s) {
    const bool optimistic = repr == PULSE_COO_DOWNSCALED && !validate_args && !em.idx64;
    if (!optimistic) {  // (the optimistic k2_layout clears these itself)
        cudaMemsetAsync(p.t_resc, 0, p.n_tensors * sizeof(uint32_t), s);
        cudaMemsetAsync(p.t_cesc, 0, p.n_tensors * sizeof(uint32_t), s);
        cudaMemsetAsync(p.err, 0xFF, sizeof(uint64_t), s);
    }
    static PerDeviceInt occ_scan_d, occ_emit_d;
    int& occ_scan = occ_scan_d.here();
    int& occ_emit = occ_emit_d.here();
    if (!occ_scan) {  // per device: the shared-memory opt-in, then occupancy
        cudaFuncSetAttribute(k2_scan_escapes, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWarps * kScanWarpSmem));
        cudaFuncSetAttribute(k2_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWarps * kEmitWarpSmem));
        int a = 0, b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k2_scan_escapes, kThreads, kWarps * kScanWarpSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k2_emit, kThreads, kWarps * kEmitWarpSmem);
        occ_emit = std::max(b, 1);
        occ_scan = std::max(a, 1);
    }
    LayoutArgs a;
    a.range_cnt = p.range_cnt;
    a.range_pre = p.range_pre;
    a.em = em;
    a.n_tensors = p.n_tensors;
    a.numel = p.numel;
    a.repr = repr;
    a.t_resc = p.t_resc;
    a.t_cesc = p.t_cesc;
    a.tlay = p.tlay;
    a.gathered = gathered;
    a.n_ranks = n_ranks;
    a.rank = rank;
    a.body_cap = body_cap;
    a.entries = entries;
    a.result = result;
    a.err = p.err;
    a.cap = cap;
    a.run_if = nullptr;
    a.optimistic = false;
    const unsigned g_scan = unsigned(sm_count() * occ_scan), g_emit = unsigned(sm_count() * occ_emit);
    auto exact = [&](const uint32_t* run_if, cudaStream_t s) {  // K2a escape counts -> layout -> emit
        if (repr == PULSE_COO_DOWNSCALED || validate_args) {
            k2_scan_escapes<<<g_scan, kThreads, kWarps * kScanWarpSmem, s>>>(em, repr, p.range_cnt, p.t_resc, p.t_cesc,
                                                                            p.err, run_if);
            PULSE_LAUNCHED("k2_scan_escapes", s);
        }
        a.run_if = run_if;
        a.optimistic = false;
        k2_layout<<<1, kLayoutThreads, 0, s>>>(a);
        PULSE_LAUNCHED("k2_layout", s);
        k2_emit<<<g_emit, kThreads, kWarps * kEmitWarpSmem, s>>>(em, repr, p.tlay, p.range_pre, vals, result, body,
                                                                 run_if, nullptr);
        PULSE_LAUNCHED("k2_emit", s);
    };
    a.zero_u32[0] = p.t_resc;
    a.zero_u32[1] = p.t_cesc;
    a.zero_u32[2] = p.d_flags + 2;
    if (optimistic) {
        // Optimistic COO_DOWNSCALED: lay out and emit assuming no entry needs an
        // escape (none does on these shapes at <= 99.9% sparsity); the emit flags
        // any escape it meets, and only then the exact pipeline re-runs (its three
        // kernels return at once otherwise).
        uint32_t* esc = p.d_flags + 2;
        a.optimistic = true;
        k2_layout<<<1, kLayoutThreads, 0, s>>>(a);
        PULSE_LAUNCHED("k2_layout (optimistic)", s);
        k2_emit<<<g_emit, kThreads, kWarps * kEmitWarpSmem, s>>>(em, repr, p.tlay, p.range_pre, vals, result, body,
                                                                 nullptr, esc);
        PULSE_LAUNCHED("k2_emit (optimistic)", s);
        launch_gated(s, esc, [&](cudaStream_t gs) { exact(esc, gs); });
    } else {
        exact(nullptr, s);
    }
}

void launch_encode_emit(const PlanDev& p, uint32_t repr, const pulse_scan_summary* gathered, uint32_t n_ranks,
                        uint32_t rank, uint8_t* body, uint64_t body_cap, pulse_patch_entry* entries,
                        pulse_result* result, cudaStream_t s) {
    EntryMap em{p.segs, p.seg_first, p.seg_start, p.n_segs, p.idx32, nullptr, p.coldiv, p.numel, p.tlay, p.cap};
    emit_common(p, em, repr, false, gathered, n_ranks, rank, p.val16, body, body_cap, entries, result, p.cap, s);
}

void launch_encode_emit_idx64(const PlanDev& p, uint32_t repr, const int64_t* idx64, const uint16_t* vals,
                              uint8_t* body, uint64_t body_cap, pulse_patch_entry* entries, pulse_result* result,
                              cudaStream_t s) {
    EntryMap em{p.id_segs, p.id_first, p.id_start, p.n_tensors, nullptr, idx64, p.coldiv, p.numel, p.tlay, ~0ull};
    emit_common(p, em, repr, true, nullptr, 1, 0, vals, body, body_cap, entries, result, ~0ull, s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_index)

}  // namespace dev
}  // namespace pulse
