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
//   F1 f_range_agg   per warp range of 4096 entries: segmented-sum aggregates
//                    (rows: restart at each tensor; columns: restart at each new
//                    row, index_coding.hpp:141-153); flags escape markers.
//   F2 f_range_scan  one CTA: exclusive scan of the range aggregates.
//   F3 f_validate    recompute every (row, col) / index and apply the reference
//                    checks (zero gap, column range, index range) -- no writes.
//   F4 f_scatter     only if nothing failed: recompute and W[flat] = value.
//
// If d_layout or F1 finds anything the fixed layout cannot express (escapes,
// short/long payloads, marker bytes), `flags[0]` routes the patch to the
// general parser in decode.cu instead; every kernel checks it on entry.
#include "device.cuh"
#include "internal.hpp"

namespace pulse {
namespace dev {

namespace {

constexpr uint32_t kRange = 4096;  // entries per warp range
constexpr uint64_t H = SegSumOp::kHead;

__device__ __forceinline__ uint32_t lanemask_le() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

// Warp-uniform context: the patch entry a round starts in.
struct ECtx {
    uint32_t e;
    uint64_t lo, hi;   // entries [lo, hi) belong to e
    EntryLayout L;
    uint32_t magic, shift;
};

__device__ __forceinline__ ECtx load_ectx(const EntryLayout* el, const uint64_t* es, const ColDiv* cdv, uint32_t e) {
    ECtx c;
    c.e = e;
    c.lo = es[e];
    c.hi = es[e + 1];
    c.L = el[e];
    const ColDiv d = cdv[c.L.tensor];
    c.magic = d.magic;
    c.shift = d.shift;
    return c;
}

// One round of 32 consecutive entries: per-lane entry, ordinal and raw fields.
struct Fields {
    bool valid;
    uint32_t e;
    uint64_t o;
    uint32_t a;  // COO: row gap byte; int32: the u32 gap
    uint32_t b;  // COO: column entry (u16)
    // this lane's entry layout (by value: the warp context may move on)
    uint32_t tensor;
    uint64_t val_off, numel, cols, flat_base;
};

struct EWalker {
    const EntryLayout* el;
    const uint64_t* es;
    const ColDiv* cdv;
    uint32_t n_e;
    uint64_t base, end;
    ECtx ctx;

    __device__ EWalker(const EntryLayout* el_, const uint64_t* es_, const ColDiv* cdv_, uint32_t n_e_, uint64_t first,
                       uint64_t last)
        : el(el_), es(es_), cdv(cdv_), n_e(n_e_), base(first), end(last) {
        const uint64_t f = first < end ? first : first;
        ctx = load_ectx(el, es, cdv, upper_index<uint64_t>(es, 0, n_e, f));
    }

    // Reads this lane's fields for `repr`; entries past a boundary walk per lane.
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
            if (last_e != ctx.e) ctx = load_ectx(el, es, cdv, last_e);
        }
        base += 32;
        return f;
    }
};

// Segmented warp aggregate of (head, value) items in lane order.
__device__ __forceinline__ uint64_t seg_round_agg(bool head, uint64_t v) {
    const uint32_t hm = __ballot_sync(0xffffffffu, head);
    const int lane = threadIdx.x & 31;
    const int last = hm ? 31 - __clz(hm) : 0;
    uint64_t x = (hm == 0 || lane >= last) ? v : 0;
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    return x | (hm ? H : 0);
}

// Inclusive segmented scan within the round, continuing `carry` (a plain
// running value).  Returns this lane's value; updates carry to lane 31's.
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

__device__ __forceinline__ bool fast_blocked(const uint32_t* flags) { return *(volatile const uint32_t*)flags != 0; }

}  // namespace

// =============================================================================================
// F1
// =============================================================================================
__global__ void __launch_bounds__(kThreads)
f_range_agg(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ es, const ColDiv* __restrict__ cdv,
            uint32_t n_e, const uint8_t* __restrict__ body, uint32_t repr, const uint64_t* __restrict__ totals,
            ulonglong2* __restrict__ agg, uint32_t* __restrict__ flags) {
    if (fast_blocked(flags)) return;
    const uint64_t n = totals[0];
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
    const bool coo = repr == PULSE_COO_DOWNSCALED;
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;
    for (uint64_t rg = uint64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5); rg < n_ranges; rg += stride) {
        const uint64_t first = rg * kRange;
        EWalker w(el, es, cdv, n_e, first, min(first + kRange, n));
        uint64_t ar = 0, ac = 0;  // SegSum aggregates (earlier ⊕ later)
        bool marker = false;
        while (w.base < w.end) {
            const Fields f = w.next(body, coo);
            if (coo) {
                marker |= f.valid && (f.a == 0xFF || f.b == 0xFFFF);
                const bool hr = f.valid && f.o == 0;
                const bool hc = f.valid && (f.o == 0 || f.a != 0);
                ar = SegSumOp::op(ar, seg_round_agg(hr, f.a));
                ac = SegSumOp::op(ac, seg_round_agg(hc, f.b));
            } else {
                const bool hr = repr == PULSE_COO_INT32 && f.valid && f.o == 0;
                ar = SegSumOp::op(ar, seg_round_agg(hr, f.a));
            }
        }
        if (__any_sync(0xffffffffu, marker) && (threadIdx.x & 31) == 0) atomicExch(flags, 1u);
        if ((threadIdx.x & 31) == 0) agg[rg] = make_ulonglong2(ar, ac);
    }
}

// =============================================================================================
// F2: exclusive SegSum scan of the range aggregates (one CTA of 1024)
// =============================================================================================
constexpr int kScanThreads = 1024;

__device__ __forceinline__ void cta_seg_exclusive(uint64_t& vr, uint64_t& vc, uint64_t* s_r, uint64_t* s_c) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t ir = vr, ic = vc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o1 = __shfl_up_sync(0xffffffffu, ir, off);
        const uint64_t o2 = __shfl_up_sync(0xffffffffu, ic, off);
        if (lane >= off) {
            ir = SegSumOp::op(o1, ir);
            ic = SegSumOp::op(o2, ic);
        }
    }
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

__global__ void __launch_bounds__(kScanThreads, 1)
f_range_scan(const uint64_t* __restrict__ totals, ulonglong2* __restrict__ agg, const uint32_t* __restrict__ flags) {
    __shared__ uint64_t s_r[32], s_c[32];
    if (fast_blocked(flags)) return;
    const uint64_t n = totals[0];
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
    const uint64_t per = (n_ranges + kScanThreads - 1) / kScanThreads;
    const uint64_t q0 = min(n_ranges, per * threadIdx.x), q1 = min(n_ranges, q0 + per);
    uint64_t sr = 0, sc = 0;
    for (uint64_t q = q0; q < q1; ++q) {
        const ulonglong2 v = agg[q];
        sr = SegSumOp::op(sr, v.x);
        sc = SegSumOp::op(sc, v.y);
    }
    cta_seg_exclusive(sr, sc, s_r, s_c);
    for (uint64_t q = q0; q < q1; ++q) {  // in place: aggregate -> exclusive prefix
        const ulonglong2 v = agg[q];
        agg[q] = make_ulonglong2(sr & (H - 1), sc & (H - 1));
        sr = SegSumOp::op(sr, v.x);
        sc = SegSumOp::op(sc, v.y);
    }
}

// =============================================================================================
// F3 / F4: recompute per entry; validate, then scatter
// =============================================================================================
template <bool kScatter>
__global__ void __launch_bounds__(kThreads)
f_apply(const EntryLayout* __restrict__ el, const uint64_t* __restrict__ es, const ColDiv* __restrict__ cdv,
        uint32_t n_e, const uint8_t* __restrict__ body, uint32_t repr, const pulse_flat_carry* __restrict__ carry,
        const uint64_t* __restrict__ totals, const ulonglong2* __restrict__ pre, const uint32_t* __restrict__ flags,
        uint64_t* __restrict__ err, uint16_t* const* __restrict__ weights, int64_t* __restrict__ out_idx) {
    if (fast_blocked(flags)) return;
    if (kScatter && *(volatile const uint64_t*)err != kNoError) return;
    const uint64_t n = totals[0];
    const uint64_t n_ranges = (n + kRange - 1) / kRange;
    const bool coo = repr == PULSE_COO_DOWNSCALED;
    const bool has_prev = carry && carry->has_prev;
    const uint64_t gap_base = has_prev ? carry->gap_base : 0;
    const uint64_t stride = uint64_t(gridDim.x) * kWarps;
    for (uint64_t rg = uint64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5); rg < n_ranges; rg += stride) {
        const uint64_t first = rg * kRange;
        EWalker w(el, es, cdv, n_e, first, min(first + kRange, n));
        const ulonglong2 p = pre[rg];
        uint64_t cr = p.x, cc = p.y;  // running (row, col) or running index / global sum
        while (w.base < w.end) {
            const uint64_t i = w.base + (threadIdx.x & 31);
            const Fields f = w.next(body, coo);
            if (coo) {
                const bool hr = f.valid && f.o == 0;
                const bool nr = f.valid && (f.o == 0 || f.a != 0);
                const uint64_t row = seg_round_scan(hr, f.a, cr);
                const uint64_t col = seg_round_scan(nr, f.b, cc);
                if (!f.valid) continue;
                if (!kScatter) {
                    if (!nr && f.b == 0) { report(err, error_key(f.e, kStageCols, f.o, kZeroColGap)); continue; }
                    if (col >= f.cols) { report(err, error_key(f.e, kStageRange, f.o, kColRange)); continue; }
                }
                uint64_t flat;
                if (f.cols < (1ull << 32) && row < (1ull << 32)) {
                    flat = uint64_t(uint32_t(row)) * uint32_t(f.cols) + col;
                } else {
                    flat = row * f.cols + col;
                }
                if (!kScatter) {
                    if (flat >= f.numel) report(err, error_key(f.e, kStageRange, f.o, kIdxRange));
                } else if (out_idx) {
                    out_idx[i] = int64_t(flat);
                } else {
                    weights[f.tensor][flat] = uint16_t(rd_u16(body + f.val_off + 2 * f.o));
                }
            } else if (repr == PULSE_COO_INT32) {
                const bool hr = f.valid && f.o == 0;
                const uint64_t idx = seg_round_scan(hr, f.a, cr);
                if (!f.valid) continue;
                if (!kScatter) {
                    if (f.o > 0 && f.a == 0) { report(err, error_key(f.e, kStageRows, f.o, kZeroGap)); continue; }
                    if (idx >= f.numel) report(err, error_key(f.e, kStageRows, f.o, kIdxRange));
                } else if (out_idx) {
                    out_idx[i] = int64_t(idx);
                } else {
                    weights[f.tensor][idx] = uint16_t(rd_u16(body + f.val_off + 2 * f.o));
                }
            } else {  // FLAT_INT32: one running global sum (patch.hpp:219-237)
                const uint64_t S = seg_round_scan(false, f.a, cr);
                if (!f.valid) continue;
                const int64_t local = int64_t(S) - int64_t(gap_base) - int64_t(f.flat_base);
                if (!kScatter) {
                    if (f.a == 0 && (i > 0 || has_prev)) { report(err, error_key(f.e, kStageRows, f.o, kZeroGap)); continue; }
                    if (local < 0 || uint64_t(local) >= f.numel) report(err, error_key(f.e, kStageRows, f.o, kIdxRange));
                } else if (out_idx) {
                    out_idx[i] = local;
                } else {
                    weights[f.tensor][local] = uint16_t(rd_u16(body + f.val_off + 2 * f.o));
                }
            }
        }
    }
}

// =============================================================================================
// launcher (called from launch_decode after d_layout)
// =============================================================================================
void launch_apply_fast(const PlanDev& p, uint32_t repr, const uint8_t* body, uint32_t n_entries,
                       const pulse_flat_carry* carry, int weights_slot, int64_t* out_indices, uint32_t* flags,
                       cudaStream_t s) {
    const unsigned grid = unsigned(sm_count() * 4);
    ulonglong2* agg = reinterpret_cast<ulonglong2*>(p.flat);  // flat scratch is free on this path
    f_range_agg<<<grid, kThreads, 0, s>>>(p.elay, p.d_es, p.coldiv, n_entries, body, repr, p.d_totals, agg, flags);
    f_range_scan<<<1, kScanThreads, 0, s>>>(p.d_totals, agg, flags);
    f_apply<false><<<grid, kThreads, 0, s>>>(p.elay, p.d_es, p.coldiv, n_entries, body, repr, carry, p.d_totals, agg,
                                             flags, p.err, nullptr, nullptr);
    if (weights_slot >= 0 || out_indices)
        f_apply<true><<<grid, kThreads, 0, s>>>(p.elay, p.d_es, p.coldiv, n_entries, body, repr, carry, p.d_totals,
                                                agg, flags, p.err, weights_slot >= 0 ? p.slot[weights_slot] : nullptr,
                                                out_indices);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_apply)

}  // namespace dev
}  // namespace pulse
