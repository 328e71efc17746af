// Whole-snapshot reductions on sm_100a (absorption.hpp analyses):
//
//   k_count_changed  elements whose bf16 bit patterns differ between two slots
//                    -- the count behind sparsity() (absorption.hpp:55-78):
//                    the same bitwise compare as K1 without the compaction.
//   k_count_above    elements with |w| > threshold -- frozen_fraction()
//                    (absorption.hpp:38-46).  bf16 magnitudes order like their
//                    15-bit patterns (NaNs excluded), so the host turns the
//                    threshold into the largest magnitude pattern <= it and
//                    the device compares integers, exactly.
//
// Both stream HBM once (16-byte loads, no L1 allocation) over the plan's
// 8192-element tiles, grid-stride, one 64-bit atomic per CTA.
#include <algorithm>

#include "device.cuh"
#include "internal.hpp"

namespace pulse {
namespace dev {

namespace {

constexpr uint32_t kTile = kTileElems;  // 8192

struct TileSpan {
    const uint16_t* a;
    const uint16_t* b;
    uint32_t n;  // elements in this tile
};

__device__ __forceinline__ TileSpan tile_span(const PlanDev& p, uint16_t* const* sa, uint16_t* const* sb,
                                              uint64_t tile) {
    const uint32_t sg = p.tile_seg[tile];
    const SegDesc d = p.segs[sg];
    const uint64_t off = (tile - d.tile_start) * kTile;
    TileSpan t;
    t.a = sa[d.tensor] + d.elem_off + off;
    t.b = sb ? sb[d.tensor] + d.elem_off + off : nullptr;
    t.n = uint32_t(d.numel - off < kTile ? d.numel - off : kTile);
    return t;
}

__device__ __forceinline__ uint32_t pop_diff(const uint4& x, const uint4& y) {
    uint32_t c = 0;
    const uint32_t w[4] = {x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) c += (w[i] & 0xFFFFu ? 1u : 0u) + (w[i] >> 16 ? 1u : 0u);
    return c;
}

// |w| > threshold for a bf16 pattern: magnitude pattern above `thr` (signed, so
// thr = -1 counts every non-NaN weight), NaN magnitudes never compare greater.
__device__ __forceinline__ uint32_t above(uint32_t bits, uint32_t thr) {
    const int32_t m = int32_t(bits & 0x7FFFu);
    return (m > int32_t(thr) && m <= 0x7F80) ? 1u : 0u;
}

__device__ __forceinline__ uint32_t pop_above(const uint4& x, uint32_t thr) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) c += above(w[i] & 0xFFFFu, thr) + above(w[i] >> 16, thr);
    return c;
}

template <bool kDiff>
__global__ void __launch_bounds__(kThreads)
k_count(PlanDev p, uint16_t* const* sa, uint16_t* const* sb, uint32_t thr, unsigned long long* out) {
    __shared__ uint64_t s_w[kWarps];
    uint64_t cnt = 0;
    for (uint64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const TileSpan t = tile_span(p, sa, kDiff ? sb : nullptr, tile);
        const uint32_t nvec = t.n / 8;
        const uint4* va = reinterpret_cast<const uint4*>(t.a);
        const uint4* vb = reinterpret_cast<const uint4*>(t.b);
        for (uint32_t v = threadIdx.x; v < nvec; v += kThreads) {
            const uint4 x = ld_stream(va + v);
            if (kDiff) cnt += pop_diff(x, ld_stream(vb + v));
            else cnt += pop_above(x, thr);
        }
        for (uint32_t e = nvec * 8 + threadIdx.x; e < t.n; e += kThreads)  // < 8-element tail
            cnt += kDiff ? (t.a[e] != t.b[e] ? 1u : 0u) : above(t.a[e], thr);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < kWarps; ++w) tot += s_w[w];
        if (tot) atomicAdd(out, tot);
    }
}

}  // namespace

void launch_count_changed(const PlanDev& p, uint32_t slot_a, uint32_t slot_b, uint64_t* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
    if (!p.n_tiles) return;
    const unsigned grid = unsigned(std::min<uint64_t>(p.n_tiles, uint64_t(sm_count()) * 8));
    k_count<true><<<grid, kThreads, 0, s>>>(p, p.slot[slot_a], p.slot[slot_b], 0u,
                                            reinterpret_cast<unsigned long long*>(out));
    PULSE_LAUNCHED("k_count<diff>", s);
}

void launch_count_above(const PlanDev& p, uint32_t slot, uint32_t magnitude_bits, uint64_t* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
    if (!p.n_tiles) return;
    const unsigned grid = unsigned(std::min<uint64_t>(p.n_tiles, uint64_t(sm_count()) * 8));
    k_count<false><<<grid, kThreads, 0, s>>>(p, p.slot[slot], nullptr, magnitude_bits,
                                             reinterpret_cast<unsigned long long*>(out));
    PULSE_LAUNCHED("k_count<above>", s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_reduce)

}  // namespace dev
}  // namespace pulse
