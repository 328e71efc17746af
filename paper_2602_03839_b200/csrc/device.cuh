// Device-side building blocks shared by the PULSE kernels (sm_100a).
//
//  * single-pass decoupled look-back over tile status words (K1, K3 scans)
//  * 256-thread block scans
//  * streaming 128-bit loads that do not pollute L1 (each snapshot byte is
//    read exactly once per encode)
//  * first-error keys that reproduce the reference's sequential error order
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pulse_cuda.h"
#include "errors.hpp"

namespace pulse {
namespace dev {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ------------------------------------------------------------------------------------------
// Watchdog for device spin-waits (look-back polling, mbarrier waits).  A wait
// that exceeds kSpinLimit polls records where it was stuck into a host-mapped
// slot and gives up, so a protocol bug surfaces as PULSE_E_CUDA on the host
// instead of a hung GPU.  One slot pointer per translation unit.
// ------------------------------------------------------------------------------------------
constexpr uint64_t kSpinLimit = 1ull << 25;
static __device__ unsigned long long* g_wd_slot = nullptr;

static __device__ __noinline__ void watchdog_fire(uint32_t kind, uint64_t a, uint64_t b, uint64_t c) {
    unsigned long long* w = g_wd_slot;
    if (!w) return;
    if (atomicCAS(w, 0ull, 1ull) == 0ull) {
        w[1] = kind;
        w[2] = blockIdx.x;
        w[3] = threadIdx.x;
        w[4] = a;
        w[5] = b;
        w[6] = c;
        __threadfence_system();
    }
}
// Host side: point this translation unit's watchdog at `slot` (device address).
#define PULSE_DEFINE_WATCHDOG_SETTER(name)                                                         \
    void name(unsigned long long* slot) { cudaMemcpyToSymbol(g_wd_slot, &slot, sizeof(slot)); }

__device__ __forceinline__ void report(uint64_t* err, uint64_t key) {
    atomicMin(reinterpret_cast<unsigned long long*>(err), static_cast<unsigned long long>(key));
}

// ------------------------------------------------------------------------------------------
// Memory helpers
// ------------------------------------------------------------------------------------------
// 128-bit streaming load: read-only path, no L1 allocation, 256-B L2 prefetch.
__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- mbarrier / TMA bulk-copy helpers (sm_90+ PTX, used on sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    uint64_t spins = 0;
    while (!done) {
        if (++spins > kSpinLimit) {
            watchdog_fire(2, smem_u32(bar), parity, 0);
            return;
        }
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// Bulk async copy global -> shared (TMA engine), completion counted in bytes on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Named barriers for warp-specialised groups (id 0 is __syncthreads).
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Unaligned little-endian reads from a byte stream.
__device__ __forceinline__ uint32_t rd_u16(const uint8_t* p) { return uint32_t(p[0]) | uint32_t(p[1]) << 8; }
__device__ __forceinline__ uint32_t rd_u32(const uint8_t* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}
__device__ __forceinline__ void wr_u16(uint8_t* p, uint32_t v) {
    p[0] = uint8_t(v);
    p[1] = uint8_t(v >> 8);
}
__device__ __forceinline__ void wr_u32(uint8_t* p, uint32_t v) {
    p[0] = uint8_t(v);
    p[1] = uint8_t(v >> 8);
    p[2] = uint8_t(v >> 16);
    p[3] = uint8_t(v >> 24);
}

// Largest i in [lo, hi) with a[i] <= x (a non-decreasing, a[lo] <= x).
template <class T>
__device__ __forceinline__ uint32_t upper_index(const T* a, uint32_t lo, uint32_t hi, T x) {
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

// Largest i in [0, n) with a[i] <= x (a[0] <= x), by the whole warp: 32 probes
// per round, so a few hundred segments take two dependent loads, not nine.
__device__ __forceinline__ uint32_t warp_upper_index(const uint64_t* a, uint32_t n, uint64_t x) {
    const int lane = threadIdx.x & 31;
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t p = lo + uint32_t(lane) * step;
        const uint32_t m = __ballot_sync(0xffffffffu, p < hi && a[p] <= x);
        lo += uint32_t(31 - __clz(m)) * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// ------------------------------------------------------------------------------------------
// Scan operators over 62-bit payloads (status words keep 2 flag bits).
// ------------------------------------------------------------------------------------------
struct SumOp {
    static __device__ __forceinline__ uint64_t op(uint64_t earlier, uint64_t later) { return earlier + later; }
};
// Segmented sum: bit 61 marks "a segment head lies in this span"; a later
// span with a head discards everything before it.
struct SegSumOp {
    static constexpr uint64_t kHead = 1ull << 61;
    static __device__ __forceinline__ uint64_t op(uint64_t earlier, uint64_t later) {
        return (later & kHead) ? later : earlier + later;
    }
};

// Max with 0 as identity (callers store x + 1 so "none" is 0).
struct MaxOp {
    static __device__ __forceinline__ uint64_t op(uint64_t earlier, uint64_t later) {
        return earlier > later ? earlier : later;
    }
};

// CTA-wide exclusive scan of K independent 64-bit lanes of values (lane k uses Ops<k>::op,
// identity 0) over the kT threads of the block: one warp-shuffle pass for all K, the kT/32
// warp aggregates scanned by warp 0 -- two barriers for all K values (a serial per-thread walk
// over the warp totals with two barriers per value made the one-CTA layout kernels
// barrier-bound).  x[k] becomes the exclusive prefix, total[k] the block aggregate.
// s_tmp: 33 * K words of shared memory.  Ends with a barrier (s_tmp reusable).
template <int K, int kT, class Ops>
__device__ __forceinline__ void cta_exclusive_scan(uint64_t (&x)[K], uint64_t (&total)[K], uint64_t* s_tmp) {
    static_assert(kT % 32 == 0 && kT <= 1024, "block of whole warps");
    constexpr int kW = kT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t inc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) inc[k] = x[k];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t o = __shfl_up_sync(0xffffffffu, inc[k], off);
            if (lane >= off) inc[k] = Ops::op(k, o, inc[k]);
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int k = 0; k < K; ++k) s_tmp[32 * k + warp] = inc[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint64_t w = lane < kW ? s_tmp[32 * k + lane] : 0;
            uint64_t wi = w;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint64_t o = __shfl_up_sync(0xffffffffu, wi, off);
                if (lane >= off) wi = Ops::op(k, o, wi);
            }
            uint64_t we = __shfl_up_sync(0xffffffffu, wi, 1);
            if (lane == 0) we = 0;
            s_tmp[32 * k + lane] = we;  // exclusive prefix of warp `lane`
            if (lane == 31) s_tmp[32 * K + k] = wi;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        // exclusive within the warp: the inclusive value of the lane before
        uint64_t ex = __shfl_up_sync(0xffffffffu, inc[k], 1);
        if (lane == 0) ex = 0;
        x[k] = lane == 0 ? s_tmp[32 * k + warp] : Ops::op(k, s_tmp[32 * k + warp], ex);
        total[k] = s_tmp[32 * K + k];
    }
    __syncthreads();
}
struct AllSum {
    static __device__ __forceinline__ uint64_t op(int, uint64_t a, uint64_t b) { return a + b; }
};
struct AllSegSum {
    static __device__ __forceinline__ uint64_t op(int, uint64_t a, uint64_t b) { return SegSumOp::op(a, b); }
};

enum : uint64_t { kStatInvalid = 0, kStatAggregate = 1, kStatPrefix = 2 };

// Decoupled look-back (single-pass scan).  Called by all 32 lanes of ONE warp
// of the tile's block; `tile` ids must be handed out in launch order (dynamic
// ticket) so every predecessor is already resident.  Publishes this tile's
// aggregate, walks back over predecessors 32 at a time until it meets an
// inclusive prefix, publishes the inclusive prefix and returns the exclusive
// prefix (identity 0 for tile 0).
template <class Op>
__device__ __forceinline__ uint64_t lookback(uint64_t* status, uint64_t tile, uint64_t agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_relaxed(status, (agg << 2) | kStatPrefix);
        return 0;
    }
    if (lane == 0) st_relaxed(status + tile, (agg << 2) | kStatAggregate);
    uint64_t excl = 0;
    int64_t base = int64_t(tile) - 1;
    while (true) {
        const int64_t idx = base - lane;
        uint64_t s = kStatPrefix;  // before tile 0: an identity prefix
        if (idx >= 0) {
            uint64_t spins = 0;
            do {
                s = ld_relaxed(status + idx);
                if (++spins > kSpinLimit) {
                    watchdog_fire(1, tile, uint64_t(idx), s);
                    s = kStatPrefix;
                    break;
                }
            } while ((s & 3) == kStatInvalid);
        }
        const uint32_t pmask = __ballot_sync(0xffffffffu, (s & 3) == kStatPrefix);
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        uint64_t v = lane <= stop ? (s >> 2) : 0;
        // Ordered reduction: higher lanes are earlier tiles.
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t o = __shfl_down_sync(0xffffffffu, v, off);
            if (lane + off < 32) v = Op::op(o, v);
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        excl = Op::op(v, excl);
        if (pmask) break;
        base -= 32;
    }
    if (lane == 0) st_relaxed(status + tile, (Op::op(excl, agg) << 2) | kStatPrefix);
    return excl;
}

// Look-back for a tile whose aggregate the caller already published (so the
// tile could be counted on by successors before this warp started waiting).
template <class Op>
__device__ __forceinline__ uint64_t lookback_published(uint64_t* status, uint64_t tile, uint64_t agg) {
    const int lane = threadIdx.x & 31;
    uint64_t excl = 0;
    int64_t base = int64_t(tile) - 1;
    while (true) {
        const int64_t idx = base - lane;
        uint64_t s = kStatPrefix;
        if (idx >= 0) {
            uint64_t spins = 0;
            do {
                s = ld_relaxed(status + idx);
                if (++spins > kSpinLimit) {
                    watchdog_fire(1, tile, uint64_t(idx), s);
                    s = kStatPrefix;
                    break;
                }
            } while ((s & 3) == kStatInvalid);
        }
        const uint32_t pmask = __ballot_sync(0xffffffffu, (s & 3) == kStatPrefix);
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        uint64_t v = lane <= stop ? (s >> 2) : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t o = __shfl_down_sync(0xffffffffu, v, off);
            if (lane + off < 32) v = Op::op(o, v);
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        excl = Op::op(v, excl);
        if (pmask) break;
        base -= 32;
    }
    if (lane == 0) st_relaxed(status + tile, (Op::op(excl, agg) << 2) | kStatPrefix);
    return excl;
}

// Block-wide exclusive scan of one value per thread (kThreads threads).
// `s_warp` holds kWarps entries.  Returns the exclusive prefix; `total` gets
// the block aggregate.  Contains two __syncthreads().
template <class Op>
__device__ __forceinline__ uint64_t block_exclusive(uint64_t v, uint64_t* s_warp, uint64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc = Op::op(o, inc);
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint64_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint64_t x = s_warp[w];
        if (w < warp) before = Op::op(before, x);
        all = Op::op(all, x);
    }
    total = all;
    // exclusive within warp
    uint64_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = 0;
    __syncthreads();
    return Op::op(before, ex);
}

}  // namespace dev
}  // namespace pulse
