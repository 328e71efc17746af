// PULSE encode on sm_100a.
//
//   K1  k1_tma            bitwise diff of two resident bf16 snapshots and order-preserving
//                         compaction of every changed element (reference loop:
//                         patch.hpp:296-301).  One persistent CTA per SM, warp-specialised: a
//                         producer warp streams 65,536-element tickets into a shared-memory ring
//                         with TMA (cp.async.bulk), eight consumer warps diff and stage the
//                         changes, a look-back / flush group orders the tickets (decoupled
//                         look-back) and writes them out.  Output: u32 segment-relative index +
//                         u16 value per change.  Five staging shapes (tma::Cfg, chosen from the
//                         plan's change capacity) trade ring depth against staging room.
//   K1b k1_deferred       tickets too dense for the staging, re-streamed after K1 (gated).
//   k1_static / k1_ticket the earlier non-TMA K1 (8,192-element tiles), kept for A/B runs.
// The index coders (K2) are in index_code.cu.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "internal.hpp"

namespace pulse {
namespace dev {

// =============================================================================================
// K1
// =============================================================================================
// Tile = 8192 elements of one segment (16 KiB of each snapshot): 256 threads x
// 4 x 128-bit vectors per snapshot.  Two schedules share the tile body:
//   static  persistent grid launched cooperatively (co-residency guaranteed);
//           CTA b owns tiles b, b+G, b+2G ... and issues the loads of its next
//           tile before the current tile's look-back, so the look-back latency
//           hides behind memory traffic.  All CTAs sit at the same iteration,
//           so the predecessors a look-back needs are being counted concurrently.
//   ticket  one tile per dynamic ticket (atomic counter), no prefetch; kept as a
//           fallback when a cooperative launch is unavailable.
struct TileCtx {
    const uint16_t* pp;  // prev tile base
    const uint16_t* cp;  // curr tile base
    uint32_t si;         // segment
    uint32_t toff;       // element offset of the tile inside its segment
    uint32_t nin;        // elements in the tile (<= kTileElems)
};

__device__ __forceinline__ TileCtx locate_tile(uint64_t tile, const uint32_t* __restrict__ tile_seg,
                                               const SegDesc* __restrict__ segs,
                                               const uint16_t* const* __restrict__ prev_ptrs,
                                               const uint16_t* const* __restrict__ curr_ptrs) {
    TileCtx c;
    c.si = tile_seg[tile];
    const SegDesc sd = segs[c.si];
    c.toff = uint32_t((tile - sd.tile_start) * kTileElems);
    c.nin = min(kTileElems, sd.numel - c.toff);
    c.pp = prev_ptrs[sd.tensor] + sd.elem_off + c.toff;
    c.cp = curr_ptrs[sd.tensor] + sd.elem_off + c.toff;
    return c;
}

__device__ __forceinline__ void load_tile(const TileCtx& c, int tid, uint4 (&a)[4], uint4 (&b)[4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t e = (uint32_t(j) * kThreads + tid) * 8;
        if (e + 8 <= c.nin) {
            a[j] = ld_stream(c.pp + e);
            b[j] = ld_stream(c.cp + e);
        } else {
            uint32_t ta[4] = {0, 0, 0, 0}, tb[4] = {0, 0, 0, 0};
            for (uint32_t k = 0; k < 8 && e + k < c.nin; ++k) {
                ta[k >> 1] |= uint32_t(c.pp[e + k]) << ((k & 1) * 16);
                tb[k >> 1] |= uint32_t(c.cp[e + k]) << ((k & 1) * 16);
            }
            a[j] = make_uint4(ta[0], ta[1], ta[2], ta[3]);
            b[j] = make_uint4(tb[0], tb[1], tb[2], tb[3]);
        }
    }
}

__device__ __forceinline__ uint32_t change_mask(const uint4& a, const uint4& b) {
    const uint32_t w0 = __vcmpne2(a.x, b.x), w1 = __vcmpne2(a.y, b.y);
    const uint32_t w2 = __vcmpne2(a.z, b.z), w3 = __vcmpne2(a.w, b.w);
    return (w0 & 1) | ((w0 >> 15) & 2) | ((w1 & 1) << 2) | ((w1 >> 13) & 8) | ((w2 & 1) << 4) |
           ((w2 >> 11) & 32) | ((w3 & 1) << 6) | ((w3 >> 9) & 128);
}

__device__ __forceinline__ uint16_t lane_value(const uint4& v, int k) {
    const uint32_t w = k < 4 ? (k < 2 ? v.x : v.y) : (k < 6 ? v.z : v.w);
    return uint16_t(w >> ((k & 1) * 16));
}

struct K1Args {
    uint32_t* trace;  // optional per-ticket progress trace (debug)
    int experiment;   // 1: consumers only release stages (TMA streaming rate); 4: coalesced dummy write-back; 2: no global
                      // write-back of staged entries; 3: consumers count but do not stage
    const SegDesc* segs;
    const uint32_t* tile_seg;
    uint32_t n_segs;
    uint64_t n_tiles;
    const uint16_t* const* prev_ptrs;
    const uint16_t* const* curr_ptrs;
    uint32_t* out_idx;
    uint16_t* out_val;
    uint64_t capacity;
    uint64_t* seg_start;
    uint64_t* status;
    unsigned long long* ticket;
    ulonglong2* defer;              // (ticket, output offset) of the tickets K1b writes
    unsigned long long* n_defer;
};

// Count / order / look-back / write for one loaded tile.  `prefetch` is called
// after the count is known and before the look-back (issues the next loads).
template <class Prefetch>
__device__ __forceinline__ void k1_tile(const K1Args& k, uint64_t tile, const TileCtx& cur, const uint4 (&a)[4],
                                        const uint4 (&b)[4], uint64_t* s_warp, uint64_t* s_excl,
                                        Prefetch&& prefetch) {
    const int tid = threadIdx.x;
    uint32_t m[4];
    uint64_t packed = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        m[j] = change_mask(a[j], b[j]);
        packed |= uint64_t(__popc(m[j])) << (16 * j);
    }
    uint64_t tot;
    const uint64_t ex = block_exclusive<SumOp>(packed, s_warp, tot);
    const uint64_t count = (tot & 0xFFFF) + ((tot >> 16) & 0xFFFF) + ((tot >> 32) & 0xFFFF) + (tot >> 48);
    prefetch();
    const bool seg_first = cur.toff == 0;
    const bool last = tile == k.n_tiles - 1;
    if (tid < 32) {
        uint64_t excl = 0;
        if (count > 0 || seg_first || last) {
            excl = lookback<SumOp>(k.status, tile, count);
        } else if (tid == 0) {
            st_relaxed(k.status + tile, kStatAggregate);  // aggregate 0; never needs its prefix
        }
        if (tid == 0) {
            *s_excl = excl;
            if (seg_first) k.seg_start[cur.si] = excl;
            if (last) k.seg_start[k.n_segs] = excl + count;
        }
    }
    __syncthreads();
    if (count > 0) {
        uint64_t base = *s_excl;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t mj = m[j];
            uint64_t pos = base + ((ex >> (16 * j)) & 0xFFFF);
            const uint32_t e = cur.toff + (uint32_t(j) * kThreads + tid) * 8;
            while (mj) {
                const int q = __ffs(mj) - 1;
                mj &= mj - 1;
                if (pos < k.capacity) {
                    k.out_idx[pos] = e + q;
                    k.out_val[pos] = lane_value(b[j], q);
                }
                ++pos;
            }
            base += (tot >> (16 * j)) & 0xFFFF;
        }
    }
}

__global__ void __launch_bounds__(kThreads, 3) k1_static(K1Args k) {
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x;
    uint64_t tile = blockIdx.x;
    if (tile >= k.n_tiles) return;
    TileCtx cur = locate_tile(tile, k.tile_seg, k.segs, k.prev_ptrs, k.curr_ptrs);
    uint4 a[4], b[4];
    load_tile(cur, tid, a, b);
    while (true) {
        const uint64_t next = tile + gridDim.x;
        const bool more = next < k.n_tiles;
        TileCtx nx = cur;
        if (more) nx = locate_tile(next, k.tile_seg, k.segs, k.prev_ptrs, k.curr_ptrs);
        uint4 an[4], bn[4];
        k1_tile(k, tile, cur, a, b, s_warp, &s_excl, [&] {
            if (more) load_tile(nx, tid, an, bn);
        });
        if (!more) break;
        __syncthreads();  // s_excl / s_warp reuse
        cur = nx;
        tile = next;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            a[j] = an[j];
            b[j] = bn[j];
        }
    }
}

__global__ void __launch_bounds__(kThreads, 4) k1_ticket(K1Args k) {
    __shared__ uint64_t s_warp[kWarps];
    __shared__ uint64_t s_excl, s_tile;
    const int tid = threadIdx.x;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(k.ticket, 1ull);
        __syncthreads();
        const uint64_t tile = s_tile;
        if (tile >= k.n_tiles) break;
        const TileCtx cur = locate_tile(tile, k.tile_seg, k.segs, k.prev_ptrs, k.curr_ptrs);
        uint4 a[4], b[4];
        load_tile(cur, tid, a, b);
        k1_tile(k, tile, cur, a, b, s_warp, &s_excl, [] {});
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// K1 (default): warp-specialised, TMA-fed.  One CTA per SM.
//   warp 8      producer: takes 64 Ki-element tickets, streams each as 8
//               sub-tiles of 8192 elements (16 KiB prev + 16 KiB curr) into a
//               4-stage shared-memory ring with cp.async.bulk + mbarriers.
//   warps 0-7   consumers: bitwise compare from shared memory, ordered
//               compaction into a per-ticket staging buffer, publish the
//               ticket aggregate as soon as the ticket is counted.
//   warps 9-12  look-back group: decoupled look-back for a counted ticket
//               (warp 9, 4 status words per lane per round), then a coalesced
//               flush of the staged (index, value) pairs -- overlapped with the
//               consumers streaming the next ticket (double-buffered staging).
// A ticket is taken only after the previous one is fully issued and its
// aggregate depends on nothing but its own data, so look-backs never wait on
// a ticket held by a stalled CTA.
// ---------------------------------------------------------------------------------------------
namespace tma {
// Two staging shapes, picked per plan (launch_encode_scan).  Sparse patches gain
// from more ring stages and more tickets in flight between the consumers and
// the look-back/flush group (measured at 7B / 99%: 4 stages x 3 buffers 4.83 ms,
// 5 x 5 4.49 ms); dense ones need room for element entries per buffer (90%:
// 3 x 4 with 8192 entries 13.7 ms; the sparse shape would overflow its staging
// and re-stream nearly every ticket).  PULSE_K1_* macros override the sparse
// shape for experiments; PULSE_K1_SHAPE=sparse|sparse_low|dense|dense2|dense3 forces one per launch.
#ifndef PULSE_K1_STAGES
#define PULSE_K1_STAGES 5
#endif
#ifndef PULSE_K1_BUFS
#define PULSE_K1_BUFS 5
#endif
#ifndef PULSE_K1_COOP_STAGE
#define PULSE_K1_COOP_STAGE 1  // element mode: warp-cooperative staging (0: per-lane loop over mask bits)
#endif
#ifndef PULSE_K1_FLAT_FLUSH
#define PULSE_K1_FLAT_FLUSH 0  // element flush over the whole ticket when < this many entries per chunk
#endif
#ifndef PULSE_K1_COOP_MIN_BITS
#define PULSE_K1_COOP_MIN_BITS 2  // ... only for warp chunks with a vector of more changes than this
#endif
#ifndef PULSE_K1_RECCAP
#define PULSE_K1_RECCAP 448
#endif
#ifndef PULSE_K1_STAGECAP
#define PULSE_K1_STAGECAP 2688
#endif
#ifndef PULSE_K1_DSTAGES
#define PULSE_K1_DSTAGES 3
#endif
#ifndef PULSE_K1_DBUFS
#define PULSE_K1_DBUFS 4
#endif
#ifndef PULSE_K1_DRECCAP
#define PULSE_K1_DRECCAP 1344
#endif
#ifndef PULSE_K1_DSTAGECAP
#define PULSE_K1_DSTAGECAP 8192
#endif
#ifndef PULSE_K1_DDENSE
#define PULSE_K1_DDENSE 3072
#endif
template <int S, int B, uint32_t RC, uint32_t SC, uint32_t DT, uint32_t DF, int LB = 4>
struct Cfg {
    static constexpr int kLbWarps = LB;        // look-back / flush warps (the flush expands every change)
    static constexpr int kStages = S;          // TMA ring stages (16 KiB prev + 16 KiB curr each)
    static constexpr int kBufs = B;            // ticket staging buffers (consumers may run ahead)
    static constexpr uint32_t kRecCap = RC;    // record mode: staged changed 16-byte vectors per buffer
    static constexpr uint32_t kStageCap = SC;  // element mode: staged changed elements per buffer
    static constexpr uint32_t kDenseTicket = DT;  // changes above which the next ticket stages element entries
    static constexpr uint32_t kDeferTicket = DF;  // ... above which it is only counted and deferred to K1b
};
#ifndef PULSE_K1_LB
#define PULSE_K1_LB 4
#endif
#ifndef PULSE_K1_DLB
#define PULSE_K1_DLB 4
#endif
#ifndef PULSE_K1_D2LB
#define PULSE_K1_D2LB 4
#endif
using SparseCfg = Cfg<PULSE_K1_STAGES, PULSE_K1_BUFS, PULSE_K1_RECCAP, PULSE_K1_STAGECAP,
                      (PULSE_K1_STAGECAP * 3 / 4 < 3072 ? PULSE_K1_STAGECAP * 3 / 4 : 3072), PULSE_K1_STAGECAP,
                      PULSE_K1_LB>;
// plans sized for < 1.5% changes: one more ticket in flight between the consumers and the
// flush group, smaller staging per ticket (99%: K1 4.50 -> 4.44 ms; at 98% it would overflow
// the staging: 5.1 -> 6.7 ms, so plans sized for more changes keep SparseCfg)
using SparseLowCfg = Cfg<5, 6, 384, 2304, 1728, 2304, PULSE_K1_LB>;
using DenseCfg = Cfg<PULSE_K1_DSTAGES, PULSE_K1_DBUFS, PULSE_K1_DRECCAP, PULSE_K1_DSTAGECAP, PULSE_K1_DDENSE,
                     PULSE_K1_DSTAGECAP, PULSE_K1_DLB>;
// patches denser than ~4.5%: records only (no element staging), larger record buffers, fewer
// stages; tickets too dense even for those are counted in K1 and written by K1b
using Dense2Cfg = Cfg<2, 3, 2200, 0, 0xFFFFFFFFu, 8000, PULSE_K1_D2LB>;
// patches denser than ~5.6%: the same staging and six flush warps -- at 90% the four-warp flush
// (expanding ~6,500 changes per ticket) was the bottleneck: K1 10.3 -> 9.0 ms; at 95% the extra
// warps cost more issue slots than they save (6.87 -> 7.00 ms), hence a separate shape
#ifndef PULSE_K1_D3S
#define PULSE_K1_D3S 2
#endif
#ifndef PULSE_K1_D3B
#define PULSE_K1_D3B 3
#endif
#ifndef PULSE_K1_D3RC
#define PULSE_K1_D3RC 2200
#endif
#ifndef PULSE_K1_D3LB
#define PULSE_K1_D3LB 6
#endif
using Dense3Cfg = Cfg<PULSE_K1_D3S, PULSE_K1_D3B, PULSE_K1_D3RC, 0, 0xFFFFFFFFu, 8000, PULSE_K1_D3LB>;
constexpr uint32_t kSubElems = 8192;                 // elements per stage (16 KiB + 16 KiB)
constexpr uint32_t kSubs = kTicketElems / kSubElems; // 8 sub-tiles per ticket
constexpr int kConsumerWarps = 8;
constexpr uint32_t kVecPerWarp = kSubElems / 8 / kConsumerWarps;  // 128 vectors = 4 per lane
constexpr int kProducerWarp = kConsumerWarps;        // warp 8
constexpr int kLbFirst = kConsumerWarps + 1;         // flush warps: 9 .. 9 + Cfg::kLbWarps - 1
constexpr int kLbWarpsMax = 8;
template <class C>
constexpr int threads_total() { return (kConsumerWarps + 1 + C::kLbWarps) * 32; }  // 416 with 4 flush warps
enum : uint32_t { kModeRecords = 0, kModeElements = 1, kModeCount = 2 };
constexpr uint32_t kChunks = kSubs * kConsumerWarps; // (sub-tile, warp) chunks per ticket
constexpr uint32_t kBarLb = 2;                       // named barrier id of the look-back group
static_assert(kVecPerWarp % 32 == 0, "whole vectors per lane");

struct StageDesc {
    uint64_t tile;          // ticket id, ~0 = end of stream
    const uint16_t* pp;     // sub-tile bases (for the < 8-element tail)
    const uint16_t* cp;
    uint32_t si, toff;      // segment, element offset of the ticket in the segment
    uint32_t sub, n_sub;    // sub-tile index within the ticket
    uint32_t elems;         // elements in this sub-tile
    uint32_t vec_bytes;     // bytes delivered by TMA (multiple of 16)
};

struct TicketInfo {
    uint64_t tile;
    uint32_t si, toff, n_sub;
};

template <class C>
struct Smem {
    static constexpr int kStages = C::kStages, kBufs = C::kBufs;
    static constexpr uint32_t kRecCap = C::kRecCap, kStageCap = C::kStageCap;
    uint4 prev[kStages][kSubElems / 8];
    uint4 curr[kStages][kSubElems / 8];
    // Staging, one buffer per ticket in flight, in one of two layouts chosen per
    // ticket (S.mode): records -- one per changed 16-byte vector, its 8 current
    // values and meta.x = vector index in the ticket | change mask << 16,
    // meta.y = (sub, warp) chunk | element offset of its first change in the
    // chunk << 8 (cheap per change; sparse tickets) -- or elements -- (offset in
    // ticket, value) per change (more changes per byte; dense tickets).
    union StageBuf {
        struct {
            uint4 val[kRecCap];
            uint2 meta[kRecCap];
        } rec;
        struct {
            uint16_t idx[kStageCap > 0 ? kStageCap : 1];
            uint16_t val[kStageCap > 0 ? kStageCap : 1];
        } el;
    } stg[kBufs];
    uint32_t chunk_off[kBufs][kChunks];  // where each (sub, warp) chunk was staged (first record / element)
    uint32_t chunk_cnt[kBufs][kChunks];  // changed elements per (sub, warp) chunk
    uint32_t chunk_ebase[kChunks];       // record mode (flush group): element scan at each chunk's first record
    uint32_t mode[kBufs];                // staging layout of the ticket in each buffer
    uint32_t chunk_pre[kChunks + 1]; // ordered prefix (look-back group)
    uint32_t fill[kBufs];            // staging bump allocator (records or elements)
    uint32_t overflow[kBufs];
    uint32_t tk_cnt[kBufs];          // ticket count, summed by the consumer warps
    uint32_t tk_arrived[kBufs];      // consumer warps done with the ticket
    uint32_t vcnt[kBufs];            // element mode: changed 16-byte vectors (what records would need)
    StageDesc desc[kStages];
    TicketInfo info[kBufs];
    uint64_t full[kStages], empty[kStages];
    uint64_t tk_full[kBufs], tk_empty[kBufs];
    uint32_t lb_warp_tot[kLbWarpsMax];
    uint32_t lb_run, lb_count;
    uint64_t lb_G;
};
static_assert(sizeof(Smem<SparseCfg>) <= 232448, "K1 shared memory exceeds the 227 KiB per-block limit");
static_assert(sizeof(Smem<SparseLowCfg>) <= 232448, "K1 shared memory exceeds the 227 KiB per-block limit");
static_assert(sizeof(Smem<DenseCfg>) <= 232448, "K1 shared memory exceeds the 227 KiB per-block limit");
static_assert(sizeof(Smem<Dense2Cfg>) <= 232448, "K1 shared memory exceeds the 227 KiB per-block limit");
static_assert(sizeof(Smem<Dense3Cfg>) <= 232448, "K1 shared memory exceeds the 227 KiB per-block limit");
}  // namespace tma

// Look-back with 4 status words per lane per round (128 predecessors).
__device__ __forceinline__ uint64_t lookback_wide(uint64_t* status, uint64_t tile, uint64_t agg) {
    const int lane = threadIdx.x & 31;
    uint64_t excl = 0;
    int64_t base = int64_t(tile) - 1;  // newest predecessor not yet consumed
    while (true) {
        uint64_t w[4];
        bool stop_here = false;
        int stop_k = 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t idx = base - (lane * 4 + k);
            uint64_t v = kStatPrefix;  // before tile 0: identity prefix
            if (idx >= 0) {
                uint64_t spins = 0;
                do {
                    v = ld_relaxed(status + idx);
                    if (++spins > kSpinLimit) {
                        watchdog_fire(3, tile, uint64_t(idx), v);
                        v = kStatPrefix;
                        break;
                    }
                } while ((v & 3) == kStatInvalid);
            }
            w[k] = v;
            if (!stop_here && (v & 3) == kStatPrefix) {
                stop_here = true;
                stop_k = k;
            }
        }
        const uint32_t pmask = __ballot_sync(0xffffffffu, stop_here);
        const int stop_lane = pmask ? __ffs(pmask) - 1 : 32;
        uint64_t v = 0;
        if (lane < stop_lane) {
#pragma unroll
            for (int k = 0; k < 4; ++k) v += w[k] >> 2;
        } else if (lane == stop_lane) {
#pragma unroll
            for (int k = 0; k < 4; ++k) v += k <= stop_k ? (w[k] >> 2) : 0;
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        excl += v;
        if (pmask) break;
        base -= 128;
    }
    if (lane == 0) st_relaxed(status + tile, ((excl + agg) << 2) | kStatPrefix);
    return excl;
}

template <class C>
__global__ void __launch_bounds__((tma::kConsumerWarps + 1 + C::kLbWarps) * 32, 1) k1_tma(K1Args k) {
    using namespace tma;
    constexpr int kStages = C::kStages, kBufs = C::kBufs;
    constexpr int kLbWarps = C::kLbWarps, kLbThreads = kLbWarps * 32;
    static_assert(kLbWarps >= 1 && kLbWarps <= kLbWarpsMax, "flush warps");
    constexpr uint32_t kRecCap = C::kRecCap, kStageCap = C::kStageCap, kDenseTicket = C::kDenseTicket;
    constexpr uint32_t kDeferTicket = C::kDeferTicket;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    tma::Smem<C>& S = *reinterpret_cast<tma::Smem<C>*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&S.full[i], 1);
            mbar_init(&S.empty[i], kConsumerWarps);
        }
        for (int i = 0; i < kBufs; ++i) {
            mbar_init(&S.tk_full[i], kConsumerWarps);
            mbar_init(&S.tk_empty[i], 1);
            S.fill[i] = 0;
            S.overflow[i] = 0;
            S.mode[i] = kModeRecords;
            S.tk_cnt[i] = 0;
            S.tk_arrived[i] = 0;
            S.vcnt[i] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kProducerWarp) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            while (true) {
                const uint64_t tile = atomicAdd(k.ticket, 1ull);
                if (tile >= k.n_tiles) {
                    mbar_wait(&S.empty[stage], phase ^ 1);
                    S.desc[stage].tile = ~0ull;
                    mbar_arrive(&S.full[stage]);
                    break;
                }
                if (k.trace) k.trace[tile] = (blockIdx.x << 8) | 1u;
                const uint32_t si = k.tile_seg[tile];
                const SegDesc sd = k.segs[si];
                const uint32_t toff = uint32_t((tile - sd.ticket_start) * kTicketElems);
                const uint32_t nin = min(kTicketElems, sd.numel - toff);
                const uint16_t* pp = k.prev_ptrs[sd.tensor] + sd.elem_off + toff;
                const uint16_t* cp = k.curr_ptrs[sd.tensor] + sd.elem_off + toff;
                const uint32_t n_sub = (nin + kSubElems - 1) / kSubElems;
                for (uint32_t sub = 0; sub < n_sub; ++sub) {
                    mbar_wait(&S.empty[stage], phase ^ 1);
                    StageDesc& d = S.desc[stage];
                    d.tile = tile;
                    d.si = si;
                    d.toff = toff;
                    d.sub = sub;
                    d.n_sub = n_sub;
                    d.elems = min(kSubElems, nin - sub * kSubElems);
                    d.pp = pp + sub * kSubElems;
                    d.cp = cp + sub * kSubElems;
                    d.vec_bytes = (d.elems * 2) & ~15u;
                    if (d.vec_bytes) {
                        mbar_arrive_tx(&S.full[stage], 2 * d.vec_bytes);
                        tma_load_1d(S.prev[stage], d.pp, d.vec_bytes, &S.full[stage]);
                        tma_load_1d(S.curr[stage], d.cp, d.vec_bytes, &S.full[stage]);
                    } else {
                        mbar_arrive(&S.full[stage]);
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        return;
    }

    if (warp < kConsumerWarps) {
        // ------------------------------------------------------------ consumers
        // Warp w owns vectors [w*128, (w+1)*128) of every sub-tile, lane l the
        // vectors w*128 + 32 j + l: each warp's slice is contiguous, so it is
        // compacted with warp-level scans only -- no CTA barrier per sub-tile.
        int stage = 0, buf = 0;
        uint32_t phase = 0, bphase = 0;
        uint32_t wcount = 0;  // this warp's changes in the current ticket
        uint32_t tmode = kModeRecords;  // staging layout of the current ticket
        // Last warp of a ticket publishes its aggregate right away, so other CTAs'
        // look-backs never wait on this CTA's look-back group.
        auto finish_ticket = [&](const StageDesc& d) {
            __syncwarp();
            if (lane == 0) {
                if (warp == 0) {
                    if (k.trace) atomicOr(k.trace + d.tile, 2u);
                    TicketInfo& ti = S.info[buf];
                    ti.tile = d.tile;
                    ti.si = d.si;
                    ti.toff = d.toff;
                    ti.n_sub = d.n_sub;
                }
                atomicAdd(&S.tk_cnt[buf], wcount);
                __threadfence_block();
                if (atomicAdd(&S.tk_arrived[buf], 1u) == kConsumerWarps - 1) {
                    const uint32_t count = atomicAdd(&S.tk_cnt[buf], 0u);
                    if (d.tile == 0) st_relaxed(k.status, (uint64_t(count) << 2) | kStatPrefix);
                    else st_relaxed(k.status + d.tile, (uint64_t(count) << 2) | kStatAggregate);
                    if (k.trace) atomicOr(k.trace + d.tile, 4u);
                }
                mbar_arrive(&S.tk_full[buf]);  // release: staging + chunk table + info visible
            }
            wcount = 0;
            if (++buf == kBufs) {
                buf = 0;
                bphase ^= 1;
            }
        };
        while (true) {
            mbar_wait(&S.full[stage], phase);
            const StageDesc d = S.desc[stage];
            if (d.tile == ~0ull) {
                // End of stream.  Every warp first waits until `buf` is free, like at a
                // ticket start: warps can be skewed by several 1-sub-tile tickets, and an
                // early arrival would otherwise complete the previous ticket's phase.
                if (lane == 0) {
                    mbar_wait(&S.tk_empty[buf], bphase ^ 1);
                    if (warp == 0) S.info[buf].tile = ~0ull;
                    mbar_arrive(&S.tk_full[buf]);
                }
                break;
            }
            if (k.experiment == 1) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[stage]);
                if (d.sub + 1 == d.n_sub) {
                    if (lane == 0) {
                        if (warp == 0) {
                            S.chunk_cnt[buf][0] = 0;
                            TicketInfo& ti = S.info[buf];
                            ti.tile = d.tile; ti.si = d.si; ti.toff = d.toff; ti.n_sub = 1;
                        }
                    }
                }
                if (++stage == kStages) { stage = 0; phase ^= 1; }
                continue;
            }
            if (d.sub == 0) {
                mbar_wait(&S.tk_empty[buf], bphase ^ 1);  // staging buffer flushed
                tmode = S.mode[buf];
            }
            uint4 av[kVecPerWarp / 32], cv[kVecPerWarp / 32];
            const uint32_t v0 = warp * kVecPerWarp + lane;
            if (d.vec_bytes == kSubElems * 2) {  // full sub-tile (block-uniform)
#pragma unroll
                for (int j = 0; j < int(kVecPerWarp / 32); ++j) {
                    av[j] = S.prev[stage][v0 + 32 * j];
                    cv[j] = S.curr[stage][v0 + 32 * j];
                }
            } else {
#pragma unroll
                for (int j = 0; j < int(kVecPerWarp / 32); ++j) {
                    const uint32_t v = v0 + 32 * j, e = v * 8;
                    uint4 a = make_uint4(0, 0, 0, 0), b = a;
                    if ((v + 1) * 16 <= d.vec_bytes) {
                        a = S.prev[stage][v];
                        b = S.curr[stage][v];
                    } else if (e < d.elems) {  // < 8-element tail, straight from global
                        uint32_t ta[4] = {0, 0, 0, 0}, tb[4] = {0, 0, 0, 0};
                        for (uint32_t q = 0; q < 8 && e + q < d.elems; ++q) {
                            ta[q >> 1] |= uint32_t(d.pp[e + q]) << ((q & 1) * 16);
                            tb[q >> 1] |= uint32_t(d.cp[e + q]) << ((q & 1) * 16);
                        }
                        a = make_uint4(ta[0], ta[1], ta[2], ta[3]);
                        b = make_uint4(tb[0], tb[1], tb[2], tb[3]);
                    }
                    av[j] = a;
                    cv[j] = b;
                }
            }
            // any difference per vector? (XOR-OR, LOP3-fusable)
            uint32_t xd[kVecPerWarp / 32], diff = 0;
#pragma unroll
            for (int j = 0; j < int(kVecPerWarp / 32); ++j) {
                xd[j] = (av[j].x ^ cv[j].x) | (av[j].y ^ cv[j].y) | (av[j].z ^ cv[j].z) | (av[j].w ^ cv[j].w);
                diff |= xd[j];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[stage]);  // operands are in registers: stage may be refilled
            const bool warp_changed = __any_sync(0xffffffffu, diff != 0);
            // per-element masks only for the vector groups some lane changed in (clustered
            // updates usually touch one of the four); rbj[j] = lanes with a changed vector j
            uint32_t m[kVecPerWarp / 32] = {0, 0, 0, 0}, rbj[kVecPerWarp / 32] = {0, 0, 0, 0};
            if (warp_changed) {
#pragma unroll
                for (int j = 0; j < int(kVecPerWarp / 32); ++j) {
                    rbj[j] = __ballot_sync(0xffffffffu, xd[j] != 0);
                    if (rbj[j] && xd[j]) m[j] = change_mask(av[j], cv[j]);
                }
            }
            if (!warp_changed) {  // common case at high sparsity: nothing to stage
                if (lane == 0) S.chunk_cnt[buf][d.sub * kConsumerWarps + warp] = 0;
                if (d.sub + 1 == d.n_sub) finish_ticket(d);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
                continue;
            }

            const uint32_t chunk = d.sub * kConsumerWarps + warp;
            if (tmode == kModeCount) {
                // deferred ticket: counted here, written by K1b (k1_deferred) after K1
                const uint32_t total = __reduce_add_sync(0xffffffffu, __popc(m[0]) + __popc(m[1]) + __popc(m[2]) +
                                                                          __popc(m[3]));
                if (lane == 0) {
                    S.chunk_cnt[buf][chunk] = total;
                    if (total) S.overflow[buf] = 1;
                }
                wcount += total;
            } else if (tmode == kModeRecords) {
                // one record per changed vector, records in (j, lane) order = element
                // order; the flush group derives each record's element offset, so the
                // consumers only need the chunk total (one warp reduction)
                const uint32_t total = __reduce_add_sync(0xffffffffu, __popc(m[0]) + __popc(m[1]) + __popc(m[2]) +
                                                                          __popc(m[3]));
                uint32_t rb[4], nrec = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    rb[j] = rbj[j];  // m[j] != 0 exactly when vector j differs
                    nrec += __popc(rb[j]);
                }
                uint32_t off = 0;
                if (lane == 0 && nrec) off = atomicAdd(&S.fill[buf], nrec);
                off = __shfl_sync(0xffffffffu, off, 0);
                if (lane == 0) {
                    S.chunk_cnt[buf][chunk] = total;
                    S.chunk_off[buf][chunk] = off;  // first record of the chunk
                    if (off + nrec > kRecCap) S.overflow[buf] = 1;
                }
                if (k.experiment != 3) {
                    const uint32_t lt_mask = (1u << lane) - 1u;
                    uint32_t rbase = off;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (m[j]) {
                            const uint32_t r = rbase + __popc(rb[j] & lt_mask);
                            if (r < kRecCap) {
                                const uint32_t vec = d.sub * (kSubElems / 8) + v0 + 32 * j;
                                S.stg[buf].rec.val[r] = cv[j];
                                S.stg[buf].rec.meta[r] = make_uint2(vec | (m[j] << 16), chunk);
                            }
                        }
                        rbase += __popc(rb[j]);
                    }
                }
                wcount += total;
            } else {
                // element entries (offset in ticket, value), chunk-contiguous; element
                // order inside the warp slice: (j, lane, q), packed 16-bit scans for j pairs
                const uint32_t lo = __popc(m[0]) | (__popc(m[1]) << 16);
                const uint32_t hi = __popc(m[2]) | (__popc(m[3]) << 16);
                uint32_t ilo = lo, ihi = hi;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t a1 = __shfl_up_sync(0xffffffffu, ilo, off);
                    const uint32_t a2 = __shfl_up_sync(0xffffffffu, ihi, off);
                    if (lane >= off) {
                        ilo += a1;
                        ihi += a2;
                    }
                }
                const uint32_t tlo = __shfl_sync(0xffffffffu, ilo, 31), thi = __shfl_sync(0xffffffffu, ihi, 31);
                const uint32_t t0 = tlo & 0xFFFF, t1 = tlo >> 16, t2 = thi & 0xFFFF, t3 = thi >> 16;
                const uint32_t total = t0 + t1 + t2 + t3;
                const uint32_t exlo = ilo - lo, exhi = ihi - hi;
                const uint32_t pj[4] = {exlo & 0xFFFF, t0 + (exlo >> 16), t0 + t1 + (exhi & 0xFFFF),
                                        t0 + t1 + t2 + (exhi >> 16)};
                uint32_t off = 0;
                if (lane == 0 && total) {
                    off = atomicAdd(&S.fill[buf], total);
                    atomicAdd(&S.vcnt[buf], __popc(rbj[0]) + __popc(rbj[1]) + __popc(rbj[2]) + __popc(rbj[3]));
                }
                off = __shfl_sync(0xffffffffu, off, 0);
                if (lane == 0) {
                    S.chunk_off[buf][chunk] = off;
                    S.chunk_cnt[buf][chunk] = total;
                    if (off + total > kStageCap) S.overflow[buf] = 1;
                }
                if (total && k.experiment != 3) {
                    // warp-cooperative staging pays off when some vector holds several
                    // changes (the per-lane loop over mask bits would diverge); with at most
                    // PULSE_K1_COOP_MIN_BITS changes per vector (scattered changes) the plain
                    // per-lane loop is cheaper (99% with cluster width 1: K1 12.3 -> 9.0 ms)
                    const uint32_t vmax = __reduce_max_sync(
                        0xffffffffu, max(max(__popc(m[0]), __popc(m[1])), max(__popc(m[2]), __popc(m[3]))));
                    if (PULSE_K1_COOP_STAGE && vmax > PULSE_K1_COOP_MIN_BITS) {
                    // warp-cooperative: slot s of vector group j (element order: lane, then
                    // bit) is filled by lane s % 32 in round s / 32.  Its owner is the first
                    // lane whose inclusive count exceeds s (binary lifting over shuffles), its
                    // element the (s - owner's exclusive count)-th set bit of the owner's mask
                    // -- no per-lane loop over mask bits, so no divergence on dense vectors.
                    const uint32_t tj[4] = {t0, t1, t2, t3};
                    uint32_t pbase = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (tj[j]) {
                            const uint32_t incl = pj[j] - pbase + __popc(m[j]);
                            for (uint32_t s0 = 0; s0 < tj[j]; s0 += 32) {
                                const uint32_t s = s0 + uint32_t(lane);
                                uint32_t own = 0;
#pragma unroll
                                for (uint32_t step = 16; step; step >>= 1)
                                    if (__shfl_sync(0xffffffffu, incl, int(own + step - 1)) <= s) own += step;
                                const int src = int(own & 31);
                                const uint32_t om = __shfl_sync(0xffffffffu, m[j], src);
                                const uint32_t oin = __shfl_sync(0xffffffffu, incl, src);
                                const uint32_t w0 = __shfl_sync(0xffffffffu, cv[j].x, src);
                                const uint32_t w1 = __shfl_sync(0xffffffffu, cv[j].y, src);
                                const uint32_t w2 = __shfl_sync(0xffffffffu, cv[j].z, src);
                                const uint32_t w3 = __shfl_sync(0xffffffffu, cv[j].w, src);
                                if (s < tj[j]) {
                                    uint32_t r = s - (oin - __popc(om)), q = 0;  // r-th set bit of om
                                    uint32_t c = __popc(om & 0xFu);
                                    if (r >= c) { q = 4; r -= c; }
                                    c = __popc((om >> q) & 3u);
                                    if (r >= c) { q += 2; r -= c; }
                                    if (r >= ((om >> q) & 1u)) q += 1;
                                    const uint32_t w = q < 4 ? (q < 2 ? w0 : w1) : (q < 6 ? w2 : w3);
                                    const uint32_t pos = off + pbase + s;
                                    if (pos < kStageCap) {
                                        S.stg[buf].el.idx[pos] =
                                            uint16_t(d.sub * kSubElems + (warp * kVecPerWarp + uint32_t(src) + 32 * j) * 8 + q);
                                        S.stg[buf].el.val[pos] = uint16_t(w >> ((q & 1) * 16));
                                    }
                                }
                            }
                        }
                        pbase += tj[j];
                    }
                    } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint32_t mm = m[j];
                        uint32_t pos = off + pj[j];
                        const uint32_t e = d.sub * kSubElems + (v0 + 32 * j) * 8;
                        while (mm) {
                            const int q = __ffs(mm) - 1;
                            mm &= mm - 1;
                            if (pos < kStageCap) {
                                S.stg[buf].el.idx[pos] = uint16_t(e + q);
                                S.stg[buf].el.val[pos] = lane_value(cv[j], q);
                            }
                            ++pos;
                        }
                    }
                    }
                }
                wcount += total;
            }
            if (d.sub + 1 == d.n_sub) finish_ticket(d);
            if (++stage == kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
        return;
    }

    // ---------------------------------------------------------------- look-back group
    const int lt = tid - kLbFirst * 32;  // 0 .. kLbThreads - 1
    int buf = 0;
    uint32_t bphase = 0;
    while (true) {
        mbar_wait(&S.tk_full[buf], bphase);
        const TicketInfo ti = S.info[buf];
        if (ti.tile == ~0ull) break;
        const uint32_t nch = ti.n_sub * kConsumerWarps;
        if (warp == kLbFirst) {
            // ordered chunk prefix (kChunks = 64: two per lane) and the ticket count
            const uint32_t c0 = 2 * lane < nch ? S.chunk_cnt[buf][2 * lane] : 0;
            const uint32_t c1 = 2 * lane + 1 < nch ? S.chunk_cnt[buf][2 * lane + 1] : 0;
            uint32_t inc = c0 + c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += x;
            }
            const uint32_t ex = inc - c0 - c1;
            S.chunk_pre[2 * lane] = ex;
            S.chunk_pre[2 * lane + 1] = ex + c0;
            const uint32_t count = __shfl_sync(0xffffffffu, inc, 31);
            if (lane == 31) S.chunk_pre[kChunks] = count;
            // (the aggregate was published by the last consumer warp)
            const bool seg_first = ti.toff == 0;
            const bool last = ti.tile == k.n_tiles - 1;
            uint64_t G = 0;
            if ((count > 0 || seg_first || last) && ti.tile > 0) G = lookback_wide(k.status, ti.tile, count);
            if (lane == 0) {
                if (k.trace) atomicOr(k.trace + ti.tile, 8u);
                S.lb_G = G;
                S.lb_count = count;
                if (seg_first) k.seg_start[ti.si] = G;
                if (last) k.seg_start[k.n_segs] = G + count;
            }
        }
        named_sync(kBarLb, kLbThreads);
        const uint64_t G = S.lb_G;
        const uint32_t count = S.lb_count;
        if (k.experiment == 2 || k.experiment == 3) {
            // attribution experiments: no write-back
        } else if (k.experiment == 4) {
            // attribution: the same bytes written coalesced (consecutive threads, consecutive outputs)
            for (uint32_t i = lt; i < count; i += kLbThreads) {
                const uint64_t pos = G + i;
                if (pos < k.capacity) {
                    k.out_idx[pos] = i;
                    k.out_val[pos] = 0;
                }
            }
        } else if (!S.overflow[buf] && S.mode[buf] == kModeRecords) {
            // expand the staged records: record -> its changed elements at G + its
            // chunk's element prefix + its offset in the chunk.  Records sit in the
            // buffer chunk by chunk (each chunk contiguous, in element order), so a
            // running scan of popc(mask) in buffer order, minus its value at the
            // chunk's first record, is that offset.
            const uint32_t nrec = S.fill[buf];
            uint32_t run = 0;  // elements of the records before this round
            for (uint32_t r0 = 0; r0 < nrec; r0 += kLbThreads) {
                const uint32_t r = r0 + uint32_t(lt);
                uint2 meta = make_uint2(0, 0);
                uint4 v = make_uint4(0, 0, 0, 0);
                uint32_t cnt = 0;
                if (r < nrec) {
                    meta = S.stg[buf].rec.meta[r];
                    v = S.stg[buf].rec.val[r];
                    cnt = __popc(meta.x >> 16);
                }
                uint32_t inc = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += x;
                }
                if (lane == 31) S.lb_warp_tot[warp - kLbFirst] = inc;
                named_sync(kBarLb, kLbThreads);
                uint32_t before = 0, all = 0;
#pragma unroll
                for (int w = 0; w < kLbWarps; ++w) {
                    const uint32_t t = S.lb_warp_tot[w];
                    if (w < warp - kLbFirst) before += t;
                    all += t;
                }
                const uint32_t ex = run + before + inc - cnt;  // elements before record r (buffer order)
                const uint32_t ch = meta.y & 0xFF;
                if (r < nrec && S.chunk_off[buf][ch] == r) S.chunk_ebase[ch] = ex;
                named_sync(kBarLb, kLbThreads);  // chunk_ebase complete for this round's chunk starts
                if (r < nrec) S.stg[buf].rec.meta[r].y = ch | (ex << 8);
                run += all;
            }
            named_sync(kBarLb, kLbThreads);
            for (uint32_t r = lt; r < nrec; r += kLbThreads) {
                const uint2 meta = S.stg[buf].rec.meta[r];
                const uint4 v = S.stg[buf].rec.val[r];
                const uint32_t vec = meta.x & 0xFFFF, mask = meta.x >> 16, ch = meta.y & 0xFF;
                uint64_t pos = G + S.chunk_pre[ch] + ((meta.y >> 8) - S.chunk_ebase[ch]);
                const uint32_t ebase = ti.toff + vec * 8;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (mask & (1u << q)) {
                        if (pos < k.capacity) {
                            k.out_idx[pos] = ebase + q;
                            k.out_val[pos] = lane_value(v, q);
                        }
                        ++pos;
                    }
                }
            }
        } else if (!S.overflow[buf]) {
            if (PULSE_K1_FLAT_FLUSH && count < PULSE_K1_FLAT_FLUSH * nch) {
                // few entries per chunk (scattered changes): every flush thread takes entries of
                // the whole ticket in order, finding each one's chunk by a binary search of the
                // chunk prefix -- no per-chunk rounds that leave most lanes idle
                for (uint32_t i = uint32_t(lt); i < count; i += kLbThreads) {
                    uint32_t lo = 0, hi = nch;  // last chunk c with chunk_pre[c] <= i
                    while (hi - lo > 1) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (S.chunk_pre[mid] <= i) lo = mid;
                        else hi = mid;
                    }
                    const uint32_t off = S.chunk_off[buf][lo] + (i - S.chunk_pre[lo]);
                    const uint64_t pos = G + i;
                    if (pos < k.capacity) {
                        k.out_idx[pos] = ti.toff + S.stg[buf].el.idx[off];
                        k.out_val[pos] = S.stg[buf].el.val[off];
                    }
                }
            } else {
            // element mode: each chunk's staged entries are contiguous and go to
            // G + chunk_pre[c] onward -- one warp per chunk, lanes over its entries
            // (coalesced stores, no per-entry search for the chunk)
            for (uint32_t c = uint32_t(warp - kLbFirst); c < nch; c += kLbWarps) {
                const uint32_t base = S.chunk_pre[c], cnt = S.chunk_pre[c + 1] - base;
                const uint32_t off = S.chunk_off[buf][c];
                for (uint32_t i = lane; i < cnt; i += 32) {
                    const uint64_t pos = G + base + i;
                    if (pos < k.capacity) {
                        k.out_idx[pos] = ti.toff + S.stg[buf].el.idx[off + i];
                        k.out_val[pos] = S.stg[buf].el.val[off + i];
                    }
                }
            }
            }
        } else if (lt == 0 && count > 0) {
            // staging overflowed (or the ticket was only counted): K1b writes this ticket after
            // K1 from a list of (ticket, output offset), with the whole GPU's memory parallelism
            // -- re-streaming it here would stall the ring behind four warps
            const unsigned long long slot = atomicAdd(k.n_defer, 1ull);
            k.defer[slot] = make_ulonglong2(ti.tile, G);
        }
        named_sync(kBarLb, kLbThreads);  // flush done before the buffer is reused
        if (lt == 0) {
            if (k.trace) atomicOr(k.trace + ti.tile, 16u);
            // changed vectors staged (or asked for) in record mode: scattered changes (one per
            // 16-byte vector) overflow the records long before the element count is "dense"
            const bool rec_overflow = S.mode[buf] == kModeRecords && S.fill[buf] > kRecCap;
            // ... and stays there while its changed vectors would not fit the records either
            // (no records / elements ping-pong that defers every other ticket; clustered changes,
            // several per vector, go back to records)
            const bool el_keep = S.mode[buf] == kModeElements && S.vcnt[buf] > kRecCap;
            S.vcnt[buf] = 0;
            S.fill[buf] = 0;
            S.overflow[buf] = 0;
            // layout for the next ticket staged in this buffer: neighbouring tickets
            // have similar density (same tensor), so follow this one's
            S.mode[buf] = count > kDeferTicket                                  ? kModeCount
                          : (count > kDenseTicket || (kStageCap > 0 && (rec_overflow || el_keep))) ? kModeElements
                                                                                  : kModeRecords;
            S.tk_cnt[buf] = 0;
            S.tk_arrived[buf] = 0;
            mbar_arrive(&S.tk_empty[buf]);
        }
        if (++buf == kBufs) {
            buf = 0;
            bphase ^= 1;
        }
    }
}

// K1b: the deferred tickets -- dense beyond what K1's staging holds.  K1 counted them
// and its look-back placed them (output offset G); here a CTA re-streams one ticket at
// a time (8 loads of 16 bytes in flight per thread, several CTAs per SM) and writes
// every change at G + its ordered position.  Nothing to do (one atomic per CTA) when
// no ticket was deferred -- the common case for sparse patches.
constexpr int kDeferThreads = 256;
__global__ void __launch_bounds__(kDeferThreads, 3) k1_deferred(K1Args k, const uint64_t* __restrict__ n_defer,
                                                             unsigned long long* __restrict__ cursor) {
    __shared__ uint32_t s_warp[kDeferThreads / 32];
    __shared__ uint64_t s_t;
    __shared__ uint32_t s_out[32 * kDeferThreads];  // a round's changes: (offset in round << 16) | value
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = *n_defer;
    while (true) {
        if (tid == 0) s_t = atomicAdd(cursor, 1ull);
        __syncthreads();
        const uint64_t t = s_t;
        __syncthreads();
        if (t >= n) return;
        const ulonglong2 dt = k.defer[t];
        const uint64_t tile = dt.x;
        const uint32_t si = k.tile_seg[tile];
        const SegDesc sd = k.segs[si];
        const uint32_t toff = uint32_t((tile - sd.ticket_start) * kTicketElems);
        const uint32_t nin = min(kTicketElems, sd.numel - toff);
        const uint16_t* pp = k.prev_ptrs[sd.tensor] + sd.elem_off + toff;
        const uint16_t* cp = k.curr_ptrs[sd.tensor] + sd.elem_off + toff;
        uint64_t pos0 = dt.y;
        // rounds of 8192 elements: thread `tid` compares elements [32 tid, 32 tid + 32) of the
        // round; the next round's 8 loads are issued before this round is compacted and written
        auto load_round = [&](uint32_t r0, uint4 (&a)[4], uint4 (&c)[4]) {
            const uint32_t e = r0 + 32 * uint32_t(tid);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t ej = e + 8 * j;
                if (ej + 8 <= nin) {
                    a[j] = ld_stream(pp + ej);
                    c[j] = ld_stream(cp + ej);
                } else {
                    uint32_t ta[4] = {0, 0, 0, 0}, tb[4] = {0, 0, 0, 0};
                    for (uint32_t q = 0; q < 8 && ej + q < nin; ++q) {
                        ta[q >> 1] |= uint32_t(pp[ej + q]) << ((q & 1) * 16);
                        tb[q >> 1] |= uint32_t(cp[ej + q]) << ((q & 1) * 16);
                    }
                    a[j] = make_uint4(ta[0], ta[1], ta[2], ta[3]);
                    c[j] = make_uint4(tb[0], tb[1], tb[2], tb[3]);
                }
            }
        };
        uint4 na[4], nc[4];
        load_round(0, na, nc);
        for (uint32_t r0 = 0; r0 < nin; r0 += 32 * kDeferThreads) {
            uint4 a[4], c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                a[j] = na[j];
                c[j] = nc[j];
            }
            if (r0 + 32 * kDeferThreads < nin) load_round(r0 + 32 * kDeferThreads, na, nc);
            uint32_t m[4], cnt = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                m[j] = change_mask(a[j], c[j]);
                cnt += __popc(m[j]);
            }
            uint32_t inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += x;
            }
            if (lane == 31) s_warp[warp] = inc;
            __syncthreads();
            uint32_t before = 0, all = 0;
#pragma unroll
            for (int w = 0; w < kDeferThreads / 32; ++w) {
                const uint32_t x = s_warp[w];
                before += w < warp ? x : 0u;
                all += x;
            }
            // compact the round into shared memory (element order), then write it out with
            // consecutive threads on consecutive outputs (coalesced; per-thread runs would
            // scatter every store instruction over 32 sectors)
            uint32_t o = before + inc - cnt;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t mm = m[j];
                while (mm) {
                    const int q = __ffs(mm) - 1;
                    mm &= mm - 1;
                    s_out[o++] = (uint32_t(32 * tid + 8 * j + q) << 16) | lane_value(c[j], q);
                }
            }
            __syncthreads();
            for (uint32_t i = tid; i < all; i += kDeferThreads) {
                const uint64_t pos = pos0 + i;
                if (pos < k.capacity) {
                    const uint32_t w = s_out[i];
                    k.out_idx[pos] = toff + r0 + (w >> 16);
                    k.out_val[pos] = uint16_t(w);
                }
            }
            __syncthreads();  // s_warp / s_out are rewritten next round
            pos0 += all;
        }
    }
}

// Scan summary: totals, capacity status, and the FLAT gap base of the last
// changed tensor (needed by the next shard's first entry).
__global__ void k1_finalize(const SegDesc* __restrict__ segs, uint32_t n_segs,
                            const uint64_t* __restrict__ numel, uint64_t* __restrict__ seg_start,
                            const uint32_t* __restrict__ idx32, uint64_t capacity,
                            pulse_scan_summary* out, pulse_scan_summary* copy_out) {
    if (threadIdx.x != 0) return;
    if (n_segs == 0) seg_start[0] = 0;  // a plan with no tensors (a shard with none): K1 did not run
    const uint64_t n = seg_start[n_segs];
    pulse_scan_summary s;
    s.n_changes = n;
    s.has_change = n > 0;
    s.status = n > capacity ? PULSE_E_CAPACITY : 0;
    s.last_gap_base = 0;
    if (n > 0 && n <= capacity) {
        const uint64_t i = n - 1;
        const uint32_t sg = upper_index<uint64_t>(seg_start, 0, n_segs, i);
        const SegDesc sd = segs[sg];
        s.last_gap_base = numel[sd.tensor] - (sd.elem_off + idx32[i]);
    }
    *out = s;
    if (copy_out) *copy_out = s;
}

// =============================================================================================
// launchers
// =============================================================================================
static PerDeviceInt g_sms;
void debug_sync(const char* kernel, cudaStream_t s) {
    static const bool on = [] {
        const char* e = getenv("PULSE_DEBUG_SYNC");
        return e && *e && *e != '0';
    }();
    if (!on) return;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) fprintf(stderr, "[pulse debug] %s: %s\n", kernel, cudaGetErrorString(e));
}

int sm_count() {
    int& n = g_sms.here();
    if (!n) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device());
        n = v > 0 ? v : 148;
    }
    return n;
}

// PULSE_K1 = tma (default) | static | ticket
static int k1_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PULSE_K1");
        const std::string s = e ? e : "tma";
        v = s == "ticket" ? 1 : s == "static" ? 2 : 0;
    }
    return v;
}

void launch_encode_scan(const PlanDev& p, uint32_t curr_slot, uint32_t prev_slot, pulse_scan_summary* copy_out,
                        cudaStream_t s) {
    // status words + ticket must start at zero each launch (the TMA kernel's status words are
    // per 65536-element ticket: 8x fewer than the 8192-element tiles of the other variants)
    const bool tma_path = k1_variant() == 0 && p.tma_tiles > 0;
    cudaMemsetAsync(p.k1_status, 0, (tma_path ? p.tma_tiles : p.n_tiles) * sizeof(uint64_t), s);
    cudaMemsetAsync(p.counters, 0, 8 * sizeof(uint64_t), s);
    static const int experiment = getenv("PULSE_K1_EXPERIMENT") ? atoi(getenv("PULSE_K1_EXPERIMENT")) : 0;
    K1Args k{p.trace, experiment, p.segs, p.tile_seg, p.n_segs, p.n_tiles, p.slot[prev_slot], p.slot[curr_slot], p.idx32, p.val16,
             p.cap, p.seg_start, p.k1_status, reinterpret_cast<unsigned long long*>(p.counters),
             p.k1_defer, reinterpret_cast<unsigned long long*>(p.counters + 1)};
    if (p.n_tiles > 0) {
        static PerDeviceInt occ_static, occ_ticket, tma_attr;
        int& per_sm_static = occ_static.here();
        int& per_sm_ticket = occ_ticket.here();
        if (!per_sm_static) {
            int a = 0, b = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k1_static, kThreads, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_ticket, kThreads, 0);
            per_sm_ticket = b;
            per_sm_static = a > 0 ? a : -1;  // nonzero: configured
        }
        bool launched = false;
        if (k1_variant() == 0 && p.tma_tiles > 0) {
            int& attr = tma_attr.here();
            if (!attr) {
                cudaFuncSetAttribute(k1_tma<tma::SparseCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(tma::Smem<tma::SparseCfg>)));
                cudaFuncSetAttribute(k1_tma<tma::SparseLowCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(tma::Smem<tma::SparseLowCfg>)));
                cudaFuncSetAttribute(k1_tma<tma::DenseCfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(tma::Smem<tma::DenseCfg>)));
                cudaFuncSetAttribute(k1_tma<tma::Dense2Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(tma::Smem<tma::Dense2Cfg>)));
                cudaFuncSetAttribute(k1_tma<tma::Dense3Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(tma::Smem<tma::Dense3Cfg>)));
                attr = 1;
            }
            K1Args kt = k;
            kt.n_tiles = p.tma_tiles;
            kt.tile_seg = p.tma_tile_seg;
            const uint64_t grid = std::min<uint64_t>(uint64_t(sm_count()), p.tma_tiles);
            // the plan's change capacity says which regime the caller sized it for: >= 3% of its
            // elements -> dense staging (element entries need room), else more tickets in flight
            const int shape_override = [] {  // PULSE_K1_SHAPE=sparse|sparse_low|dense|dense2|dense3 (tests, A/B runs; per launch)
                const char* e = getenv("PULSE_K1_SHAPE");
                return !e ? -1 : std::string(e) == "dense3" ? 3 : std::string(e) == "dense2" ? 2
                               : std::string(e) == "dense" ? 1 : std::string(e) == "sparse" ? 0
                               : std::string(e) == "sparse_low" ? 4 : -1;
            }();
            const int shape = shape_override >= 0 ? shape_override : int(p.k1_dense);
            if (shape == 4) {
                k1_tma<tma::SparseLowCfg><<<unsigned(grid), tma::threads_total<tma::SparseLowCfg>(), sizeof(tma::Smem<tma::SparseLowCfg>), s>>>(kt);
            } else if (shape == 3) {
                k1_tma<tma::Dense3Cfg><<<unsigned(grid), tma::threads_total<tma::Dense3Cfg>(), sizeof(tma::Smem<tma::Dense3Cfg>), s>>>(kt);
            } else if (shape == 2) {
                k1_tma<tma::Dense2Cfg><<<unsigned(grid), tma::threads_total<tma::Dense2Cfg>(), sizeof(tma::Smem<tma::Dense2Cfg>), s>>>(kt);
            } else if (shape == 1) {
                k1_tma<tma::DenseCfg><<<unsigned(grid), tma::threads_total<tma::DenseCfg>(), sizeof(tma::Smem<tma::DenseCfg>), s>>>(kt);
            } else {
                k1_tma<tma::SparseCfg><<<unsigned(grid), tma::threads_total<tma::SparseCfg>(), sizeof(tma::Smem<tma::SparseCfg>), s>>>(kt);
            }
            PULSE_LAUNCHED("k1_tma", s);
            // K1b only if some ticket was deferred (a conditional graph node under capture;
            // eagerly it launches and returns at once on an empty list)
            launch_gated(s, reinterpret_cast<const uint32_t*>(p.counters + 1), [&](cudaStream_t gs) {
                k1_deferred<<<unsigned(sm_count() * 6), kDeferThreads, 0, gs>>>(
                    kt, p.counters + 1, reinterpret_cast<unsigned long long*>(p.counters + 2));
                PULSE_LAUNCHED("k1_deferred", gs);
            });
            launched = true;
        }
        if (!launched && k1_variant() == 2 && per_sm_static > 0) {
            const uint64_t grid = std::min<uint64_t>(uint64_t(per_sm_static) * sm_count(), p.n_tiles);
            void* args[] = {&k};
            launched = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k1_static), dim3(unsigned(grid)),
                                                   dim3(kThreads), args, 0, s) == cudaSuccess;
            if (!launched) cudaGetLastError();  // clear, fall back to tickets
        }
        if (!launched) {
            const uint64_t grid = std::min<uint64_t>(uint64_t(std::max(1, per_sm_ticket)) * sm_count(), p.n_tiles);
            k1_ticket<<<unsigned(grid), kThreads, 0, s>>>(k);
            PULSE_LAUNCHED("k1_ticket", s);
        }
    }
    k1_finalize<<<1, 32, 0, s>>>(p.segs, p.n_segs, p.numel, p.seg_start, p.idx32, p.cap, p.scan, copy_out);
    PULSE_LAUNCHED("k1_finalize", s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_encode)

}  // namespace dev
}  // namespace pulse
