// Warp-cooperative staging between global memory at arbitrary byte alignment
// and per-warp shared-memory buffers (apply_fast.cu, index_code.cu).
//
// Shared buffers are arrays of 16-byte slots.  A buffer that lanes read (or
// write) as V consecutive slots per lane is XOR-swizzled (swz<V>) so both those
// per-lane accesses and the warp-consecutive staging accesses are free of bank
// conflicts.
#pragma once
#include "device.cuh"

namespace pulse {
namespace dev {

// XOR swizzle of 16-byte vector slots for buffers read as V consecutive vectors
// per lane: within every group of 8 lanes the slots hit 8 distinct bank quads,
// and 8 consecutive slots (a staging store) stay a permutation of one 128 B row.
template <int V>
__device__ __forceinline__ uint32_t swz(uint32_t q) {
    return V == 1 ? q : (q ^ ((q >> 3) & (V - 1)));
}


// 16-byte shared-memory load kept as ONE vector access (a compiler-split load
// would turn the conflict-free swizzled pattern into 4-way bank conflicts).
__device__ __forceinline__ uint4 lds128(const uint4* p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(smem_u32(p))
                 : "memory");
    return r;
}

// 16 bytes starting at byte (4*sw + sh/8) of the 32-byte pair (lo, hi).
__device__ __forceinline__ uint4 funnel16(const uint4& lo, const uint4& hi, uint32_t sw, uint32_t sh) {
    const uint32_t W[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    switch (sw) {
        case 0: return make_uint4(__funnelshift_r(W[0], W[1], sh), __funnelshift_r(W[1], W[2], sh), __funnelshift_r(W[2], W[3], sh), __funnelshift_r(W[3], W[4], sh));
        case 1: return make_uint4(__funnelshift_r(W[1], W[2], sh), __funnelshift_r(W[2], W[3], sh), __funnelshift_r(W[3], W[4], sh), __funnelshift_r(W[4], W[5], sh));
        case 2: return make_uint4(__funnelshift_r(W[2], W[3], sh), __funnelshift_r(W[3], W[4], sh), __funnelshift_r(W[4], W[5], sh), __funnelshift_r(W[5], W[6], sh));
        default: return make_uint4(__funnelshift_r(W[3], W[4], sh), __funnelshift_r(W[4], W[5], sh), __funnelshift_r(W[5], W[6], sh), __funnelshift_r(W[6], W[7], sh));
    }
}

__device__ __forceinline__ uint4 shfl_up4(const uint4& v, int d) {
    return make_uint4(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d),
                      __shfl_up_sync(0xffffffffu, v.z, d), __shfl_up_sync(0xffffffffu, v.w, d));
}
__device__ __forceinline__ uint4 shfl4(const uint4& v, int src) {
    return make_uint4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                      __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

// Copies bytes [g, g+len) (len <= 512 * R) into shared vectors dst[swz(q)],
// packed from byte 0.  All loads are issued before any store.  Reads at most
// the 16-byte-aligned blocks that contain payload bytes (never past a page).
template <int R, int V>
__device__ __forceinline__ void stage_piece(uint4* dst, const uint8_t* g, uint32_t len, uint32_t q_base) {
    const int lane = threadIdx.x & 31;
    const uintptr_t ga = reinterpret_cast<uintptr_t>(g);
    const uint32_t s = uint32_t(ga & 15);
    const uint4* src = reinterpret_cast<const uint4*>(ga - s);
    const uint32_t nv_in = (s + len + 15) >> 4;
    const uint32_t nv_out = (len + 15) >> 4;
    uint4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t q = lane + 32 * r;
        v[r] = q < nv_in ? ld_stream(src + q) : make_uint4(0, 0, 0, 0);
    }
    if (s == 0) {  // aligned: straight copy
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t q = lane + 32 * r;
            if (q < nv_out) dst[swz<V>(q_base + q)] = v[r];
        }
        return;
    }
    uint4 extra = make_uint4(0, 0, 0, 0);
    if (lane == 0 && 32u * R < nv_in) extra = ld_stream(src + 32 * R);
    const uint32_t sw = s >> 2, sh = (s & 3) * 8;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        uint4 nx;
        nx.x = __shfl_down_sync(0xffffffffu, v[r].x, 1);
        nx.y = __shfl_down_sync(0xffffffffu, v[r].y, 1);
        nx.z = __shfl_down_sync(0xffffffffu, v[r].z, 1);
        nx.w = __shfl_down_sync(0xffffffffu, v[r].w, 1);
        const uint4 n0 = r + 1 < R ? v[r + 1 < R ? r + 1 : r] : extra;
        const uint32_t w0 = __shfl_sync(0xffffffffu, n0.x, 0), w1 = __shfl_sync(0xffffffffu, n0.y, 0);
        const uint32_t w2 = __shfl_sync(0xffffffffu, n0.z, 0), w3 = __shfl_sync(0xffffffffu, n0.w, 0);
        if (lane == 31) nx = make_uint4(w0, w1, w2, w3);
        const uint4 o = funnel16(v[r], nx, sw, sh);
        const uint32_t q = lane + 32 * r;
        if (q < nv_out) dst[swz<V>(q_base + q)] = o;
    }
}

// Stages up to `len` bytes (len <= cap) in pieces of 2 KiB (16 B aligned pieces
// keep the source alignment, so the swizzled slot index just continues).
template <int V>
__device__ __forceinline__ void stage(uint4* dst, const uint8_t* g, uint32_t len) {
    for (uint32_t off = 0; off < len; off += 2048)
        stage_piece<4, V>(dst, g + off, min(2048u, len - off), off >> 4);
}

// ---- asynchronous global -> shared copies (cp.async, no register staging) ------------------
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
// The same with the shared-memory address already in the .shared window (no per-copy cvta).
__device__ __forceinline__ void cp_async16_s(uint32_t sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Queues the 16-byte slots covering [g, g+len) (g 16-byte aligned) into the
// swizzled buffer dst; reads up to 15 bytes past len (callers pad the source).
template <int V>
__device__ __forceinline__ void stage_async(uint4* dst, const uint8_t* g, uint32_t len) {
    const int lane = threadIdx.x & 31;
    const uint32_t nslots = (len + 15) >> 4;
    const uint32_t sdst = smem_u32(dst);
    for (uint32_t q = lane; q < nslots; q += 32) cp_async16_s(sdst + 16 * swz<V>(q), g + 16 * q);
}

// 32-bit word `w` of a swizzled buffer (single scalar accesses only).
template <int V>
__device__ __forceinline__ uint32_t smem_word(const uint4* buf, uint32_t w) {
    return reinterpret_cast<const uint32_t*>(buf)[swz<V>(w >> 2) * 4 + (w & 3)];
}

// Reads lane-consecutive vector i (of V) of a swizzled buffer.
template <int V>
__device__ __forceinline__ uint4 lane_vec(const uint4* buf, int i) {
    const int lane = threadIdx.x & 31;
    return lds128(buf + swz<V>(uint32_t(lane * V + i)));
}


// Copies `len` bytes, packed from byte 0 of swizzled shared buffer `src`, to
// global `dst` (any alignment).  Lane k of a round writes aligned 16-byte block
// k of the destination: with a byte offset s = dst & 15 that block holds the
// tail of source slot k-1 and the head of slot k, so every lane loads ONE slot
// (conflict-free) and takes its neighbour's by shuffle.  Whole blocks are one
// vector store; the partial head/tail blocks are written bytewise, so bytes of
// `dst` outside [dst, dst+len) are never touched.
template <int V>
__device__ __forceinline__ void unstage(uint8_t* dst, const uint4* src, uint32_t len) {
    if (len == 0) return;
    const int lane = threadIdx.x & 31;
    const uint32_t s = uint32_t(reinterpret_cast<uintptr_t>(dst) & 15);
    uint8_t* base = dst - s;
    const uint32_t nblk = (s + len + 15) >> 4, nslots = (len + 15) >> 4;
    const uint32_t sb = (16 - s) & 15, sw = sb >> 2, sh = (sb & 3) * 8;
    const uint32_t tail_k = nblk - 1;
    const bool head_partial = s != 0 || len < 16;
    const bool tail_partial = ((s + len) & 15) != 0;
    uint4 head = make_uint4(0, 0, 0, 0), tail = head;  // partial blocks, held by their lanes
    for (uint32_t k0 = 0; k0 < nblk; k0 += 32) {
        const uint32_t k = k0 + lane;
        if (k >= nblk) continue;
        const uint4 cur = k < nslots ? lds128(src + swz<V>(k)) : make_uint4(0, 0, 0, 0);
        // the slot before: a second conflict-free load (consecutive lanes, consecutive slots)
        // instead of eight shuffles and a carry across rounds
        const uint4 prv = (s != 0 && k > 0) ? lds128(src + swz<V>(k - 1)) : make_uint4(0, 0, 0, 0);
        const uint4 out = s == 0 ? cur : funnel16(prv, cur, sw, sh);
        const bool partial = (k == 0 && head_partial) || (k == tail_k && tail_partial);
        if (!partial) *reinterpret_cast<uint4*>(base + 16 * k) = out;
        if (k == 0) head = out;
        if (k == tail_k) tail = out;
    }
    // the (at most two) partial blocks: lanes 0-15 write the head block's bytes,
    // lanes 16-31 the tail block's, each lane one byte
    const int hl = 0, tl = int(tail_k & 31);
    const uint4 h = shfl4(head, hl), t = shfl4(tail, tl);
    const bool is_tail = lane >= 16;
    const uint32_t bi = uint32_t(lane & 15);
    const uint32_t k = is_tail ? tail_k : 0u;
    if ((is_tail ? tail_partial : head_partial) && !(is_tail && tail_k == 0 && head_partial)) {
        const uint4 v = is_tail ? t : h;
        const int32_t so = int32_t(16 * k + bi) - int32_t(s);  // source offset of this byte
        if (so >= 0 && uint32_t(so) < len) {
            const uint32_t w = bi < 4 ? v.x : bi < 8 ? v.y : bi < 12 ? v.z : v.w;
            base[16 * k + bi] = uint8_t(w >> (8 * (bi & 3)));
        }
    }
}

}  // namespace dev
}  // namespace pulse
