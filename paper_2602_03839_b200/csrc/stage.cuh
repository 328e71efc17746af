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

__device__ __forceinline__ uint32_t shr_pair(uint32_t lo, uint32_t hi, uint32_t sh) {
    return __funnelshift_r(lo, hi, sh);
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
        const uint32_t W[8] = {v[r].x, v[r].y, v[r].z, v[r].w, nx.x, nx.y, nx.z, nx.w};
        uint4 o;
        switch (sw) {
            case 0: o = make_uint4(shr_pair(W[0], W[1], sh), shr_pair(W[1], W[2], sh), shr_pair(W[2], W[3], sh), shr_pair(W[3], W[4], sh)); break;
            case 1: o = make_uint4(shr_pair(W[1], W[2], sh), shr_pair(W[2], W[3], sh), shr_pair(W[3], W[4], sh), shr_pair(W[4], W[5], sh)); break;
            case 2: o = make_uint4(shr_pair(W[2], W[3], sh), shr_pair(W[3], W[4], sh), shr_pair(W[4], W[5], sh), shr_pair(W[5], W[6], sh)); break;
            default: o = make_uint4(shr_pair(W[3], W[4], sh), shr_pair(W[4], W[5], sh), shr_pair(W[5], W[6], sh), shr_pair(W[6], W[7], sh)); break;
        }
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

// Reads lane-consecutive vector i (of V) of a swizzled buffer.
template <int V>
__device__ __forceinline__ uint4 lane_vec(const uint4* buf, int i) {
    const int lane = threadIdx.x & 31;
    return buf[swz<V>(uint32_t(lane * V + i))];
}

// 32-bit word `w` of a swizzled buffer.
template <int V>
__device__ __forceinline__ uint32_t smem_word(const uint4* buf, uint32_t w) {
    return reinterpret_cast<const uint32_t*>(buf)[swz<V>(w >> 2) * 4 + (w & 3)];
}

// Copies `len` bytes, packed from byte 0 of swizzled shared buffer `src`, to
// global `dst` (any alignment): whole 16-byte blocks with one vector store
// (funnel-shifted out of shared memory), the partial head/tail blocks bytewise.
// Bytes of `dst` outside [dst, dst+len) are never written.
template <int V>
__device__ __forceinline__ void unstage(uint8_t* dst, const uint4* src, uint32_t len) {
    if (len == 0) return;
    const int lane = threadIdx.x & 31;
    const uintptr_t da = reinterpret_cast<uintptr_t>(dst);
    const uint32_t s = uint32_t(da & 15);
    uint8_t* base = dst - s;
    const uint32_t nblk = (s + len + 15) >> 4;
    const uint32_t sh = ((16 - s) & 3) * 8;  // byte shift of every block's source start
    for (uint32_t k = lane; k < nblk; k += 32) {
        const int32_t o = int32_t(16 * k) - int32_t(s);  // source offset of the block's first byte
        if (o >= 0 && uint32_t(o) + 16 <= len) {
            const uint32_t w0 = uint32_t(o) >> 2;
            const uint32_t x0 = smem_word<V>(src, w0), x1 = smem_word<V>(src, w0 + 1);
            const uint32_t x2 = smem_word<V>(src, w0 + 2), x3 = smem_word<V>(src, w0 + 3);
            uint4 out;
            if (sh == 0) {
                out = make_uint4(x0, x1, x2, x3);
            } else {
                const uint32_t x4 = smem_word<V>(src, w0 + 4);
                out = make_uint4(__funnelshift_r(x0, x1, sh), __funnelshift_r(x1, x2, sh), __funnelshift_r(x2, x3, sh),
                                 __funnelshift_r(x3, x4, sh));
            }
            *reinterpret_cast<uint4*>(base + 16 * k) = out;
        } else {
#pragma unroll 1
            for (int b = 0; b < 16; ++b) {
                const int32_t so = o + b;
                if (so >= 0 && uint32_t(so) < len) {
                    const uint32_t w = smem_word<V>(src, uint32_t(so) >> 2);
                    base[16 * k + b] = uint8_t(w >> (8 * (so & 3)));
                }
            }
        }
    }
}

}  // namespace dev
}  // namespace pulse
