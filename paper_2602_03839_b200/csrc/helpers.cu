// Device kernels behind the host-buffer API's index helpers and format
// conversions (include/pulse_cuda.h, "host-buffer API").  Sizes here are
// whatever a caller hands the reference's helper functions, so these favour
// simplicity: grid-stride maps, and single-CTA scans / single-thread stream
// parses for the inherently sequential helpers.  The hot path does not use
// them.
#include "device.cuh"
#include "internal.hpp"

namespace pulse {
namespace dev {

// K1 output -> int64 tensor-local indices (segment offset + u32), in place order.
__global__ void k_export_indices(const SegDesc* __restrict__ segs, const uint64_t* __restrict__ seg_start,
                                 uint32_t n_segs, const uint32_t* __restrict__ idx32, int64_t* __restrict__ out) {
    const uint64_t n = seg_start[n_segs];
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t sg = upper_index<uint64_t>(seg_start, 0, n_segs, i);
        out[i] = int64_t(segs[sg].elem_off + idx32[i]);
    }
}

// delta_encode_indices (index_coding.hpp:14-29): first as-is, then differences;
// negative -> check kArgNegative, not increasing -> kArgOrder (first failure wins).
__global__ void k_delta_encode(const int64_t* __restrict__ in, uint64_t n, int64_t* __restrict__ out,
                               uint64_t* __restrict__ err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const int64_t v = in[i];
        if (v < 0) { report(err, error_key(0, kStageRows, i, kArgNegative)); continue; }
        if (i > 0 && v <= in[i - 1]) { report(err, error_key(0, kStageRows, i, kArgOrder)); continue; }
        out[i] = i == 0 ? v : v - in[i - 1];
    }
}

// delta_decode_indices (index_coding.hpp:31-50): running sum; first < 0 or a
// later gap <= 0 is a FormatError (check kZeroGap reused, stage marks it).
__global__ void __launch_bounds__(1024) k_delta_decode(const int64_t* __restrict__ in, uint64_t n,
                                                       int64_t* __restrict__ out, uint64_t* __restrict__ err) {
    __shared__ int64_t s_w[32];
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t base = 0; base < n; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        int64_t v = 0;
        if (i < n) {
            v = in[i];
            if ((i == 0 && v < 0) || (i > 0 && v <= 0)) report(err, error_key(0, kStageRows, i, kZeroGap));
        }
        int64_t inc = v;
        for (int off = 1; off < 32; off <<= 1) {
            const int64_t o = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += o;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        int64_t before = 0, all = 0;
        for (int w = 0; w < int(blockDim.x / 32); ++w) {
            if (w < warp) before += s_w[w];
            all += s_w[w];
        }
        const int64_t c = s_carry;
        if (i < n) out[i] = c + before + inc;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = c + all;
        __syncthreads();
    }
}

// downscale_coo (index_coding.hpp:108-128) over explicit (row, col) pairs.
// Pass 0 validates and sizes every entry; pass 1 (after a host-side prefix of
// the sizes... kept on device: one CTA) writes the bytes.
__global__ void __launch_bounds__(1024) k_coo_pack(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                                                   uint64_t n, uint8_t* __restrict__ out, uint64_t* __restrict__ nbytes,
                                                   uint64_t* __restrict__ err) {
    __shared__ uint64_t s_w[32];
    __shared__ uint64_t s_row_carry, s_col_carry, s_row_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = int(blockDim.x / 32);
    // pass A: validation + total row-stream bytes
    uint64_t rbytes = 0;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        if (r < 0 || c < 0) { report(err, error_key(0, kStageRows, i, kArgNegative)); continue; }
        if (i > 0 && (r < rows[i - 1] || (r == rows[i - 1] && c <= cols[i - 1]))) {
            report(err, error_key(0, kStageRows, i, kArgOrder));
            continue;
        }
        const int64_t g = i == 0 ? r : r - rows[i - 1];
        if (g > 0xFFFFFFFFll) report(err, error_key(0, kStageRows, i, kDimRow));
        const bool nr = i == 0 || r != rows[i - 1];
        const int64_t cv = nr ? c : c - cols[i - 1];
        if (cv > 0xFFFFFFFFll) report(err, error_key(0, kStageCols, i, kDimCol));
        rbytes += g >= 0xFF ? 5 : 1;
    }
    for (int off = 16; off; off >>= 1) rbytes += __shfl_xor_sync(0xffffffffu, rbytes, off);
    if (lane == 0) s_w[warp] = rbytes;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < nw; ++w) t += s_w[w];
        s_row_total = t;
        s_row_carry = 0;
        s_col_carry = t;
    }
    __syncthreads();
    if (*err != kNoError) {
        if (threadIdx.x == 0) *nbytes = 0;
        return;
    }
    // pass B: ordered writes, chunk by chunk (block scans of entry sizes)
    for (uint64_t base = 0; base < n; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        uint64_t g = 0, cv = 0, rs = 0, cs = 0;
        if (i < n) {
            const int64_t r = rows[i], c = cols[i];
            g = uint64_t(i == 0 ? r : r - rows[i - 1]);
            const bool nr = i == 0 || r != rows[i - 1];
            cv = uint64_t(nr ? c : c - cols[i - 1]);
            rs = g >= 0xFF ? 5 : 1;
            cs = cv >= 0xFFFF ? 6 : 2;
        }
        uint64_t packed = rs | (cs << 32), inc = packed;
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t o = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += o;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        uint64_t before = 0, all = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < warp) before += s_w[w];
            all += s_w[w];
        }
        const uint64_t ex = before + inc - packed;
        if (i < n) {
            uint8_t* rp = out + s_row_carry + (ex & 0xFFFFFFFFull);
            if (rs == 5) { rp[0] = 0xFF; wr_u32(rp + 1, uint32_t(g)); }
            else rp[0] = uint8_t(g);
            uint8_t* cp = out + s_col_carry + (ex >> 32);
            if (cs == 6) { wr_u16(cp, 0xFFFF); wr_u32(cp + 2, uint32_t(cv)); }
            else wr_u16(cp, uint32_t(cv));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_row_carry += all & 0xFFFFFFFFull;
            s_col_carry += all >> 32;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *nbytes = s_col_carry;
    (void)s_row_total;
}

// upscale_coo (index_coding.hpp:130-158): one sequential parse, as the format
// carries no entry offsets (a helper; the apply path parses in parallel).
__global__ void k_coo_unpack(const uint8_t* __restrict__ p, uint64_t len, uint64_t count, int64_t* __restrict__ rows,
                             int64_t* __restrict__ cols, uint64_t* __restrict__ err) {
    if (threadIdx.x || blockIdx.x) return;
    uint64_t pos = 0;
    int64_t row = 0, col = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (pos + 1 > len) { report(err, error_key(0, kStageRows, i, kTrunc)); return; }
        int64_t e = p[pos++];
        if (e == 0xFF) {
            if (pos + 4 > len) { report(err, error_key(0, kStageRows, i, kTrunc)); return; }
            e = rd_u32(p + pos);
            pos += 4;
        }
        row = i == 0 ? e : row + e;
        rows[i] = row;
    }
    for (uint64_t i = 0; i < count; ++i) {
        const bool nr = i == 0 || rows[i] != rows[i - 1];
        if (pos + 2 > len) { report(err, error_key(0, kStageCols, i, kTrunc)); return; }
        int64_t e = rd_u16(p + pos);
        pos += 2;
        if (e == 0xFFFF) {
            if (pos + 4 > len) { report(err, error_key(0, kStageCols, i, kTrunc)); return; }
            e = rd_u32(p + pos);
            pos += 4;
        }
        if (nr) col = e;
        else {
            if (e <= 0) { report(err, error_key(0, kStageCols, i, kZeroColGap)); return; }
            col += e;
        }
        cols[i] = col;
    }
    if (pos != len) report(err, error_key(0, kStageTrailing, 0, kTrailing));
}

// Values at decoded indices: out[i] = W_t[idx[i]] for entry e's tensor t,
// entries [start[e], start[e+1]) (the resident apply's undo copy).
__global__ void k_gather_values(uint16_t* const* __restrict__ w, const pulse_patch_entry* __restrict__ ents,
                                const uint64_t* __restrict__ start, uint32_t n_e, const int64_t* __restrict__ idx,
                                uint16_t* __restrict__ out) {
    const uint64_t n = start[n_e];
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t e = upper_index<uint64_t>(start, 0, n_e, i);
        out[i] = w[ents[e].tensor][idx[i]];
    }
}

void launch_gather_values(const PlanDev& p, int slot, const pulse_patch_entry* ents, const uint64_t* start,
                          uint32_t n_e, const int64_t* idx, uint16_t* out, cudaStream_t s) {
    k_gather_values<<<sm_count() * 4, 256, 0, s>>>(p.slot[slot], ents, start, n_e, idx, out);
    PULSE_LAUNCHED("k_gather_values", s);
}

void launch_export_indices(const PlanDev& p, int64_t* out, cudaStream_t s) {
    k_export_indices<<<sm_count() * 4, 256, 0, s>>>(p.segs, p.seg_start, p.n_segs, p.idx32, out);
    PULSE_LAUNCHED("k_export_indices", s);
}
void launch_delta_encode(const int64_t* in, uint64_t n, int64_t* out, uint64_t* err, cudaStream_t s) {
    if (n) k_delta_encode<<<unsigned(std::min<uint64_t>((n + 255) / 256, 4096)), 256, 0, s>>>(in, n, out, err);
    PULSE_LAUNCHED("k_delta_encode", s);
}
void launch_delta_decode(const int64_t* in, uint64_t n, int64_t* out, uint64_t* err, cudaStream_t s) {
    if (n) k_delta_decode<<<1, 1024, 0, s>>>(in, n, out, err);
    PULSE_LAUNCHED("k_delta_decode", s);
}
void launch_coo_pack(const int64_t* rows, const int64_t* cols, uint64_t n, uint8_t* out, uint64_t* nbytes,
                     uint64_t* err, cudaStream_t s) {
    k_coo_pack<<<1, 1024, 0, s>>>(rows, cols, n, out, nbytes, err);
    PULSE_LAUNCHED("k_coo_pack", s);
}
void launch_coo_unpack(const uint8_t* p, uint64_t len, uint64_t count, int64_t* rows, int64_t* cols, uint64_t* err,
                       cudaStream_t s) {
    k_coo_unpack<<<1, 32, 0, s>>>(p, len, count, rows, cols, err);
    PULSE_LAUNCHED("k_coo_unpack", s);
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_helpers)

}  // namespace dev
}  // namespace pulse
