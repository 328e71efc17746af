// Device kernels behind the host-buffer API's index helpers and format
// conversions (include/pulse_cuda.h, "host-buffer API").  Sizes here are
// whatever a caller hands the reference's helper functions: grid-stride maps,
// and reduce-then-scan over up to 1024 block segments for the prefix sums of
// delta_decode_indices and downscale_coo.  upscale_coo runs on the general
// decoder's parallel parse (decode.cu launch_coo_unpack_par).  The hot path
// does not use these.
#include <mutex>

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

// ---- reduce-then-scan over contiguous block segments (helpers of any size) -----------------
// Block b of B owns elements [b * seg, (b + 1) * seg): pass 1 reduces its segment, one block
// scans the B partials (and their total), pass 2 re-scans each segment from its base.
constexpr int kHT = 256;             // threads per block
constexpr uint32_t kHMaxBlocks = 1024;

__device__ __forceinline__ uint64_t block_incl_u64(uint64_t v, uint64_t* s_w, uint64_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint64_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kHT / 32; ++w) {
        const uint64_t x = s_w[w];
        before += w < warp ? x : 0;
        all += x;
    }
    __syncthreads();
    total = all;
    return before + inc;
}

// exclusive scan of part[0..nb) in place (nb <= kHMaxBlocks), total into part[nb]
__global__ void __launch_bounds__(kHMaxBlocks) k_part_scan(uint64_t* __restrict__ part, uint32_t nb) {
    __shared__ uint64_t s_w[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t v = threadIdx.x < nb ? part[threadIdx.x] : 0;
    uint64_t inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint64_t before = 0, all = 0;
    for (int w = 0; w < int(blockDim.x / 32); ++w) {
        const uint64_t x = s_w[w];
        before += w < warp ? x : 0;
        all += x;
    }
    if (threadIdx.x < nb) part[threadIdx.x] = before + inc - v;
    if (threadIdx.x == 0) part[nb] = all;
}

__host__ __device__ inline uint32_t helper_blocks(uint64_t n) {
    const uint64_t b = (n + 8 * kHT - 1) / (8 * kHT);
    return uint32_t(b < 1 ? 1 : b > kHMaxBlocks ? kHMaxBlocks : b);
}

// delta_decode_indices (index_coding.hpp:31-50): running sum; first < 0 or a later gap
// <= 0 is a FormatError (check kZeroGap, first failure wins).  Pass 1: checks + block sums.
__global__ void __launch_bounds__(kHT) k_delta_sum(const int64_t* __restrict__ in, uint64_t n, uint64_t seg,
                                                    uint64_t* __restrict__ part, uint64_t* __restrict__ err) {
    __shared__ uint64_t s_w[kHT / 32];
    const uint64_t b0 = uint64_t(blockIdx.x) * seg, b1 = min(n, b0 + seg);
    uint64_t acc = 0;
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += kHT) {
        const int64_t v = in[i];
        if ((i == 0 && v < 0) || (i > 0 && v <= 0)) report(err, error_key(0, kStageRows, i, kZeroGap));
        acc += uint64_t(v);
    }
    uint64_t tot;
    block_incl_u64(acc, s_w, tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}
// Pass 2: each segment rescanned from its base, kHT elements per round.
__global__ void __launch_bounds__(kHT) k_delta_apply(const int64_t* __restrict__ in, uint64_t n, uint64_t seg,
                                                      const uint64_t* __restrict__ part, int64_t* __restrict__ out) {
    __shared__ uint64_t s_w[kHT / 32];
    const uint64_t b0 = uint64_t(blockIdx.x) * seg, b1 = min(n, b0 + seg);
    uint64_t base = part[blockIdx.x];
    for (uint64_t r = b0; r < b1; r += kHT) {
        const uint64_t i = r + threadIdx.x;
        const uint64_t v = i < b1 ? uint64_t(in[i]) : 0;
        uint64_t tot;
        const uint64_t inc = block_incl_u64(v, s_w, tot);
        if (i < b1) out[i] = int64_t(base + inc);
        base += tot;
    }
}

// downscale_coo (index_coding.hpp:108-128) over explicit (row, col) pairs.  Pass 1 checks
// every entry in the reference's terms (first failure wins) and sums its segment's row-stream
// bytes (1, or 5 with the 0xFF escape) and column-stream bytes (2, or 6 with 0xFFFF).
__device__ __forceinline__ void coo_sizes(const int64_t* rows, const int64_t* cols, uint64_t i, uint64_t& g,
                                          uint64_t& cv) {
    const int64_t r = rows[i], c = cols[i];
    g = uint64_t(i == 0 ? r : r - rows[i - 1]);
    cv = uint64_t((i == 0 || r != rows[i - 1]) ? c : c - cols[i - 1]);
}
__global__ void __launch_bounds__(kHT) k_coo_sum(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                                                  uint64_t n, uint64_t seg, uint64_t* __restrict__ part_r,
                                                  uint64_t* __restrict__ part_c, uint64_t* __restrict__ err) {
    __shared__ uint64_t s_w[kHT / 32];
    const uint64_t b0 = uint64_t(blockIdx.x) * seg, b1 = min(n, b0 + seg);
    uint64_t rb = 0, cb = 0;
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += kHT) {
        const int64_t r = rows[i], c = cols[i];
        if (r < 0 || c < 0) { report(err, error_key(0, kStageRows, i, kArgNegative)); continue; }
        if (i > 0 && (r < rows[i - 1] || (r == rows[i - 1] && c <= cols[i - 1]))) {
            report(err, error_key(0, kStageRows, i, kArgOrder));
            continue;
        }
        uint64_t g, cv;
        coo_sizes(rows, cols, i, g, cv);
        if (g > 0xFFFFFFFFull) report(err, error_key(0, kStageRows, i, kDimRow));
        if (cv > 0xFFFFFFFFull) report(err, error_key(0, kStageCols, i, kDimCol));
        rb += g >= 0xFF ? 5 : 1;
        cb += cv >= 0xFFFF ? 6 : 2;
    }
    uint64_t tr, tc;
    block_incl_u64(rb, s_w, tr);
    block_incl_u64(cb, s_w, tc);
    if (threadIdx.x == 0) {
        part_r[blockIdx.x] = tr;
        part_c[blockIdx.x] = tc;
    }
}
// Pass 2: row entries from the row-stream base of the segment, column entries after the
// whole row stream (part_r[nb] = its total).  Runs only if pass 1 found no failure.
__global__ void __launch_bounds__(kHT) k_coo_write(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                                                    uint64_t n, uint64_t seg, uint32_t nb,
                                                    const uint64_t* __restrict__ part_r,
                                                    const uint64_t* __restrict__ part_c, uint8_t* __restrict__ out,
                                                    uint64_t* __restrict__ nbytes, const uint64_t* __restrict__ err) {
    __shared__ uint64_t s_w[kHT / 32];
    if (*(volatile const uint64_t*)err != kNoError) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *nbytes = 0;
        return;
    }
    const uint64_t row_total = part_r[nb];
    if (blockIdx.x == 0 && threadIdx.x == 0) *nbytes = row_total + part_c[nb];
    const uint64_t b0 = uint64_t(blockIdx.x) * seg, b1 = min(n, b0 + seg);
    uint64_t rbase = part_r[blockIdx.x], cbase = row_total + part_c[blockIdx.x];
    for (uint64_t r0 = b0; r0 < b1; r0 += kHT) {
        const uint64_t i = r0 + threadIdx.x;
        uint64_t g = 0, cv = 0, rs = 0, cs = 0;
        if (i < b1) {
            coo_sizes(rows, cols, i, g, cv);
            rs = g >= 0xFF ? 5 : 1;
            cs = cv >= 0xFFFF ? 6 : 2;
        }
        uint64_t tr, tc;
        const uint64_t ir = block_incl_u64(rs, s_w, tr);
        const uint64_t ic = block_incl_u64(cs, s_w, tc);
        if (i < b1) {
            uint8_t* rp = out + rbase + ir - rs;
            if (rs == 5) { rp[0] = 0xFF; wr_u32(rp + 1, uint32_t(g)); }
            else rp[0] = uint8_t(g);
            uint8_t* cp = out + cbase + ic - cs;
            if (cs == 6) { wr_u16(cp, 0xFFFF); wr_u32(cp + 2, uint32_t(cv)); }
            else wr_u16(cp, uint32_t(cv));
        }
        rbase += tr;
        cbase += tc;
    }
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
namespace {
// per-device scratch for the block partials of the helpers (3 * (kHMaxBlocks + 1) words)
uint64_t* helper_scratch() {
    static std::mutex mu;
    static uint64_t* p[kMaxDevices] = {};
    std::lock_guard<std::mutex> lk(mu);
    uint64_t*& x = p[current_device()];
    if (!x && cudaMalloc(&x, 3 * (kHMaxBlocks + 1) * sizeof(uint64_t)) != cudaSuccess) x = nullptr;
    return x;
}
}  // namespace

void launch_delta_decode(const int64_t* in, uint64_t n, int64_t* out, uint64_t* err, cudaStream_t s) {
    if (!n) return;
    uint64_t* part = helper_scratch();
    const uint32_t nb = helper_blocks(n);
    const uint64_t seg = (n + nb - 1) / nb;
    k_delta_sum<<<nb, kHT, 0, s>>>(in, n, seg, part, err);
    PULSE_LAUNCHED("k_delta_sum", s);
    k_part_scan<<<1, kHMaxBlocks, 0, s>>>(part, nb);
    PULSE_LAUNCHED("k_part_scan", s);
    k_delta_apply<<<nb, kHT, 0, s>>>(in, n, seg, part, out);
    PULSE_LAUNCHED("k_delta_apply", s);
}
void launch_coo_pack(const int64_t* rows, const int64_t* cols, uint64_t n, uint8_t* out, uint64_t* nbytes,
                     uint64_t* err, cudaStream_t s) {
    uint64_t* part = helper_scratch();
    uint64_t* part_r = part;
    uint64_t* part_c = part + (kHMaxBlocks + 1);
    const uint32_t nb = helper_blocks(n);
    const uint64_t seg = (n + nb - 1) / nb;
    k_coo_sum<<<nb, kHT, 0, s>>>(rows, cols, n, seg, part_r, part_c, err);
    PULSE_LAUNCHED("k_coo_sum", s);
    k_part_scan<<<1, kHMaxBlocks, 0, s>>>(part_r, nb);
    PULSE_LAUNCHED("k_part_scan", s);
    k_part_scan<<<1, kHMaxBlocks, 0, s>>>(part_c, nb);
    PULSE_LAUNCHED("k_part_scan", s);
    k_coo_write<<<nb, kHT, 0, s>>>(rows, cols, n, seg, nb, part_r, part_c, out, nbytes, err);
    PULSE_LAUNCHED("k_coo_write", s);
}
PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_helpers)

}  // namespace dev
}  // namespace pulse
