// Synthetic snapshot pairs on device (benchmark fixture, K5).
//
// Same knobs as the reference generator (synthetic.hpp:21-28, 30-107):
// sign-symmetric log-normal magnitudes (median, sigma) rounded to bf16, then
// exactly n_change = llround((1 - sparsity) * n) changed positions, placed in
// windows of `cluster_width` consecutive positions at half density, each
// changed by flipping the lowest mantissa bit.  The random streams are
// counter-based (splitmix64 of seed and position) instead of a sequential
// mt19937_64, so 7B-scale pairs generate in milliseconds; the bytes therefore
// differ from the reference generator's, and parity at these sizes is checked
// by handing the *same* device bytes to the reference encoder.
#include <cmath>

#include <cuda_bf16.h>

#include "device.cuh"
#include "internal.hpp"
#include "plan.hpp"

namespace pulse {
namespace dev {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_synth_base(uint16_t* __restrict__ out, uint64_t n, uint64_t seed, float log_median, float sigma) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 8;
    for (uint64_t e0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e0 < n; e0 += stride) {
        uint16_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint64_t h1 = mix64(seed ^ mix64(e0 + k));
            const uint64_t h2 = mix64(h1 ^ 0xD1B54A32D192ED03ull);
            const float u1 = (float((h1 >> 40) + 1)) * (1.0f / 16777216.0f);  // (0, 1]
            const float u2 = float(h2 >> 40) * (1.0f / 16777216.0f);
            const float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
            float x = expf(log_median + sigma * z);
            if (h2 & 1) x = -x;
            v[k] = __bfloat16_as_ushort(__float2bfloat16_rn(x));
        }
        if (e0 + 8 <= n) {
            uint4 w = make_uint4(v[0] | uint32_t(v[1]) << 16, v[2] | uint32_t(v[3]) << 16,
                                 v[4] | uint32_t(v[5]) << 16, v[6] | uint32_t(v[7]) << 16);
            *reinterpret_cast<uint4*>(out + e0) = w;
        } else {
            for (int k = 0; k < 8 && e0 + k < n; ++k) out[e0 + k] = v[k];
        }
    }
}

// One thread per window: half-density marks (all marks when every element
// changes, synthetic.hpp:85), counted as they become new.
__global__ void k_synth_mark(uint32_t* __restrict__ bitmap, uint64_t n, uint64_t seed, uint64_t width,
                             uint64_t k0, uint64_t n_windows, bool all, unsigned long long* __restrict__ counter) {
    const uint64_t k = k0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t added = 0;
    if (k < k0 + n_windows) {
        const uint64_t start = mix64(seed ^ (k * 0x2545F4914F6CDD1Dull)) % n;
        uint64_t word = start >> 5;
        uint32_t mask = 0;
        for (uint64_t j = 0; j < width; ++j) {
            const uint64_t pos = start + j;
            if (pos >= n) break;
            const bool take = all || ((mix64(seed ^ mix64(k) ^ (j * 0x9E3779B97F4A7C15ull)) >> 63) & 1);
            if (!take) continue;
            if ((pos >> 5) != word) {
                if (mask) added += __popc(mask & ~atomicOr(bitmap + word, mask));
                word = pos >> 5;
                mask = 0;
            }
            mask |= 1u << (pos & 31);
        }
        if (mask) added += __popc(mask & ~atomicOr(bitmap + word, mask));
    }
    // warp-aggregate the count
    for (int off = 16; off; off >>= 1) added += __shfl_down_sync(0xffffffffu, added, off);
    if ((threadIdx.x & 31) == 0 && added) atomicAdd(counter, (unsigned long long)added);
}

// Final windows one position at a time, stopping at exactly `target` marks
// (the reference stops mid-window, synthetic.hpp:81-96).
__global__ void k_synth_mark_exact(uint32_t* __restrict__ bitmap, uint64_t n, uint64_t seed, uint64_t width,
                                   uint64_t k0, bool all, unsigned long long* __restrict__ counter, uint64_t target) {
    if (threadIdx.x || blockIdx.x) return;
    uint64_t marked = *counter;
    for (uint64_t k = k0; marked < target; ++k) {
        const uint64_t start = mix64(seed ^ (k * 0x2545F4914F6CDD1Dull)) % n;
        for (uint64_t j = 0; j < width && marked < target; ++j) {
            const uint64_t pos = start + j;
            if (pos >= n) break;
            const bool take = all || ((mix64(seed ^ mix64(k) ^ (j * 0x9E3779B97F4A7C15ull)) >> 63) & 1);
            if (!take) continue;
            const uint32_t bit = 1u << (pos & 31);
            if (!(bitmap[pos >> 5] & bit)) {
                bitmap[pos >> 5] |= bit;
                ++marked;
            }
        }
    }
    *counter = marked;
}

__global__ void k_synth_flip(const uint16_t* __restrict__ base, uint16_t* __restrict__ out,
                             const uint32_t* __restrict__ bitmap, uint64_t n) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * 8;
    for (uint64_t e0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; e0 < n; e0 += stride) {
        const uint32_t bits = (bitmap[e0 >> 5] >> (e0 & 31)) & 0xFF;  // e0 % 8 == 0
        if (e0 + 8 <= n) {
            uint4 w = *reinterpret_cast<const uint4*>(base + e0);
            w.x ^= (bits & 1) | ((bits & 2) << 15);
            w.y ^= ((bits >> 2) & 1) | (((bits >> 3) & 1) << 16);
            w.z ^= ((bits >> 4) & 1) | (((bits >> 5) & 1) << 16);
            w.w ^= ((bits >> 6) & 1) | (((bits >> 7) & 1) << 16);
            *reinterpret_cast<uint4*>(out + e0) = w;
        } else {
            for (uint64_t k = 0; e0 + k < n; ++k) out[e0 + k] = base[e0 + k] ^ ((bits >> k) & 1);
        }
    }
}

PULSE_DEFINE_WATCHDOG_SETTER(set_watchdog_synth)

}  // namespace dev
}  // namespace pulse

using namespace pulse::dev;

extern "C" {

pulse_status pulse_synth_base(uint16_t* dev_out, uint64_t n, uint64_t seed, double median, double sigma,
                              void* stream) {
    if (!dev_out || n == 0 || !(median > 0)) return pulse::fail(PULSE_E_ARGUMENT, "synth_base: bad argument");
    const unsigned grid = unsigned(std::min<uint64_t>((n + 2047) / 2048, uint64_t(sm_count()) * 16));
    k_synth_base<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(dev_out, n, seed, float(std::log(median)),
                                                                      float(sigma));
    PULSE_LAUNCHED("k_synth_base", static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : pulse::cuda_fail(e, "synth_base");
}

pulse_status pulse_synth_mutate(pulse_context* ctx, const uint16_t* dev_base, uint16_t* dev_out, uint64_t n,
                                double sparsity, uint64_t cluster_width, uint64_t seed, uint64_t* changed_out,
                                void* stream) {
    if (!ctx || !dev_base || !dev_out || n == 0 || !(sparsity >= 0.0 && sparsity <= 1.0) || cluster_width < 1)
        return pulse::fail(PULSE_E_ARGUMENT, "synth_mutate: bad argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t target = uint64_t(std::llround((1.0 - sparsity) * double(n)));
    const uint64_t words = ((n + 31) / 32 + 2) & ~1ull;  // even: the counter after it is 8-byte aligned
    uint32_t* bitmap = nullptr;
    unsigned long long* counter = nullptr;
    cudaError_t e = cudaMallocAsync(&bitmap, words * 4 + 64, s);
    if (e != cudaSuccess) return pulse::cuda_fail(e, "synth bitmap");
    counter = reinterpret_cast<unsigned long long*>(bitmap + words);
    cudaMemsetAsync(bitmap, 0, words * 4 + 64, s);
    const uint64_t mseed = pulse::dev::mix64(seed ^ 0x9E3779B97F4A7C15ull);
    const bool all = target == n;
    uint64_t k = 0, count = 0;
    while (target > count && target - count > cluster_width) {
        const uint64_t B = std::max<uint64_t>(1, (target - count) / cluster_width);
        const unsigned grid = unsigned((B + 255) / 256);
        k_synth_mark<<<grid, 256, 0, s>>>(bitmap, n, mseed, cluster_width, k, B, all, counter);
        PULSE_LAUNCHED("k_synth_mark", s);
        k += B;
        unsigned long long c = 0;
        cudaMemcpyAsync(&c, counter, sizeof(c), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        count = c;
    }
    if (count < target) k_synth_mark_exact<<<1, 1, 0, s>>>(bitmap, n, mseed, cluster_width, k, all, counter, target);
    PULSE_LAUNCHED("k_synth_mark_exact", s);
    const unsigned grid = unsigned(std::min<uint64_t>((n + 2047) / 2048, uint64_t(sm_count()) * 16));
    k_synth_flip<<<grid, 256, 0, s>>>(dev_base, dev_out, bitmap, n);
    PULSE_LAUNCHED("k_synth_flip", s);
    unsigned long long c = 0;
    cudaMemcpyAsync(&c, counter, sizeof(c), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(bitmap, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return pulse::cuda_fail(e, "synth_mutate");
    if (changed_out) *changed_out = c;
    return PULSE_OK;
}

}  // extern "C"
