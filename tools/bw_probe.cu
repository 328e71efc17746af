// Read-bandwidth ceiling probe for K1's access pattern (tool, not product):
// two 15 GB bf16 snapshots streamed once, 128-bit loads, XOR-OR compare, one
// counter per thread -- no compaction, no writes.  Reports TB/s of snapshot
// reads for several grid shapes / loads in flight, to set against k1_tma.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void probe(const uint4* __restrict__ a, const uint4* __restrict__ b, uint64_t n, unsigned long long* out) {
    uint32_t acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * U;
    for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x) * U + threadIdx.x; i < n; i += stride) {
        uint4 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t k = i + uint64_t(u) * blockDim.x;
            if (k < n) {
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w) : "l"(a + k));
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(y[u].x), "=r"(y[u].y), "=r"(y[u].z), "=r"(y[u].w) : "l"(b + k));
            } else {
                x[u] = y[u] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            acc += ((x[u].x ^ y[u].x) | (x[u].y ^ y[u].y) | (x[u].z ^ y[u].z) | (x[u].w ^ y[u].w)) != 0;
    }
    if (acc) atomicAdd(out, acc);
}

int main() {
    const uint64_t elems = 7615616512ull;  // the 7B state dict
    const uint64_t n = elems / 8;          // uint4 per snapshot
    uint4 *a, *b;
    unsigned long long* out;
    if (cudaMalloc(&a, n * 16) || cudaMalloc(&b, n * 16) || cudaMalloc(&out, 8)) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 0x11, n * 16);
    cudaMemset(b, 0x11, n * 16);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto kern, int blocks_per_sm, int threads) {
        float best = 1e9f;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(e0);
            kern<<<sms * blocks_per_sm, threads>>>(a, b, n, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        printf("%-10s %2d x %4d thr: %.3f ms  %.2f TB/s\n", name, blocks_per_sm, threads, best,
               2.0 * n * 16 / (best * 1e-3) / 1e12);
    };
    for (int bps : {1, 2, 4, 8}) {
        run("unroll2", probe<2>, bps, 512);
        run("unroll4", probe<4>, bps, 512);
        run("unroll8", probe<8>, bps, 256);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
