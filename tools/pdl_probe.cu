// Graph edge cost on B200: a chain of K dependent small kernels (each reads the previous one's
// output) replayed as a CUDA graph, with plain stream order vs programmatic dependent launch
// (PDL: cudaLaunchAttributeProgrammaticStreamSerialization + griddepcontrol.wait / .launch_dependents).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_probe tools/pdl_probe.cu && ./pdl_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(unsigned* buf, int i, int trigger) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (trigger) asm volatile("griddepcontrol.launch_dependents;");
    const unsigned v = buf[(i + 1023) % 1024];
    if (threadIdx.x == 0) buf[i % 1024 + blockIdx.x * 0] = v + 1;
}

static float run(int K, int grid, int block, bool pdl, int trigger) {
    unsigned* buf;
    cudaMalloc(&buf, 4096 * 4);
    cudaMemset(buf, 0, 4096 * 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < K; ++i) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, step, buf, i, trigger);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return -1; }
    for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    const int R = 200;
    for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(buf);
    cudaStreamDestroy(s);
    return ms * 1000.f / R / K;  // us per kernel
}

int main() {
    const int K = 16;
    int grids[] = {1, 148, 444, 1184};
    for (int gi = 0; gi < 4; ++gi) {
        for (int block : {256, 1024}) {
            if (grids[gi] * block > 1184 * 256 * 4) continue;
            printf("grid %5d x %4d: plain %.2f us/kernel, pdl %.2f, pdl+trigger %.2f\n", grids[gi], block,
                   run(K, grids[gi], block, false, 0), run(K, grids[gi], block, true, 0),
                   run(K, grids[gi], block, true, 1));
        }
    }
    return 0;
}
