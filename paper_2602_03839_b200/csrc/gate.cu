// Stream-ordered work that runs only if a device flag is set when the stream
// reaches it: the escape-aware decoder behind the fixed-layout apply, and K2's
// exact re-run behind the optimistic emit.  Eagerly, those kernels launch and
// return at once on their own flag checks.  Under stream capture (the
// benchmark's CUDA graphs) they become the body of a conditional graph node
// whose condition a one-thread kernel sets from the flag, so an idle path costs
// one tiny launch instead of a grid per kernel.
#include <cstdlib>

#include "device.cuh"
#include "internal.hpp"

namespace pulse {
namespace dev {

__global__ void k_set_cond(cudaGraphConditionalHandle h, const uint32_t* __restrict__ flag,
                           const uint64_t* __restrict__ key) {
    const bool on = flag ? *(volatile const uint32_t*)flag != 0 : *(volatile const uint64_t*)key != kNoError;
    cudaGraphSetConditional(h, on ? 1u : 0u);
}

namespace {
struct AuxStreams {
    cudaStream_t s[kMaxDevices] = {};
    cudaStream_t get() {
        cudaStream_t& x = s[current_device()];
        if (!x) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
        return x;
    }
};
AuxStreams g_aux;

bool gating_enabled() {
    static const bool off = [] {
        const char* e = getenv("PULSE_NO_GRAPH_GATE");
        return e && *e && *e != '0';
    }();
    return !off;
}
}  // namespace

static void gate(cudaStream_t s, const uint32_t* flag, const uint64_t* key,
                 const std::function<void(cudaStream_t)>& body) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    if (!gating_enabled() || cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd) != cudaSuccess ||
        st != cudaStreamCaptureStatusActive) {
        cudaGetLastError();
        body(s);
        return;
    }
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) {
        cudaGetLastError();
        body(s);
        return;
    }
    k_set_cond<<<1, 1, 0, s>>>(h, flag, key);
    PULSE_LAUNCHED("k_set_cond", s);
    cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd);  // now: after k_set_cond
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, g, deps, nd, &np) != cudaSuccess) {
        cudaGetLastError();
        body(s);  // the flag checks inside the kernels still gate them
        return;
    }
    cudaGraph_t inner = np.conditional.phGraph_out[0];
    cudaStream_t aux = g_aux.get();
    cudaStreamBeginCaptureToGraph(aux, inner, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    body(aux);
    cudaStreamEndCapture(aux, &inner);
    cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
}

void launch_gated(cudaStream_t s, const uint32_t* flag, const std::function<void(cudaStream_t)>& body) {
    gate(s, flag, nullptr, body);
}

void launch_gated_on_error(cudaStream_t s, const uint64_t* err_key, const std::function<void(cudaStream_t)>& body) {
    gate(s, nullptr, err_key, body);
}

}  // namespace dev
}  // namespace pulse
