// Contexts, plans and the device-resident C ABI (include/pulse_cuda.h).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "device.cuh"
#include "internal.hpp"
#include "plan.hpp"

using namespace pulse::dev;

namespace pulse {

thread_local std::string g_last_error;

pulse_status fail(pulse_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

pulse_status cuda_fail(cudaError_t e, const char* what) {
    return fail(PULSE_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace pulse

using pulse::cuda_fail;
using pulse::fail;

// ---------------------------------------------------------------------------------------------
// Device arena helpers
// ---------------------------------------------------------------------------------------------
template <class T>
static cudaError_t dalloc(std::vector<void*>& owned, T** p, size_t n) {
    void* raw = nullptr;
    const cudaError_t e = cudaMalloc(&raw, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) owned.push_back(raw);
    *p = static_cast<T*>(raw);
    return e;
}

pulse_context::~pulse_context() {
    for (auto* p : owned) cudaFree(p);
    if (pinned) cudaFreeHost(pinned);
}

pulse_plan::~pulse_plan() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (auto* p : owned) cudaFree(p);
    if (host_pinned) cudaFreeHost(host_pinned);
    cudaSetDevice(prev);
}

// Host-mapped watchdog slot shared by all devices of the process (see device.cuh).
static unsigned long long* g_wd_host = nullptr;
static unsigned long long* g_wd_dev = nullptr;
static std::mutex g_wd_mu;

void pulse_install_watchdog(int device);
static void install_watchdog(int device) { pulse_install_watchdog(device); }
void pulse_install_watchdog(int device) {
    std::lock_guard<std::mutex> lk(g_wd_mu);
    if (!g_wd_host) {
        void* h = nullptr;
        if (cudaHostAlloc(&h, 8 * sizeof(unsigned long long), cudaHostAllocMapped | cudaHostAllocPortable) !=
            cudaSuccess)
            return;
        std::memset(h, 0, 8 * sizeof(unsigned long long));
        g_wd_host = static_cast<unsigned long long*>(h);
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&g_wd_dev), h, 0);
    }
    static bool done[64] = {};
    if (device >= 0 && device < 64 && !done[device]) {
        set_watchdog_encode(g_wd_dev);
        set_watchdog_decode(g_wd_dev);
        set_watchdog_synth(g_wd_dev);
        set_watchdog_index(g_wd_dev);
        set_watchdog_apply(g_wd_dev);
        set_watchdog_helpers(g_wd_dev);
        set_watchdog_reduce(g_wd_dev);
        done[device] = true;
    }
}

extern "C" {

int pulse_watchdog(uint64_t* out7) {
    if (!g_wd_host) return 0;
    volatile unsigned long long* w = g_wd_host;
    const int fired = w[0] != 0;
    if (out7)
        for (int i = 0; i < 7; ++i) out7[i] = w[i];
    if (fired)
        for (int i = 0; i < 8; ++i) w[i] = 0;
    return fired;
}

const char* pulse_last_error(void) { return pulse::g_last_error.c_str(); }
const char* pulse_version(void) { return "pulse-b200 0.1 (sm_100a)"; }

pulse_status pulse_context_create(int device, pulse_context** out) {
    if (!out) return fail(PULSE_E_ARGUMENT, "null output pointer");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    auto* c = new pulse_context();
    c->device = device;
    install_watchdog(device);
    *out = c;
    return PULSE_OK;
}

void pulse_context_destroy(pulse_context* ctx) { delete ctx; }

pulse_status pulse_plan_create(pulse_context* ctx, const pulse_tensor_geom* tensors, uint32_t n_tensors,
                               uint64_t max_changes, pulse_plan** out) {
    if (!ctx || !out || (n_tensors && !tensors)) return fail(PULSE_E_ARGUMENT, "null argument");
    if (n_tensors >= (1u << 20)) return fail(PULSE_E_ARGUMENT, "too many tensors (max 2^20)");
    cudaSetDevice(ctx->device);
    auto plan = new pulse_plan();
    plan->ctx = ctx;
    plan->device = ctx->device;
    plan->geom.assign(tensors, tensors + n_tensors);

    // segments (<= 2^31 elements) and K1 tiles
    std::vector<SegDesc> segs;
    std::vector<uint32_t> seg_first(n_tensors + 1);
    uint64_t tiles = 0, tickets = 0;
    for (uint32_t t = 0; t < n_tensors; ++t) {
        const uint64_t n = tensors[t].numel;
        if (n == 0 || tensors[t].cols == 0 || n % tensors[t].cols != 0) {
            delete plan;
            return fail(PULSE_E_ARGUMENT, "tensor " + std::to_string(t) + " has invalid geometry");
        }
        seg_first[t] = uint32_t(segs.size());
        for (uint64_t off = 0; off < n; off += kSegElems) {
            SegDesc d;
            d.elem_off = off;
            d.tile_start = tiles;
            d.ticket_start = tickets;
            d.tensor = t;
            d.numel = uint32_t(std::min<uint64_t>(kSegElems, n - off));
            tiles += (d.numel + kTileElems - 1) / kTileElems;
            tickets += (d.numel + kTicketElems - 1) / kTicketElems;
            segs.push_back(d);
        }
    }
    seg_first[n_tensors] = uint32_t(segs.size());
    PlanDev& p = plan->dev;
    std::memset(&p, 0, sizeof(p));
    p.n_tensors = n_tensors;
    p.n_segs = uint32_t(segs.size());
    p.n_tiles = tiles;
    p.tma_tiles = tickets;
    p.cap = std::max<uint64_t>(max_changes, 1);
    uint64_t elems = 0;
    for (uint32_t t = 0; t < n_tensors; ++t) elems += tensors[t].numel;
    // K1 staging shape from the change capacity (profiles/r2e_k1_sparse_shapes.txt: the sparse
    // shape's 448 records per ticket overflow from ~2.2% clustered changes on)
    p.k1_dense = p.cap * 1000 >= elems * 56 ? 3u : p.cap * 1000 >= elems * 45 ? 2u : p.cap * 1000 >= elems * 22 ? 1u
               : p.cap * 1000 < elems * 15 ? 4u : 0u;
    const uint64_t T = n_tensors, S = segs.size(), cap = p.cap;
    const uint64_t n_chunks = cap / kChunkEntries + 2;
    p.dec_bytes_cap = 10 * cap + kParseBytes * (T + 1);
    p.d_status_len = std::max<uint64_t>(n_chunks, p.dec_bytes_cap / kParseTile + T + 2);

    auto& o = plan->owned;
    cudaError_t e = cudaSuccess;
    SegDesc* segs_d; uint32_t* first_d; uint64_t *numel_d, *cols_d; uint32_t* tile_seg_d; uint32_t* ticket_seg_d;
    SegDesc* id_segs_d; uint32_t* id_first_d;
#define A(ptr, n) if (e == cudaSuccess) e = dalloc(o, &(ptr), (n))
    A(segs_d, S); A(first_d, T + 1); A(numel_d, T); A(cols_d, T); A(tile_seg_d, tiles); A(ticket_seg_d, tickets);
    for (int s = 0; s < PULSE_MAX_SLOTS; ++s) { uint16_t** sp = nullptr; A(sp, T); p.slot[s] = sp; }
    // idx32 / val16: +8 entries so 16-byte async copies of a partial last chunk stay in bounds
    A(p.idx32, cap + 8); A(p.val16, cap + 8); A(p.seg_start, S + 1); A(p.k1_status, tiles + 1);
    A(p.counters, 8); A(p.scan, 1); A(p.k1_defer, tickets + 1);
    ColDiv* coldiv_d = nullptr; A(coldiv_d, T);
    A(p.range_cnt, cap / kK2RangeEntries + 2); A(p.range_pre, cap / kK2RangeEntries + 2);
    A(p.t_resc, T); A(p.t_cesc, T); A(p.tlay, T); A(p.err, 1); A(p.result, 1);
    A(id_segs_d, T); A(id_first_d, T + 1); A(p.id_start, T + 1);
    A(p.elay, T); A(p.d_es, T + 1); A(p.d_ck, T + 1); A(p.d_cu, T + 1);
    A(p.rowgap, cap); A(p.colent, cap); A(p.flat, cap);
    A(p.d_status, 4 * p.d_status_len); A(p.d_totals, 16); A(p.d_flags, 4);
    if (getenv("PULSE_TRACE")) A(p.trace, tickets);
#undef A
    if (e != cudaSuccess) {
        delete plan;
        return cuda_fail(e, "plan allocation");
    }
    p.segs = segs_d;
    p.coldiv = coldiv_d;
    p.tile_seg = tile_seg_d;
    p.tma_tile_seg = ticket_seg_d;
    p.seg_first = first_d;
    p.numel = numel_d;
    p.cols = cols_d;
    p.id_segs = id_segs_d;
    p.id_first = id_first_d;

    std::vector<uint64_t> numel(T), cols(T);
    std::vector<ColDiv> coldiv(T);
    for (uint32_t t = 0; t < n_tensors; ++t) coldiv[t] = make_coldiv(tensors[t].cols);
    cudaMemcpy(coldiv_d, coldiv.data(), T * sizeof(ColDiv), cudaMemcpyHostToDevice);
    std::vector<SegDesc> id_segs(T);
    std::vector<uint32_t> id_first(T + 1);
    for (uint32_t t = 0; t < n_tensors; ++t) {
        numel[t] = tensors[t].numel;
        cols[t] = tensors[t].cols;
        id_segs[t] = SegDesc{0, 0, 0, t, 0};
        id_first[t] = t;
    }
    id_first[T] = uint32_t(T);
    std::vector<uint32_t> tile_seg(tiles);
    for (uint32_t si = 0; si < S; ++si) {
        const uint64_t t0 = segs[si].tile_start;
        const uint64_t t1 = si + 1 < S ? segs[si + 1].tile_start : tiles;
        for (uint64_t t = t0; t < t1; ++t) tile_seg[t] = si;
    }
    cudaMemcpy(tile_seg_d, tile_seg.data(), tiles * sizeof(uint32_t), cudaMemcpyHostToDevice);
    std::vector<uint32_t> ticket_seg(tickets);
    for (uint32_t si = 0; si < S; ++si) {
        const uint64_t t0 = segs[si].ticket_start;
        const uint64_t t1 = si + 1 < S ? segs[si + 1].ticket_start : tickets;
        for (uint64_t t = t0; t < t1; ++t) ticket_seg[t] = si;
    }
    cudaMemcpy(ticket_seg_d, ticket_seg.data(), tickets * sizeof(uint32_t), cudaMemcpyHostToDevice);
    cudaMemcpy(segs_d, segs.data(), S * sizeof(SegDesc), cudaMemcpyHostToDevice);
    cudaMemcpy(first_d, seg_first.data(), (T + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice);
    cudaMemcpy(numel_d, numel.data(), T * sizeof(uint64_t), cudaMemcpyHostToDevice);
    cudaMemcpy(cols_d, cols.data(), T * sizeof(uint64_t), cudaMemcpyHostToDevice);
    cudaMemcpy(id_segs_d, id_segs.data(), T * sizeof(SegDesc), cudaMemcpyHostToDevice);
    e = cudaMemcpy(id_first_d, id_first.data(), (T + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        delete plan;
        return cuda_fail(e, "plan upload");
    }
    *out = plan;
    return PULSE_OK;
}

void pulse_plan_destroy(pulse_plan* plan) { delete plan; }

pulse_status pulse_plan_bind(pulse_plan* plan, uint32_t slot, const void* const* dev_ptrs) {
    if (!plan || slot >= PULSE_MAX_SLOTS || (plan->dev.n_tensors && !dev_ptrs))
        return fail(PULSE_E_ARGUMENT, "bad plan/slot/pointers");
    for (uint32_t t = 0; t < plan->dev.n_tensors; ++t)
        if (reinterpret_cast<uintptr_t>(dev_ptrs[t]) % 16 != 0)
            return fail(PULSE_E_ARGUMENT, "tensor " + std::to_string(t) + " is not 16-byte aligned");
    cudaSetDevice(plan->device);
    cudaError_t e = cudaMemcpy(const_cast<uint16_t**>(plan->dev.slot[slot]), dev_ptrs,
                               plan->dev.n_tensors * sizeof(void*), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "bind");
    plan->bound[slot] = true;
    return PULSE_OK;
}

pulse_status pulse_encode_scan(pulse_plan* plan, uint32_t curr_slot, uint32_t prev_slot,
                               pulse_scan_summary* dev_summary_out, void* stream) {
    if (!plan || curr_slot >= PULSE_MAX_SLOTS || prev_slot >= PULSE_MAX_SLOTS ||
        !plan->bound[curr_slot] || !plan->bound[prev_slot])
        return fail(PULSE_E_ARGUMENT, "encode_scan: unbound slot");
    cudaSetDevice(plan->device);
    launch_encode_scan(plan->dev, curr_slot, prev_slot, dev_summary_out, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "encode_scan launch");
}

pulse_scan_summary* pulse_plan_scan_summary(pulse_plan* plan) { return plan ? plan->dev.scan : nullptr; }

// Debug: device pointer + length of the K1 ticket trace (NULL unless PULSE_TRACE is set).
uint32_t* pulse_plan_trace(pulse_plan* plan, uint64_t* n) {
    if (n) *n = plan ? plan->dev.tma_tiles : 0;
    return plan ? plan->dev.trace : nullptr;
}

pulse_status pulse_encode_emit(pulse_plan* plan, uint32_t repr, const pulse_scan_summary* gathered,
                               uint32_t n_ranks, uint32_t rank, uint8_t* dev_body, uint64_t body_capacity,
                               pulse_patch_entry* dev_entries, pulse_result* dev_result, void* stream) {
    if (!plan || repr > 2 || !dev_entries || !dev_result || (gathered && rank >= n_ranks))
        return fail(PULSE_E_ARGUMENT, "encode_emit: bad argument");
    cudaSetDevice(plan->device);
    launch_encode_emit(plan->dev, repr, gathered, n_ranks, rank, dev_body, dev_body ? body_capacity : 0,
                       dev_entries, dev_result, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "encode_emit launch");
}

pulse_status pulse_apply(pulse_plan* plan, uint32_t weights_slot, uint32_t repr, const uint8_t* dev_body,
                         const pulse_patch_entry* dev_entries, uint32_t n_entries,
                         const pulse_flat_carry* dev_carry, pulse_result* dev_result, void* stream) {
    if (!plan || repr > 2 || weights_slot >= PULSE_MAX_SLOTS || !plan->bound[weights_slot] || !dev_result ||
        n_entries > plan->dev.n_tensors)
        return fail(PULSE_E_ARGUMENT, "apply: bad argument");
    cudaSetDevice(plan->device);
    launch_decode(plan->dev, repr, dev_body, dev_entries, n_entries, dev_carry, int(weights_slot), nullptr,
                  dev_result, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "apply launch");
}

pulse_status pulse_apply_patch(pulse_plan* plan, uint32_t weights_slot, uint32_t repr, const uint8_t* dev_body,
                               const pulse_patch_entry* dev_entries, const pulse_result* dev_patch_result,
                               const pulse_flat_carry* dev_carry, pulse_result* dev_result, void* stream) {
    if (!plan || repr > 2 || weights_slot >= PULSE_MAX_SLOTS || !plan->bound[weights_slot] || !dev_result ||
        !dev_patch_result)
        return fail(PULSE_E_ARGUMENT, "apply_patch: bad argument");
    cudaSetDevice(plan->device);
    launch_decode(plan->dev, repr, dev_body, dev_entries, plan->dev.n_tensors, dev_carry, int(weights_slot), nullptr,
                  dev_result, static_cast<cudaStream_t>(stream), dev_patch_result);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "apply launch");
}

pulse_status pulse_count_changed(pulse_plan* plan, uint32_t slot_a, uint32_t slot_b, uint64_t* dev_count,
                                 void* stream) {
    if (!plan || !dev_count || slot_a >= PULSE_MAX_SLOTS || slot_b >= PULSE_MAX_SLOTS || !plan->bound[slot_a] ||
        !plan->bound[slot_b])
        return fail(PULSE_E_ARGUMENT, "count_changed: bad argument");
    cudaSetDevice(plan->device);
    launch_count_changed(plan->dev, slot_a, slot_b, dev_count, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "count_changed launch");
}

pulse_status pulse_count_above(pulse_plan* plan, uint32_t slot, uint32_t magnitude_bits, uint64_t* dev_count,
                               void* stream) {
    if (!plan || !dev_count || slot >= PULSE_MAX_SLOTS || !plan->bound[slot])
        return fail(PULSE_E_ARGUMENT, "count_above: bad argument");
    cudaSetDevice(plan->device);
    launch_count_above(plan->dev, slot, magnitude_bits, dev_count, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "count_above launch");
}

pulse_status pulse_flat_carry_from_summaries(const pulse_scan_summary* dev_gathered, uint32_t rank,
                                             pulse_flat_carry* dev_out, void* stream) {
    if (!dev_gathered || !dev_out) return fail(PULSE_E_ARGUMENT, "flat_carry: null argument");
    launch_flat_carry(dev_gathered, rank, dev_out, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "flat_carry launch");
}

pulse_status pulse_store_to_peers(const void* dev_src, void* const* dsts, uint32_t n_dst, uint32_t nbytes,
                                  int device, void* stream) {
    if (!dev_src || (n_dst && !dsts) || nbytes == 0 || nbytes > 256 || n_dst > 64)
        return fail(PULSE_E_ARGUMENT, "store_to_peers: bad argument");
    if (n_dst == 0) return PULSE_OK;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int dev = device;
    cudaError_t e = cudaSetDevice(dev);
    if (e != cudaSuccess) return cuda_fail(e, "store_to_peers: device");
    PeerPtrs pp{};
    for (uint32_t i = 0; i < n_dst; ++i) pp.p[i] = dsts[i];
    // peer access from this device to every device it can reach, once per device (the
    // destinations are usually IPC mappings another runtime opened on their own device)
    static std::mutex mu;
    static std::set<int> enabled;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (enabled.insert(dev).second) {
            int n = 0;
            cudaGetDeviceCount(&n);
            for (int q = 0; q < n; ++q) {
                int can = 0;
                if (q == dev || cudaDeviceCanAccessPeer(&can, dev, q) != cudaSuccess || !can) continue;
                const cudaError_t pe = cudaDeviceEnablePeerAccess(q, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
                    enabled.erase(dev);
                    return cuda_fail(pe, "store_to_peers: peer access");
                }
            }
            cudaGetLastError();
        }
    }
    launch_store_to_peers(dev_src, pp, n_dst, nbytes, s);
    e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "store_to_peers launch");
}

pulse_status pulse_peer_allgather(const void* dev_src, void* const* tables, uint32_t world, uint32_t rank,
                                  uint32_t nbytes, uint64_t* dev_epoch, void* dev_out, int device, void* stream) {
    if (!dev_src || !tables || !dev_epoch || !dev_out || world == 0 || world > 64 || rank >= world ||
        nbytes == 0 || nbytes > 48)
        return fail(PULSE_E_ARGUMENT, "peer_allgather: bad argument");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "peer_allgather: device");
    PeerPtrs pp{};
    for (uint32_t i = 0; i < world; ++i) pp.p[i] = tables[i];
    launch_peer_allgather(dev_src, pp, tables[rank], world, rank, nbytes,
                          reinterpret_cast<unsigned long long*>(dev_epoch), dev_out, static_cast<cudaStream_t>(stream));
    e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "peer_allgather launch");
}

pulse_status pulse_ipc_open(const void* ipc_handle, int device, void** dev_ptr) {
    if (!ipc_handle || !dev_ptr) return fail(PULSE_E_ARGUMENT, "ipc_open: null argument");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "ipc_open: device");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof(h));
    e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "ipc_open");
}

pulse_status pulse_ipc_close(void* dev_ptr, int device) {
    if (!dev_ptr) return PULSE_OK;
    cudaSetDevice(device);
    const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "ipc_close");
}

pulse_status pulse_decode_indices(pulse_plan* plan, uint32_t repr, const uint8_t* dev_body,
                                  const pulse_patch_entry* dev_entries, uint32_t n_entries,
                                  const pulse_flat_carry* dev_carry, int64_t* dev_indices,
                                  pulse_result* dev_result, void* stream) {
    if (!plan || repr > 2 || !dev_result || n_entries > plan->dev.n_tensors)
        return fail(PULSE_E_ARGUMENT, "decode_indices: bad argument");
    cudaSetDevice(plan->device);
    launch_decode(plan->dev, repr, dev_body, dev_entries, n_entries, dev_carry, -1, dev_indices, dev_result,
                  static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PULSE_OK : cuda_fail(e, "decode launch");
}

}  // extern "C"
