// Host-buffer C ABI (include/pulse_cuda.h, "host-buffer API"): the reference's
// functions over host memory, one entry point each.  Every per-element step
// of the path (diff/compaction, index coding, payload parsing, validation,
// scatter, and the index helpers) runs in the CUDA kernels; the host keeps what
// the reference keeps on the host and the GPU cannot reproduce bit-exactly:
// validation of names/shapes, the PULP JSON header (nlohmann, as the
// reference), the codec stage (the same libzstd / liblz4 / zlib calls as
// compression.hpp:79-147) and SHA-256 (OpenSSL EVP, as sha256.hpp:51-87;
// a serial Merkle-Damgard chain).
//
// Inputs are staged to the device through a pinned double buffer; the memcpy
// into pinned memory is split across a small thread pool.
#include <openssl/evp.h>
#include <sys/mman.h>
#include <zlib.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <future>
#include <memory>
#include <mutex>
#include <nlohmann/json.hpp>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "errors.hpp"
#include "internal.hpp"
#include "plan.hpp"

extern "C" {
size_t ZSTD_compress(void* dst, size_t dst_capacity, const void* src, size_t src_size, int level);
size_t ZSTD_decompress(void* dst, size_t dst_capacity, const void* src, size_t src_size);
size_t ZSTD_compressBound(size_t src_size);
unsigned long long ZSTD_decompressBound(const void* src, size_t src_size);
unsigned ZSTD_isError(size_t code);
int LZ4_compress_default(const char* src, char* dst, int src_size, int dst_capacity);
int LZ4_decompress_safe(const char* src, char* dst, int compressed_size, int dst_capacity);
int LZ4_compressBound(int input_size);
}

using pulse::fail;
using namespace pulse::dev;

// ---------------------------------------------------------------------------------------------
// library-owned objects
// ---------------------------------------------------------------------------------------------
// Allocator that leaves elements uninitialised: the big host buffers below are
// fully overwritten (by copies or DMA), so zero-filling them is wasted time.
// Buffers of 64 MB and more (a 7B patch's indices: 608 MB) are 2 MB-aligned and
// advised as transparent huge pages: first-touch page faults were most of
// read_patch_bytes' host time (150 K 4 KB faults for the indices alone).
constexpr size_t kHugeBytes = size_t(64) << 20, kHugeAlign = size_t(2) << 20;
// Freed large blocks are kept (up to 4 GiB, 16 blocks) and reused by the next allocation of a
// similar size: a patch per call (7B: 608 MB of indices, 152 MB of values, 381 MB of bytes)
// then neither unmaps nor first-touches its pages again -- those costs made the host legs of
// the end-to-end step vary 0.07-0.55 s between boxes.
struct BigBlocks {
    static constexpr size_t kMaxBytes = size_t(4) << 30, kMaxBlocks = 16;
    std::mutex mu;
    std::vector<std::pair<void*, size_t>> free_blocks;
    size_t held = 0;
    void* take(size_t len) {
        std::lock_guard<std::mutex> lk(mu);
        size_t best = free_blocks.size();
        for (size_t i = 0; i < free_blocks.size(); ++i) {
            const size_t l = free_blocks[i].second;
            if (l >= len && l <= 2 * len && (best == free_blocks.size() || l < free_blocks[best].second)) best = i;
        }
        if (best == free_blocks.size()) return nullptr;
        void* p = free_blocks[best].first;
        held -= free_blocks[best].second;
        free_blocks.erase(free_blocks.begin() + long(best));
        return p;
    }
    bool keep(void* p, size_t len) {
        std::lock_guard<std::mutex> lk(mu);
        if (held + len > kMaxBytes || free_blocks.size() >= kMaxBlocks) return false;
        free_blocks.emplace_back(p, len);
        held += len;
        return true;
    }
};
inline BigBlocks& big_blocks() {
    static BigBlocks* b = new BigBlocks();  // never destroyed: vectors may be freed during exit
    return *b;
}
template <class T>
struct NoInit : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInit<U>;
    };
    NoInit() = default;
    template <class U>
    NoInit(const NoInit<U>&) noexcept {}
    T* allocate(size_t n) {
        const size_t bytes = n * sizeof(T);
        if (bytes < kHugeBytes) return std::allocator<T>::allocate(n);
        const size_t len = (bytes + kHugeAlign - 1) / kHugeAlign * kHugeAlign;
        if (void* q = big_blocks().take(len)) return static_cast<T*>(q);
        void* p = std::aligned_alloc(kHugeAlign, len);
        if (!p) throw std::bad_alloc();
        madvise(p, len, MADV_HUGEPAGE);  // advisory: ignored where THP is off
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t n) {
        const size_t bytes = n * sizeof(T);
        if (bytes < kHugeBytes) {
            std::allocator<T>::deallocate(p, n);
            return;
        }
        const size_t len = (bytes + kHugeAlign - 1) / kHugeAlign * kHugeAlign;
        if (!big_blocks().keep(p, len)) std::free(p);
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        if constexpr (sizeof...(A) == 0) ::new (static_cast<void*>(p)) U;
        else ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using RawVec = std::vector<T, NoInit<T>>;

struct pulse_bytes {
    RawVec<uint8_t> v;
};

struct PatchTensor {
    std::string name;
    std::vector<int64_t> shape;
    RawVec<int64_t> indices;  // no zero fill on resize: always overwritten (hundreds of MB at 7B)
    RawVec<uint16_t> values;
};

// The identity-coded payloads of a patch, as K2 lays them out: one body with
// each tensor's [index payload][value payload] (write_patch_bytes' blobs).
struct Coded {
    RawVec<uint8_t> body;
    std::vector<std::pair<uint64_t, uint64_t>> payload;  // per tensor; len 0 if no indices
    std::vector<uint64_t> val_off;                        // per tensor (valid when indices exist)
};

struct pulse_patch {
    int64_t base_step = 0, target_step = 0, anchor_step = 0;
    uint32_t representation = PULSE_COO_DOWNSCALED, codec = PULSE_ZSTD1;
    uint8_t target_hash[32] = {};
    std::vector<PatchTensor> tensors;
    // encode() also runs K2 while the snapshots are resident; write_patch_bytes reuses
    // that body for the same representation.  Any change to the tensors drops it.
    Coded coded;
    bool coded_valid = false;
    uint32_t coded_repr = 0;
    // read_patch_bytes decodes the indices on the device; they stay there (tensor order, flat)
    // so decode() need not upload them again.  Any change to the tensors drops them.
    int64_t* dev_idx = nullptr;
    int dev_idx_device = -1;
    uint64_t dev_idx_n = 0;
    bool dev_idx_valid = false;
    ~pulse_patch() {
        if (!dev_idx) return;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(dev_idx_device);
        // stream-ordered free into the device's pool (no device-wide sync per patch); the
        // call that filled dev_idx synchronized its stream before returning
        cudaFreeAsync(dev_idx, 0);
        cudaSetDevice(prev);
    }
};

struct pulse_sha256_ctx {
    EVP_MD_CTX* ctx;
};

namespace {

// PULSE_TIMING=1: per-stage wall times of the host API calls on stderr.
struct StageTimer {
    const char* what;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    static bool on() {
        static const bool v = [] {
            const char* e = getenv("PULSE_TIMING");
            return e && *e && *e != '0';
        }();
        return v;
    }
    void lap(const char* stage) {
        if (!on()) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[pulse timing] %s %s %.1f ms\n", what, stage,
                     std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

// A failure with the reference's exception class and message.
struct Failure {
    pulse_status st;
    std::string msg;
};

[[noreturn]] void raise(pulse_status st, std::string msg) { throw Failure{st, std::move(msg)}; }

template <class F>
pulse_status guarded(F&& f) {
    try {
        f();
        return PULSE_OK;
    } catch (const Failure& e) {
        return fail(e.st, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(PULSE_E_ERROR, "out of memory");
    } catch (const std::exception& e) {
        return fail(PULSE_E_ERROR, e.what());
    }
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(PULSE_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- thread pool -----------------------------------------------------------------------------
class Pool {
public:
    explicit Pool(unsigned n) {
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    // f(i) for i in [0, n), parallel.  Returns only after every helper has left
    // the loop, so the shared counters may live on the caller's stack.
    void parallel_for(size_t n, const std::function<void(size_t)>& f) {
        if (n <= 1 || workers_.empty()) {
            for (size_t i = 0; i < n; ++i) f(i);
            return;
        }
        std::atomic<size_t> next{0};
        std::mutex m;
        std::condition_variable c;
        size_t helpers = std::min<size_t>(workers_.size(), n - 1);
        size_t running = helpers;
        auto loop = [&] {
            size_t i;
            while ((i = next.fetch_add(1)) < n) f(i);
        };
        for (size_t h = 0; h < helpers; ++h)
            submit([&] {
                loop();
                std::lock_guard<std::mutex> lk(m);
                if (--running == 0) c.notify_all();
            });
        loop();
        std::unique_lock<std::mutex> lk(m);
        c.wait(lk, [&] { return running == 0; });
    }

private:
    void submit(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push(std::move(f));
        }
        cv_.notify_one();
    }
    void loop() {
        while (true) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                f = std::move(q_.front());
                q_.pop();
            }
            f();
        }
    }
    std::vector<std::thread> workers_;
    std::queue<std::function<void()>> q_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p(std::max(2u, std::min(16u, std::thread::hardware_concurrency())) - 1);
    return p;
}

void par_memcpy(void* dst, const void* src, size_t n) {
    constexpr size_t kPiece = 4 << 20;
    const size_t pieces = (n + kPiece - 1) / kPiece;
    if (pieces <= 1) {
        if (n) std::memcpy(dst, src, n);
        return;
    }
    pool().parallel_for(pieces, [&](size_t i) {
        const size_t off = i * kPiece, len = std::min(kPiece, n - off);
        std::memcpy(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, len);
    });
}

// Every host<->device copy the host API issues goes through here, so the
// end-to-end benchmark can report the bytes it really moved.
std::atomic<uint64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

cudaError_t counted_copy(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t s) {
    if (kind == cudaMemcpyHostToDevice) g_h2d_bytes += n;
    else if (kind == cudaMemcpyDeviceToHost) g_d2h_bytes += n;
    return cudaMemcpyAsync(dst, src, n, kind, s);
}

// Page-locked (cudaHostAlloc'd or registered) host memory can be the DMA
// source/target directly; pageable memory goes through the staging buffers.
bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// ---- device buffers + staging ----------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            const size_t want = std::max<size_t>(bytes + bytes / 8, 1 << 20);
            cuda_check(cudaMalloc(&p, want), "device arena");
            cap = want;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) { return static_cast<T*>(get(std::max<size_t>(count, 1) * sizeof(T))); }
};

// Pinned double buffer between pageable host memory and the device.
class Stager {
public:
    static constexpr size_t kChunk = 64u << 20;
    Stager() {
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaHostAlloc(&buf_[i], kChunk, cudaHostAllocDefault), "pinned staging");
            cuda_check(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming), "event");
        }
    }
    void h2d(void* dst, const void* src, size_t n, cudaStream_t s) {
        if (n < (1 << 20) || is_pinned(src)) {
            cuda_check(counted_copy(dst, src, n, cudaMemcpyHostToDevice, s), "H2D");
            return;
        }
        for (size_t off = 0, k = 0; off < n; off += kChunk, ++k) {
            const int b = int(k & 1);
            const size_t len = std::min(kChunk, n - off);
            cuda_check(cudaEventSynchronize(ev_[b]), "staging wait");
            par_memcpy(buf_[b], static_cast<const uint8_t*>(src) + off, len);
            cuda_check(counted_copy(static_cast<uint8_t*>(dst) + off, buf_[b], len, cudaMemcpyHostToDevice, s), "H2D");
            cuda_check(cudaEventRecord(ev_[b], s), "event");
        }
    }
    void d2h(void* dst, const void* src, size_t n, cudaStream_t s) {
        if (n < (1 << 20) || is_pinned(dst)) {
            cuda_check(counted_copy(dst, src, n, cudaMemcpyDeviceToHost, s), "D2H");
            cuda_check(cudaStreamSynchronize(s), "D2H sync");
            return;
        }
        // two chunks in flight: copy k+1 runs while k is unpacked
        const size_t chunks = (n + kChunk - 1) / kChunk;
        auto issue = [&](size_t k) {
            const int b = int(k & 1);
            const size_t off = k * kChunk, len = std::min(kChunk, n - off);
            cuda_check(counted_copy(buf_[b], static_cast<const uint8_t*>(src) + off, len, cudaMemcpyDeviceToHost, s), "D2H");
            cuda_check(cudaEventRecord(ev_[b], s), "event");
        };
        issue(0);
        for (size_t k = 0; k < chunks; ++k) {
            if (k + 1 < chunks) issue(k + 1);
            const int b = int(k & 1);
            cuda_check(cudaEventSynchronize(ev_[b]), "D2H wait");
            const size_t off = k * kChunk, len = std::min(kChunk, n - off);
            par_memcpy(static_cast<uint8_t*>(dst) + off, buf_[b], len);
        }
    }

    // One pipelined D2H of a contiguous device range into several host buffers (the
    // per-tensor index vectors of a patch): `segs` lists (destination, bytes) in device order.
    // One copy instead of one synchronised copy per tensor (339 at 7B).
    void d2h_scatter(const std::vector<std::pair<void*, size_t>>& segs, const void* src, cudaStream_t s) {
        size_t n = 0;
        for (const auto& g : segs) n += g.second;
        if (n == 0) return;
        const size_t chunks = (n + kChunk - 1) / kChunk;
        auto issue = [&](size_t k) {
            const int b = int(k & 1);
            const size_t off = k * kChunk, len = std::min(kChunk, n - off);
            cuda_check(counted_copy(buf_[b], static_cast<const uint8_t*>(src) + off, len, cudaMemcpyDeviceToHost, s), "D2H");
            cuda_check(cudaEventRecord(ev_[b], s), "event");
        };
        size_t seg = 0, seg_off = 0;  // segment holding byte `off` of the range, its start
        struct Piece {
            uint8_t* dst;
            const uint8_t* src;
            size_t len;
        };
        std::vector<Piece> pieces;
        issue(0);
        for (size_t k = 0; k < chunks; ++k) {
            if (k + 1 < chunks) issue(k + 1);
            const int b = int(k & 1);
            cuda_check(cudaEventSynchronize(ev_[b]), "D2H wait");
            const size_t off = k * kChunk, len = std::min(kChunk, n - off);
            pieces.clear();
            for (size_t at = off; at < off + len;) {
                while (seg_off + segs[seg].second <= at) seg_off += segs[seg++].second;
                const size_t in_seg = at - seg_off;
                const size_t take = std::min({off + len - at, segs[seg].second - in_seg, size_t(4) << 20});
                pieces.push_back({static_cast<uint8_t*>(segs[seg].first) + in_seg,
                                  static_cast<const uint8_t*>(buf_[b]) + (at - off), take});
                at += take;
            }
            pool().parallel_for(pieces.size(), [&](size_t i) { std::memcpy(pieces[i].dst, pieces[i].src, pieces[i].len); });
        }
    }

private:
    void* buf_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2];
};

// One per device: context, stream, cached plan and arenas.
struct Engine {
    int device = 0;
    pulse_context* ctx = nullptr;
    cudaStream_t stream = nullptr;
    Stager stager;
    // plans by geometry, least recently used last: encode (the whole checkpoint), read
    // (the patch's tensors) and decode alternate in one end-to-end step, and rebuilding a
    // plan (device scratch for its change capacity) on every switch cost 0.1-0.4 s
    struct CachedPlan {
        pulse_plan* plan;
        std::vector<pulse_tensor_geom> geom;
        uint64_t cap;
    };
    static constexpr size_t kMaxPlans = 3;
    std::vector<CachedPlan> plans;
    DevBuf arena_a, arena_b, idx64, vals, body, entries, result, misc, out64;
    std::mutex mu;
    // decode pipeline: upload and download streams + per-group events (lazy)
    cudaStream_t s_up = nullptr, s_dn = nullptr;
    std::vector<cudaEvent_t> ev_up, ev_cmp;

    void pipeline_streams(size_t groups) {
        if (!s_up) {
            cuda_check(cudaStreamCreateWithFlags(&s_up, cudaStreamNonBlocking), "stream");
            cuda_check(cudaStreamCreateWithFlags(&s_dn, cudaStreamNonBlocking), "stream");
        }
        while (ev_up.size() < groups) {
            cudaEvent_t a, b;
            cuda_check(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "event");
            ev_up.push_back(a);
            ev_cmp.push_back(b);
        }
    }

    explicit Engine(int dev) : device(dev) {
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        if (pulse_context_create(dev, &ctx) != PULSE_OK) raise(PULSE_E_CUDA, "context");
        cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    }

    pulse_plan* get_plan(const std::vector<pulse_tensor_geom>& geom, uint64_t cap) {
        auto same_geom = [&](const CachedPlan& c) {
            return geom.size() == c.geom.size() &&
                   std::equal(geom.begin(), geom.end(), c.geom.begin(),
                              [](auto& a, auto& b) { return a.numel == b.numel && a.cols == b.cols; });
        };
        for (size_t i = 0; i < plans.size(); ++i) {
            if (!same_geom(plans[i])) continue;
            CachedPlan c = plans[i];
            plans.erase(plans.begin() + long(i));
            if (cap <= c.cap) {
                plans.insert(plans.begin(), c);
                return c.plan;
            }
            cudaStreamSynchronize(stream);  // too small: replaced below
            pulse_plan_destroy(c.plan);
            break;
        }
        if (plans.size() >= kMaxPlans) {
            cudaStreamSynchronize(stream);
            pulse_plan_destroy(plans.back().plan);
            plans.pop_back();
        }
        const uint64_t c = std::max<uint64_t>(cap, 1024);
        pulse_plan* np = nullptr;
        if (pulse_plan_create(ctx, geom.data(), uint32_t(geom.size()), c, &np) != PULSE_OK)
            raise(PULSE_E_CUDA, std::string("plan: ") + pulse_last_error());
        plans.insert(plans.begin(), CachedPlan{np, geom, c});
        return np;
    }

    void sync() { cuda_check(cudaStreamSynchronize(stream), "stream sync"); }
};

Engine& engine() {
    static std::mutex mu;
    static std::unordered_map<int, std::unique_ptr<Engine>> engines;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto& e = engines[dev];
    if (!e) e = std::make_unique<Engine>(dev);
    cudaSetDevice(dev);
    return *e;
}

// ---- checkpoint helpers (checkpoint.hpp:54-80) -----------------------------------------------
uint64_t shape_numel(const int64_t* shape, uint32_t rank) {
    uint64_t n = 1;
    for (uint32_t i = 0; i < rank; ++i) n *= uint64_t(shape[i]);
    return n;
}

void validate_checkpoint(const pulse_checkpoint* c) {
    std::vector<std::string_view> seen;
    seen.reserve(c->n_tensors);
    for (uint32_t i = 0; i < c->n_tensors; ++i) {
        const pulse_tensor& t = c->tensors[i];
        const std::string name = t.name ? t.name : "";
        if (name.empty()) raise(PULSE_E_ARGUMENT, "tensor with empty name");
        if (std::find(seen.begin(), seen.end(), std::string_view(t.name)) != seen.end())
            raise(PULSE_E_ARGUMENT, "duplicate tensor name: " + name);
        seen.emplace_back(t.name);
        if (t.rank == 0) raise(PULSE_E_ARGUMENT, "tensor " + name + " has empty shape");
        uint64_t n = 1;
        for (uint32_t k = 0; k < t.rank; ++k) {
            if (t.shape[k] <= 0) raise(PULSE_E_ARGUMENT, "tensor " + name + " has non-positive extent");
            n *= uint64_t(t.shape[k]);
        }
        if (n != t.numel) raise(PULSE_E_ARGUMENT, "tensor " + name + " shape/data length mismatch");
    }
}

std::vector<uint32_t> sorted_order(const pulse_checkpoint* c) {
    std::vector<uint32_t> o(c->n_tensors);
    for (uint32_t i = 0; i < c->n_tensors; ++i) o[i] = i;
    std::stable_sort(o.begin(), o.end(),
                     [&](uint32_t a, uint32_t b) { return std::strcmp(c->tensors[a].name, c->tensors[b].name) < 0; });
    return o;
}

// SHA-256 over raw LE bf16 bytes, tensors in name order (sha256.hpp:93-116).
void hash_tensors(const std::vector<std::pair<const uint16_t*, uint64_t>>& parts, uint8_t out[32]) {
    EVP_MD_CTX* ctx = EVP_MD_CTX_new();
    if (!ctx || EVP_DigestInit_ex(ctx, EVP_sha256(), nullptr) != 1) raise(PULSE_E_ERROR, "failed to initialize SHA-256 context");
    for (auto& [p, n] : parts)
        if (n && EVP_DigestUpdate(ctx, p, n * 2) != 1) raise(PULSE_E_ERROR, "SHA-256 update failed");
    unsigned int len = 0;
    if (EVP_DigestFinal_ex(ctx, out, &len) != 1 || len != 32) raise(PULSE_E_ERROR, "SHA-256 finalize failed");
    EVP_MD_CTX_free(ctx);
}

void hash_checkpoint(const pulse_checkpoint* c, uint8_t out[32]) {
    std::vector<std::pair<const uint16_t*, uint64_t>> parts;
    for (uint32_t i : sorted_order(c)) parts.emplace_back(c->tensors[i].data, c->tensors[i].numel);
    hash_tensors(parts, out);
}

std::string hex(const uint8_t* h) {
    static const char* d = "0123456789abcdef";
    std::string s;
    for (int i = 0; i < 32; ++i) {
        s.push_back(d[h[i] >> 4]);
        s.push_back(d[h[i] & 15]);
    }
    return s;
}

// Arena layout: tensors packed at 16-byte aligned element offsets.
std::vector<uint64_t> arena_offsets(const std::vector<uint64_t>& numel, uint64_t& total) {
    std::vector<uint64_t> off(numel.size());
    uint64_t o = 0;
    for (size_t i = 0; i < numel.size(); ++i) {
        off[i] = o;
        o += (numel[i] + 7) & ~7ull;
    }
    total = o;
    return off;
}

pulse_result fetch_result(Engine& E, const void* dev_result) {
    pulse_result r{};
    cuda_check(counted_copy(&r, dev_result, sizeof(r), cudaMemcpyDeviceToHost, E.stream), "result");
    E.sync();
    uint64_t wd[7];
    if (pulse_watchdog(wd)) raise(PULSE_E_CUDA, "device watchdog fired (kind " + std::to_string(wd[1]) + ")");
    return r;
}

// Boundaries [0 = b0 < b1 < ... = n] of the runs of consecutive patch entries in which
// no target tensor repeats (greedy, in patch order).  One run (two boundaries) when
// the patch names every tensor at most once.
std::vector<uint32_t> distinct_target_runs(const uint32_t* target, uint32_t n) {
    std::vector<uint32_t> b{0};
    std::unordered_set<uint32_t> seen;
    for (uint32_t k = 0; k < n; ++k) {
        if (!seen.insert(target[k]).second) {
            b.push_back(k);
            seen.clear();
            seen.insert(target[k]);
        }
    }
    b.push_back(n);
    return b;
}

// Exception text for a device-detected failure, in the reference's words.
std::string device_message(const pulse_result& r, const std::string& name, const RawVec<int64_t>* idx,
                           uint32_t repr = PULSE_COO_INT32) {
    switch (r.err_check) {
        case PULSE_CHECK_TRUNCATED: return "unexpected end of data";
        case PULSE_CHECK_ZERO_GAP: return "zero index gap in tensor '" + name + "'";
        case PULSE_CHECK_ZERO_COL_GAP: return "non-positive column gap within a row";
        case PULSE_CHECK_COL_RANGE: return "column index out of range in tensor '" + name + "'";
        case PULSE_CHECK_INDEX_RANGE: return "index out of range in tensor '" + name + "'";
        case PULSE_CHECK_TRAILING:
            // patch.hpp:211-213 / 238-240 (int32 payloads) vs upscale_coo, index_coding.hpp:154-156
            return repr == PULSE_COO_DOWNSCALED ? "downscaled payload has trailing bytes"
                                                : "index payload has trailing bytes";
        case PULSE_CHECK_NEGATIVE: return "indices must be non-negative";
        case PULSE_CHECK_ORDER: return "indices must be strictly increasing";
        case PULSE_CHECK_FLAT_GAP: return "index gap exceeds 32 bits";
        case PULSE_CHECK_ROW_GAP: return "row gap exceeds 32 bits";
        case PULSE_CHECK_COL_ENTRY: return "column entry exceeds 32 bits";
        case PULSE_CHECK_INT32: return "tensor '" + name + "' is too large for 32-bit indices";
        case PULSE_CHECK_APPLY_ORDER: return "tensor '" + name + "' indices are not strictly increasing";
        case PULSE_CHECK_APPLY_RANGE: {
            std::string v = idx && r.err_elem < idx->size() ? std::to_string((*idx)[r.err_elem]) : "?";
            return "tensor '" + name + "' index " + v + " out of range";
        }
        default: return "capacity exceeded";
    }
}

// ---- codecs (compression.hpp:71-204, same libraries and calls) -----------------------------
std::vector<uint8_t> codec_compress(const uint8_t* raw, size_t n, uint32_t codec) {
    if (codec == PULSE_IDENTITY) return std::vector<uint8_t>(raw, raw + n);
    std::vector<uint8_t> out(8);
    for (int i = 0; i < 8; ++i) out[i] = uint8_t(uint64_t(n) >> (8 * i));
    if (n == 0) return out;
    size_t produced = 0;
    std::vector<uint8_t> stream;
    switch (codec) {
        case PULSE_LZ4: {
            if (n > 0x7E000000) raise(PULSE_E_ARGUMENT, "input too large for lz4 block format");
            stream.resize(size_t(LZ4_compressBound(int(n))));
            const int r = LZ4_compress_default(reinterpret_cast<const char*>(raw), reinterpret_cast<char*>(stream.data()),
                                               int(n), int(stream.size()));
            if (r <= 0) raise(PULSE_E_ERROR, "lz4 compression failed");
            produced = size_t(r);
            break;
        }
        case PULSE_ZSTD1:
        case PULSE_ZSTD3: {
            stream.resize(ZSTD_compressBound(n));
            produced = ZSTD_compress(stream.data(), stream.size(), raw, n, codec == PULSE_ZSTD1 ? 1 : 3);
            if (ZSTD_isError(produced)) raise(PULSE_E_ERROR, "zstd compression failed");
            break;
        }
        case PULSE_GZIP6: {
            uLongf p = compressBound(uLong(n));
            stream.resize(size_t(p));
            if (compress2(stream.data(), &p, raw, uLong(n), 6) != Z_OK) raise(PULSE_E_ERROR, "deflate compression failed");
            produced = size_t(p);
            break;
        }
        default: raise(PULSE_E_ARGUMENT, "unknown codec");
    }
    out.insert(out.end(), stream.begin(), stream.begin() + produced);
    return out;
}

std::vector<uint8_t> codec_decompress(const uint8_t* env, size_t n, uint32_t codec) {
    if (codec == PULSE_IDENTITY) return std::vector<uint8_t>(env, env + n);
    if (n < 8) raise(PULSE_E_CORRUPT_STREAM, "codec envelope shorter than its size prefix");
    uint64_t raw = 0;
    for (int i = 0; i < 8; ++i) raw |= uint64_t(env[i]) << (8 * i);
    if (raw > (1ull << 40)) raise(PULSE_E_CORRUPT_STREAM, "declared decompressed size is implausible");
    const uint8_t* body = env + 8;
    const size_t bn = n - 8;
    if (raw == 0) {
        if (bn) raise(PULSE_E_CORRUPT_STREAM, "codec envelope has trailing bytes");
        return {};
    }
    // A declared size the stream cannot possibly produce fails exactly as the
    // reference's decompression would (produced != raw_size), but without first
    // zero-filling up to 1 TiB of host memory for it: lz4 expands at most ~255x,
    // deflate ~1032x, and zstd reports a bound over all frames of the stream.
    {
        const char* what = nullptr;
        unsigned long long bound = 0;
        switch (codec) {
            case PULSE_LZ4: bound = 255ull * bn + 64; what = "lz4 stream is corrupt"; break;
            case PULSE_GZIP6: bound = 1032ull * bn + 64; what = "deflate stream is corrupt"; break;
            case PULSE_ZSTD1:
            case PULSE_ZSTD3: {
                const unsigned long long b = ZSTD_decompressBound(body, bn);
                bound = b >= (0ULL - 2) ? 0 : b;  // ZSTD_CONTENTSIZE_ERROR: no valid frame, nothing decodes
                what = "zstd stream is corrupt";
                break;
            }
            default: break;
        }
        if (what && raw > bound) raise(PULSE_E_CORRUPT_STREAM, what);
    }
    std::vector<uint8_t> out(raw);
    switch (codec) {
        case PULSE_LZ4: {
            if (bn > 0x7E000000) raise(PULSE_E_CORRUPT_STREAM, "lz4 stream is corrupt");
            const int r = LZ4_decompress_safe(reinterpret_cast<const char*>(body), reinterpret_cast<char*>(out.data()),
                                              int(bn), int(out.size()));
            if (r < 0 || uint64_t(r) != raw) raise(PULSE_E_CORRUPT_STREAM, "lz4 stream is corrupt");
            break;
        }
        case PULSE_ZSTD1:
        case PULSE_ZSTD3: {
            const size_t r = ZSTD_decompress(out.data(), out.size(), body, bn);
            if (ZSTD_isError(r) || r != raw) raise(PULSE_E_CORRUPT_STREAM, "zstd stream is corrupt");
            break;
        }
        case PULSE_GZIP6: {
            uLongf p = uLongf(raw);
            const int rc = uncompress(out.data(), &p, body, uLong(bn));
            if (rc != Z_OK || p != raw) raise(PULSE_E_CORRUPT_STREAM, "deflate stream is corrupt");
            break;
        }
        default: raise(PULSE_E_ARGUMENT, "unknown codec");
    }
    return out;
}

const char* repr_name(uint32_t r) {
    switch (r) {
        case PULSE_COO_DOWNSCALED: return "COO_DOWNSCALED";
        case PULSE_COO_INT32: return "COO_INT32";
        case PULSE_FLAT_INT32: return "FLAT_INT32";
    }
    raise(PULSE_E_ARGUMENT, "unknown representation");
}

// ---- device index coding over a host patch (patch.hpp:116-174) ----------------------------
// Returns the body (per tensor [index payload][value payload] for tensors with
// indices) and, per patch tensor, (index payload offset, length).
Coded device_index_code(Engine& E, const pulse_patch* p, bool with_values) {
    StageTimer tm{"index_code"};
    const uint32_t T = uint32_t(p->tensors.size());
    Coded out;
    out.payload.assign(T, {0, 0});
    out.val_off.assign(T, 0);
    if (T == 0) return out;
    // patch.hpp:99-103: int32 representations reject tensors of 2^31+ elements,
    // checked per tensor before its entries -- the host knows them up front.
    int64_t host_dim = -1;
    if (p->representation != PULSE_COO_DOWNSCALED)
        for (uint32_t t = 0; t < T; ++t)
            if (shape_numel(p->tensors[t].shape.data(), uint32_t(p->tensors[t].shape.size())) >= (1ull << 31)) {
                host_dim = t;
                break;
            }
    std::vector<pulse_tensor_geom> geom(T);
    std::vector<uint64_t> start(T + 1, 0);
    for (uint32_t t = 0; t < T; ++t) {
        const auto& tp = p->tensors[t];
        if (tp.shape.empty()) raise(PULSE_E_ARGUMENT, "tensor '" + tp.name + "' has empty shape");
        geom[t].numel = shape_numel(tp.shape.data(), uint32_t(tp.shape.size()));
        geom[t].cols = uint64_t(tp.shape.back());
        if (geom[t].numel == 0 || geom[t].cols == 0)
            raise(PULSE_E_ARGUMENT, "tensor '" + tp.name + "' has non-positive extent");
        start[t + 1] = start[t] + tp.indices.size();
    }
    const uint64_t n = start[T];
    pulse_plan* plan = E.get_plan(geom, std::max<uint64_t>(n, 1));
    const PlanDev& d = plan->dev;
    int64_t* didx = E.idx64.as<int64_t>(n);
    uint16_t* dval = E.vals.as<uint16_t>(n);
    RawVec<int64_t> flat_idx(n);
    RawVec<uint16_t> flat_val(n);
    pool().parallel_for(T, [&](size_t t) {  // per-tensor gather into the flat upload buffers
        const auto& tp = p->tensors[t];
        const size_t m = tp.indices.size();
        if (m) std::memcpy(flat_idx.data() + start[t], tp.indices.data(), m * 8);
        if (with_values && tp.values.size() == m) {
            if (m) std::memcpy(flat_val.data() + start[t], tp.values.data(), m * 2);
        } else if (m) {
            std::memset(flat_val.data() + start[t], 0, m * 2);
        }
    });
    tm.lap("gather");
    E.stager.h2d(didx, flat_idx.data(), n * 8, E.stream);
    E.stager.h2d(dval, flat_val.data(), n * 2, E.stream);
    cuda_check(counted_copy(d.id_start, start.data(), (T + 1) * 8, cudaMemcpyHostToDevice, E.stream), "H2D");
    tm.lap("h2d");
    // worst case per entry: COO_DOWNSCALED with both escapes, 5 + 6 index bytes + 2 value bytes
    const uint64_t cap = 13 * n + 64;
    uint8_t* dbody = E.body.as<uint8_t>(cap);
    auto* dent = E.entries.as<pulse_patch_entry>(T);
    auto* dres = E.result.as<pulse_result>(1);
    launch_encode_emit_idx64(d, p->representation, didx, dval, dbody, cap, dent, dres, E.stream);
    const pulse_result r = fetch_result(E, dres);
    tm.lap("device K2");
    if (host_dim >= 0 && (r.status == PULSE_OK || r.err_tensor >= uint64_t(host_dim)))
        raise(PULSE_E_DIMENSION, "tensor '" + p->tensors[host_dim].name + "' is too large for 32-bit indices");
    if (r.status != PULSE_OK) {
        const std::string nm = r.err_tensor < T ? p->tensors[r.err_tensor].name : "?";
        raise(pulse_status(r.status), device_message(r, nm, nullptr));
    }
    std::vector<pulse_patch_entry> ents(r.n_entries);
    if (r.n_entries)
        cuda_check(counted_copy(ents.data(), dent, r.n_entries * sizeof(pulse_patch_entry), cudaMemcpyDeviceToHost,
                                   E.stream), "D2H");
    out.body.resize(r.body_bytes);
    E.stager.d2h(out.body.data(), dbody, r.body_bytes, E.stream);
    E.sync();
    tm.lap("d2h");
    for (const auto& e : ents) {
        out.payload[e.tensor] = {e.idx_off, e.idx_nbytes};
        out.val_off[e.tensor] = e.val_off;
    }
    return out;
}

// Device decode of raw index payloads into indices (patch.hpp:178-262).
void device_decode_payloads(Engine& E, pulse_patch* p, const std::vector<const uint8_t*>& pl,
                            const std::vector<uint64_t>& lens) {
    const uint32_t T = uint32_t(p->tensors.size());
    if (T == 0) return;
    StageTimer tm{"read_patch_bytes decode"};
    std::vector<pulse_tensor_geom> geom(T);
    std::vector<pulse_patch_entry> ents(T);
    uint64_t body_len = 0, n = 0;
    for (uint32_t t = 0; t < T; ++t) {
        const auto& tp = p->tensors[t];
        geom[t].numel = shape_numel(tp.shape.data(), uint32_t(tp.shape.size()));
        geom[t].cols = uint64_t(tp.shape.back());
        ents[t].tensor = t;
        ents[t].reserved = 0;
        ents[t].count = tp.values.size();
        ents[t].idx_off = body_len;
        ents[t].idx_nbytes = lens[t];
        ents[t].val_off = body_len + lens[t];
        body_len += lens[t];
        n += tp.values.size();
    }
    pulse_plan* plan = E.get_plan(geom, std::max<uint64_t>({n, body_len / 3 + 1, 1}));
    // each payload straight into its place in the device body (one pass through the staging)
    uint8_t* dbody = E.body.as<uint8_t>(body_len + 64);
    for (uint32_t t = 0; t < T; ++t)
        if (lens[t]) E.stager.h2d(dbody + ents[t].idx_off, pl[t], lens[t], E.stream);
    auto* dent = E.entries.as<pulse_patch_entry>(T);
    cuda_check(counted_copy(dent, ents.data(), T * sizeof(pulse_patch_entry), cudaMemcpyHostToDevice, E.stream), "H2D");
    p->dev_idx_valid = false;
    if (p->dev_idx && (p->dev_idx_n < n || p->dev_idx_device != E.device)) {
        E.sync();
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(p->dev_idx_device);
        cudaFreeAsync(p->dev_idx, 0);
        cudaSetDevice(prev);
        p->dev_idx = nullptr;
    }
    tm.lap("upload");
    if (!p->dev_idx) {
        // from the device's stream-ordered pool: a patch per read must not pay cudaMalloc
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&p->dev_idx), std::max<uint64_t>(n, 1) * 8, E.stream),
                   "patch indices");
        p->dev_idx_n = std::max<uint64_t>(n, 1);
        p->dev_idx_device = E.device;
    }
    int64_t* dout = p->dev_idx;
    auto* dres = E.result.as<pulse_result>(1);
    launch_decode(plan->dev, p->representation, dbody, dent, T, nullptr, -1, dout, dres, E.stream);
    const pulse_result r = fetch_result(E, dres);
    tm.lap("device decode");
    if (r.status != PULSE_OK) {
        const std::string nm = r.err_tensor < T ? p->tensors[r.err_tensor].name : "?";
        raise(pulse_status(r.status), device_message(r, nm, nullptr, p->representation));
    }
    // each tensor's indices straight into its vector (no intermediate host copy), one pipelined D2H
    std::vector<std::pair<void*, size_t>> segs;
    segs.reserve(T);
    for (uint32_t t = 0; t < T; ++t) {
        auto& tp = p->tensors[t];
        tp.indices.resize(tp.values.size());
        if (!tp.indices.empty()) segs.emplace_back(tp.indices.data(), tp.indices.size() * 8);
    }
    E.stager.d2h_scatter(segs, dout, E.stream);
    E.sync();
    tm.lap("indices to host");
    p->dev_idx_valid = true;
}

void validate_for_write(const pulse_patch* p) {  // patch_file.hpp:31-42
    for (size_t i = 0; i < p->tensors.size(); ++i) {
        const auto& tp = p->tensors[i];
        if (tp.name.empty()) raise(PULSE_E_ARGUMENT, "tensor patch with empty name");
        if (i > 0 && !(p->tensors[i - 1].name < tp.name))
            raise(PULSE_E_ARGUMENT, "tensor patches must be in ascending name order");
        if (tp.shape.empty()) raise(PULSE_E_ARGUMENT, "tensor '" + tp.name + "' has empty shape");
        for (auto e : tp.shape)
            if (e <= 0) raise(PULSE_E_ARGUMENT, "tensor '" + tp.name + "' has non-positive extent");
        if (tp.indices.size() != tp.values.size())
            raise(PULSE_E_ARGUMENT, "tensor '" + tp.name + "' has mismatched index and value counts");
    }
}

std::vector<uint8_t> value_payload(const RawVec<uint16_t>& v) {  // patch.hpp:78-83 (LE u16)
    std::vector<uint8_t> out(v.size() * 2);
    for (size_t i = 0; i < v.size(); ++i) {
        out[2 * i] = uint8_t(v[i]);
        out[2 * i + 1] = uint8_t(v[i] >> 8);
    }
    return out;
}

// One tensor's record and its two (codec-applied) blobs for assemble_pulp.
struct PulpTensorRef {
    const std::string* name;
    const std::vector<int64_t>* shape;
    uint64_t count;
    const uint8_t* ip;
    uint64_t in;
    const uint8_t* vp;
    uint64_t vn;
};

// patch_file.hpp:44-83: the sorted-key JSON header (nlohmann, as the reference)
// and the container; blobs are copied in on the thread pool.
std::unique_ptr<pulse_bytes> assemble_pulp(int64_t anchor_step, int64_t base_step, int64_t target_step,
                                           const uint8_t* target_hash, uint32_t codec, uint32_t representation,
                                           const std::vector<PulpTensorRef>& refs) {
    const size_t T = refs.size();
    nlohmann::json header;
    header["anchor_step"] = anchor_step;
    header["base_step"] = base_step;
    header["target_step"] = target_step;
    header["target_hash"] = hex(target_hash);
    header["codec"] = codec;
    header["representation"] = repr_name(representation);
    auto& table = header["tensors"] = nlohmann::json::array();
    for (size_t t = 0; t < T; ++t) {
        const auto& r = refs[t];
        nlohmann::json e = {{"name", *r.name},
                            {"shape", *r.shape},
                            {"count", r.count},
                            {"index_nbytes", r.in},
                            {"value_nbytes", r.vn}};
        if (representation == PULSE_COO_DOWNSCALED) {
            e["row_bits"] = 8;
            e["col_bits"] = 16;
        }
        table.push_back(std::move(e));
    }
    const std::string js = header.dump();
    auto res = std::make_unique<pulse_bytes>();
    std::vector<uint64_t> at(T + 1);
    at[0] = 16 + js.size();
    for (size_t t = 0; t < T; ++t) at[t + 1] = at[t] + refs[t].in + refs[t].vn;
    res->v.resize(at[T]);
    uint8_t* w = res->v.data();
    std::memcpy(w, "PULP", 4);
    const uint32_t ver = 1;
    const uint64_t hl = js.size();
    for (int i = 0; i < 4; ++i) w[4 + i] = uint8_t(ver >> (8 * i));
    for (int i = 0; i < 8; ++i) w[8 + i] = uint8_t(hl >> (8 * i));
    std::memcpy(w + 16, js.data(), js.size());
    pool().parallel_for(T, [&](size_t t) {
        if (refs[t].in) std::memcpy(w + at[t], refs[t].ip, refs[t].in);
        if (refs[t].vn) std::memcpy(w + at[t] + refs[t].in, refs[t].vp, refs[t].vn);
    });
    return res;
}

// PULP container -> header, tensors (values filled, indices not yet decoded) and
// each tensor's raw (decompressed) index payload: patch_file.hpp:85-147 up to
// the index decoding, with the reference's checks and error order.
struct ParsedPulp {
    std::unique_ptr<pulse_patch> p;
    std::vector<std::vector<uint8_t>> store;  // decompressed index payloads (non-identity codecs)
    std::vector<const uint8_t*> pl;           // index payload of each tensor
    std::vector<uint64_t> lens;
};

ParsedPulp parse_pulp(const uint8_t* bytes, uint64_t n) {
    uint64_t pos = 0;
    auto need = [&](uint64_t k) {
        if (n - pos < k) raise(PULSE_E_TRUNCATION, "unexpected end of data");
    };
    if (n < 4) raise(PULSE_E_TRUNCATION, "patch shorter than magic");
    if (std::memcmp(bytes, "PULP", 4) != 0) raise(PULSE_E_BAD_MAGIC, "not a patch file (bad magic)");
    pos = 4;
    need(4);
    uint32_t version = 0;
    for (int i = 0; i < 4; ++i) version |= uint32_t(bytes[pos + i]) << (8 * i);
    pos += 4;
    if (version != 1) raise(PULSE_E_VERSION, "unsupported patch version " + std::to_string(version));
    need(8);
    uint64_t hl = 0;
    for (int i = 0; i < 8; ++i) hl |= uint64_t(bytes[pos + i]) << (8 * i);
    pos += 8;
    if (hl > n - pos) raise(PULSE_E_TRUNCATION, "patch header truncated");
    nlohmann::json header;
    try {
        header = nlohmann::json::parse(bytes + pos, bytes + pos + hl);
    } catch (const nlohmann::json::exception& e) {
        raise(PULSE_E_FORMAT, std::string("patch header is not valid JSON: ") + e.what());
    }
    pos += hl;
    auto p = std::make_unique<pulse_patch>();
    // Pass 1 (sequential, cheap): header fields and blob bounds of every tensor.
    // The first failure is recorded, not raised: an earlier tensor's codec
    // error must still win, as in the reference's one-tensor-at-a-time read.
    struct Blob {
        uint64_t count, ipos, inb, vpos, vnb;
        bool vtrunc;  // value blob runs past the end: raised after this tensor's index blob decompresses
    };
    std::vector<Blob> blobs;
    pulse_status stop_st = PULSE_OK;
    std::string stop_msg;
    try {
        p->anchor_step = header.at("anchor_step").get<int64_t>();
        p->base_step = header.at("base_step").get<int64_t>();
        p->target_step = header.at("target_step").get<int64_t>();
        const std::string hx = header.at("target_hash").get<std::string>();
        if (hx.size() != 64) raise(PULSE_E_FORMAT, "sha256 hex digest must be 64 characters");
        for (int i = 0; i < 32; ++i) {
            auto nib = [](char ch) -> int {
                if (ch >= '0' && ch <= '9') return ch - '0';
                if (ch >= 'a' && ch <= 'f') return ch - 'a' + 10;
                if (ch >= 'A' && ch <= 'F') return ch - 'A' + 10;
                raise(PULSE_E_FORMAT, "invalid hex character in digest");
            };
            p->target_hash[i] = uint8_t(nib(hx[2 * i]) << 4 | nib(hx[2 * i + 1]));
        }
        const uint32_t codec = header.at("codec").get<uint32_t>();
        if (codec > PULSE_GZIP6) raise(PULSE_E_FORMAT, "unknown codec id " + std::to_string(codec));
        p->codec = codec;
        const std::string rn = header.at("representation").get<std::string>();
        if (rn == "COO_DOWNSCALED") p->representation = PULSE_COO_DOWNSCALED;
        else if (rn == "COO_INT32") p->representation = PULSE_COO_INT32;
        else if (rn == "FLAT_INT32") p->representation = PULSE_FLAT_INT32;
        else raise(PULSE_E_FORMAT, "unknown representation name: " + rn);
    } catch (const nlohmann::json::exception& e) {
        raise(PULSE_E_FORMAT, std::string("patch header schema error: ") + e.what());
    }
    try {
        for (const auto& entry : header.at("tensors")) {
            PatchTensor tp;
            tp.name = entry.at("name").get<std::string>();
            tp.shape = entry.at("shape").get<std::vector<int64_t>>();
            for (auto e : tp.shape)
                if (e <= 0) raise(PULSE_E_FORMAT, "non-positive extent in tensor " + tp.name);
            Blob b{};
            b.count = entry.at("count").get<uint64_t>();
            b.inb = entry.at("index_nbytes").get<uint64_t>();
            b.vnb = entry.at("value_nbytes").get<uint64_t>();
            if (p->representation == PULSE_COO_DOWNSCALED) {
                if (entry.at("row_bits").get<int>() != 8 || entry.at("col_bits").get<int>() != 16)
                    raise(PULSE_E_FORMAT, "unsupported delta widths for tensor " + tp.name);
            }
            if (b.inb > n - pos) raise(PULSE_E_TRUNCATION, "index blob truncated");
            b.ipos = pos;
            pos += b.inb;
            if (b.vnb > n - pos) {
                // patch_file.hpp:129-131: the reference decompresses this tensor's index
                // blob before it finds the value blob short, so a codec error there wins
                b.vtrunc = true;
                blobs.push_back(b);
                p->tensors.push_back(std::move(tp));
                raise(PULSE_E_TRUNCATION, "value blob truncated");
            }
            b.vpos = pos;
            pos += b.vnb;
            blobs.push_back(b);
            p->tensors.push_back(std::move(tp));
        }
    } catch (const nlohmann::json::exception& e) {
        stop_st = PULSE_E_FORMAT;
        stop_msg = std::string("patch header schema error: ") + e.what();
    } catch (const Failure& f) {
        stop_st = f.st;
        stop_msg = f.msg;
    }
    // Pass 2 (parallel over tensors): decompress, values (LE u16, memcpy on
    // this little-endian host).  The identity codec's index blobs are used in place.
    const size_t T = blobs.size();
    ParsedPulp out;
    std::vector<std::vector<uint8_t>>& payloads = out.store;
    std::vector<const uint8_t*>& pl = out.pl;
    std::vector<uint64_t>& lens = out.lens;
    payloads.resize(T);
    pl.resize(T);
    lens.resize(T);
    std::vector<pulse_status> tst(T, PULSE_OK);
    std::vector<std::string> tmsg(T);
    pool().parallel_for(T, [&](size_t t) {
        const Blob& b = blobs[t];
        auto& tp = p->tensors[t];
        try {
            if (p->codec == PULSE_IDENTITY) {
                pl[t] = bytes + b.ipos;
                lens[t] = b.inb;
                if (b.vtrunc) raise(PULSE_E_TRUNCATION, "value blob truncated");
                if (b.vnb != b.count * 2)
                    raise(PULSE_E_FORMAT, "value payload length does not match change count for tensor " + tp.name);
                tp.values.resize(b.count);
                if (b.count) std::memcpy(tp.values.data(), bytes + b.vpos, b.count * 2);
            } else {
                payloads[t] = codec_decompress(bytes + b.ipos, b.inb, p->codec);
                pl[t] = payloads[t].data();
                lens[t] = payloads[t].size();
                if (b.vtrunc) raise(PULSE_E_TRUNCATION, "value blob truncated");
                const auto vp = codec_decompress(bytes + b.vpos, b.vnb, p->codec);
                if (vp.size() != b.count * 2)
                    raise(PULSE_E_FORMAT, "value payload length does not match change count for tensor " + tp.name);
                tp.values.resize(b.count);
                if (b.count) std::memcpy(tp.values.data(), vp.data(), b.count * 2);
            }
        } catch (const Failure& f) {
            tst[t] = f.st;
            tmsg[t] = f.msg;
        }
    });
    for (size_t t = 0; t < T; ++t)
        if (tst[t] != PULSE_OK) raise(tst[t], tmsg[t]);
    if (stop_st != PULSE_OK) raise(stop_st, stop_msg);
    if (pos != n) raise(PULSE_E_FORMAT, "patch has trailing bytes");
    out.p = std::move(p);
    return out;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

// ---- objects --------------------------------------------------------------------------------
pulse_status pulse_patch_new(pulse_patch** out) {
    if (!out) return fail(PULSE_E_ARGUMENT, "null output");
    *out = new pulse_patch();
    return PULSE_OK;
}
void pulse_patch_free(pulse_patch* p) { delete p; }

pulse_status pulse_patch_get_header(const pulse_patch* p, pulse_patch_header* h) {
    if (!p || !h) return fail(PULSE_E_ARGUMENT, "null argument");
    h->base_step = p->base_step;
    h->target_step = p->target_step;
    h->anchor_step = p->anchor_step;
    h->representation = p->representation;
    h->codec = p->codec;
    std::memcpy(h->target_hash, p->target_hash, 32);
    return PULSE_OK;
}
pulse_status pulse_patch_set_header(pulse_patch* p, const pulse_patch_header* h) {
    if (!p || !h) return fail(PULSE_E_ARGUMENT, "null argument");
    p->base_step = h->base_step;
    p->target_step = h->target_step;
    p->anchor_step = h->anchor_step;
    p->representation = h->representation;
    p->codec = h->codec;
    std::memcpy(p->target_hash, h->target_hash, 32);
    return PULSE_OK;
}
uint32_t pulse_patch_num_tensors(const pulse_patch* p) { return p ? uint32_t(p->tensors.size()) : 0; }
pulse_status pulse_patch_get_tensor(const pulse_patch* p, uint32_t i, pulse_tensor_patch* v) {
    if (!p || !v || i >= p->tensors.size()) return fail(PULSE_E_ARGUMENT, "bad tensor index");
    const auto& t = p->tensors[i];
    v->name = t.name.c_str();
    v->shape = t.shape.data();
    v->rank = uint32_t(t.shape.size());
    v->indices = t.indices.data();
    v->n_indices = t.indices.size();
    v->values = t.values.data();
    v->n_values = t.values.size();
    return PULSE_OK;
}
pulse_status pulse_patch_add_tensor(pulse_patch* p, const pulse_tensor_patch* v) {
    if (!p || !v) return fail(PULSE_E_ARGUMENT, "null argument");
    PatchTensor t;
    t.name = v->name ? v->name : "";
    t.shape.assign(v->shape, v->shape + v->rank);
    t.indices.assign(v->indices, v->indices + v->n_indices);
    t.values.assign(v->values, v->values + v->n_values);
    p->tensors.push_back(std::move(t));
    p->coded_valid = false;
    p->dev_idx_valid = false;
    return PULSE_OK;
}

const uint8_t* pulse_bytes_data(const pulse_bytes* b) { return b ? b->v.data() : nullptr; }
uint64_t pulse_bytes_size(const pulse_bytes* b) { return b ? b->v.size() : 0; }
void pulse_bytes_free(pulse_bytes* b) { delete b; }

// ---- patch.hpp ------------------------------------------------------------------------------
pulse_status pulse_encode(const pulse_checkpoint* current, const pulse_checkpoint* previous, uint32_t repr,
                          uint32_t codec, pulse_patch** out) {
    return guarded([&] {
        if (!current || !previous || !out) raise(PULSE_E_ARGUMENT, "null argument");
        validate_checkpoint(current);
        validate_checkpoint(previous);
        const auto co = sorted_order(current), po = sorted_order(previous);
        if (co.size() != po.size()) raise(PULSE_E_TENSOR_SET, "checkpoints have different tensor counts");
        auto patch = std::make_unique<pulse_patch>();
        patch->base_step = int64_t(previous->step);
        patch->target_step = int64_t(current->step);
        patch->anchor_step = int64_t(previous->step);
        patch->representation = repr;
        patch->codec = codec;
        repr_name(repr);
        // target hash on a host thread, overlapping the device work
        auto hash = std::async(std::launch::async, [&] { hash_checkpoint(current, patch->target_hash); });
        struct HashJoin {
            std::future<void>& f;
            ~HashJoin() {
                if (f.valid()) f.wait();
            }
        } join{hash};
        const uint32_t T = uint32_t(co.size());
        std::vector<pulse_tensor_geom> geom(T);
        std::vector<uint64_t> numel(T);
        for (uint32_t k = 0; k < T; ++k) {
            const pulse_tensor& c = current->tensors[co[k]];
            const pulse_tensor& q = previous->tensors[po[k]];
            if (std::strcmp(c.name, q.name) != 0)
                raise(PULSE_E_TENSOR_SET, std::string("tensor sets differ: '") + c.name + "' vs '" + q.name + "'");
            if (c.rank != q.rank || !std::equal(c.shape, c.shape + c.rank, q.shape))
                raise(PULSE_E_SHAPE_MISMATCH, std::string("tensor '") + c.name + "' changed shape between checkpoints");
            geom[k].numel = c.numel;
            geom[k].cols = uint64_t(c.shape[c.rank - 1]);
            numel[k] = c.numel;
        }
        StageTimer tm{"encode"};
        if (T > 0) {
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            uint64_t total = 0;
            const auto off = arena_offsets(numel, total);
            uint16_t* A = E.arena_a.as<uint16_t>(total);
            uint16_t* B = E.arena_b.as<uint16_t>(total);
            for (uint32_t k = 0; k < T; ++k) {
                E.stager.h2d(A + off[k], previous->tensors[po[k]].data, numel[k] * 2, E.stream);
                E.stager.h2d(B + off[k], current->tensors[co[k]].data, numel[k] * 2, E.stream);
            }
            uint64_t cap = std::max<uint64_t>(total / 64, 1 << 20);
            pulse_scan_summary sm{};
            pulse_plan* plan = nullptr;
            for (int attempt = 0; attempt < 2; ++attempt) {
                plan = E.get_plan(geom, cap);
                std::vector<const void*> pa(T), pb(T);
                for (uint32_t k = 0; k < T; ++k) {
                    pa[k] = A + off[k];
                    pb[k] = B + off[k];
                }
                if (pulse_plan_bind(plan, 0, pa.data()) || pulse_plan_bind(plan, 1, pb.data()))
                    raise(PULSE_E_CUDA, pulse_last_error());
                if (pulse_encode_scan(plan, 1, 0, nullptr, E.stream)) raise(PULSE_E_CUDA, pulse_last_error());
                cuda_check(counted_copy(&sm, plan->dev.scan, sizeof(sm), cudaMemcpyDeviceToHost, E.stream), "D2H");
                E.sync();
                if (sm.status != PULSE_E_CAPACITY) break;
                cap = sm.n_changes + sm.n_changes / 16 + 1024;
            }
            tm.lap("upload + scan");
            const uint64_t n = sm.n_changes;
            const PlanDev& d = plan->dev;
            std::vector<uint64_t> seg_start(d.n_segs + 1);
            cuda_check(counted_copy(seg_start.data(), d.seg_start, seg_start.size() * 8, cudaMemcpyDeviceToHost, E.stream), "D2H");
            int64_t* didx = E.out64.as<int64_t>(n);
            launch_export_indices(d, didx, E.stream);
            RawVec<int64_t> idx(n);
            RawVec<uint16_t> val(n);
            E.stager.d2h(idx.data(), didx, n * 8, E.stream);
            E.stager.d2h(val.data(), d.val16, n * 2, E.stream);
            E.sync();
            tm.lap("indices + values to host");
            // K2 too, while the snapshots are resident and the target hash is still running:
            // write_patch_bytes then reuses these payloads instead of uploading the indices again
            if (n > 0) {
                const uint64_t bcap = 14 * n + 1024;  // >= any escape-coded body
                uint8_t* dbody = E.body.as<uint8_t>(bcap + 64);
                auto* dent = E.entries.as<pulse_patch_entry>(T);
                auto* dres = E.result.as<pulse_result>(1);
                if (pulse_encode_emit(plan, repr, nullptr, 1, 0, dbody, bcap, dent, dres, E.stream) == PULSE_OK) {
                    const pulse_result er = fetch_result(E, dres);
                    if (er.status == PULSE_OK) {  // e.g. DimensionError: write_patch_bytes reports it
                        std::vector<pulse_patch_entry> ents(er.n_entries);
                        cuda_check(counted_copy(ents.data(), dent, er.n_entries * sizeof(pulse_patch_entry),
                                                cudaMemcpyDeviceToHost, E.stream), "D2H");
                        patch->coded.body.resize(er.body_bytes);
                        E.stager.d2h(patch->coded.body.data(), dbody, er.body_bytes, E.stream);
                        E.sync();
                        for (const auto& e : ents) {
                            patch->coded.payload.emplace_back(e.idx_off, e.idx_nbytes);
                            patch->coded.val_off.push_back(e.val_off);
                        }
                        patch->coded_valid = true;
                        patch->coded_repr = repr;
                    }
                }
            }
            // per-tensor ranges: segments of a tensor are consecutive (2^31-element splits)
            uint32_t sg = 0;
            for (uint32_t k = 0; k < T; ++k) {
                const uint64_t nseg = (numel[k] + kSegElems - 1) / kSegElems;
                const uint64_t lo = seg_start[sg], hi = seg_start[sg + nseg];
                sg += uint32_t(nseg);
                if (hi == lo) continue;  // unchanged tensors are omitted (patch.hpp:302-304)
                const pulse_tensor& c = current->tensors[co[k]];
                PatchTensor tp;
                tp.name = c.name;
                tp.shape.assign(c.shape, c.shape + c.rank);
                tp.indices.assign(idx.begin() + lo, idx.begin() + hi);
                tp.values.assign(val.begin() + lo, val.begin() + hi);
                patch->tensors.push_back(std::move(tp));
            }
            tm.lap("K2 body + patch tensors");
        }
        hash.get();
        tm.lap("target hash (overlapped)");
        *out = patch.release();
    });
}

pulse_status pulse_decode(const pulse_checkpoint* previous, const pulse_patch* patch, int verify_hash,
                          uint16_t* const* out_data, uint64_t* out_step) {
    return guarded([&] {
        if (!previous || !patch || (previous->n_tensors && !out_data)) raise(PULSE_E_ARGUMENT, "null argument");
        const uint32_t T = previous->n_tensors;
        // host checks in patch order (patch.hpp:314-324); the first failing tensor stops
        // the device validation there so errors surface in the reference's order
        const uint32_t P = uint32_t(patch->tensors.size());
        uint32_t stop = P;
        Failure host_err{PULSE_OK, ""};
        std::vector<uint32_t> target(P);
        for (uint32_t k = 0; k < P && stop == P; ++k) {
            const auto& tp = patch->tensors[k];
            int64_t f = -1;
            for (uint32_t i = 0; i < T; ++i)
                if (tp.name == previous->tensors[i].name) {
                    f = i;
                    break;
                }
            if (f < 0) {
                stop = k;
                host_err = {PULSE_E_TENSOR_SET, "patch references unknown tensor '" + tp.name + "'"};
                break;
            }
            const pulse_tensor& t = previous->tensors[f];
            if (t.rank != tp.shape.size() || !std::equal(tp.shape.begin(), tp.shape.end(), t.shape)) {
                stop = k;
                host_err = {PULSE_E_SHAPE_MISMATCH, "tensor '" + tp.name + "' shape differs between patch and checkpoint"};
                break;
            }
            if (tp.values.size() != tp.indices.size()) {
                stop = k;
                host_err = {PULSE_E_ARGUMENT, "tensor '" + tp.name + "' has mismatched index and value counts"};
                break;
            }
            target[k] = uint32_t(f);
        }
        StageTimer tm{"decode"};
        if (T > 0) {
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            tm.lap("host checks");
            std::vector<pulse_tensor_geom> geom(T);
            std::vector<uint64_t> numel(T);
            for (uint32_t i = 0; i < T; ++i) {
                const pulse_tensor& t = previous->tensors[i];
                numel[i] = t.numel;
                geom[i].numel = t.numel ? t.numel : 1;
                geom[i].cols = t.rank ? uint64_t(std::max<int64_t>(1, t.shape[t.rank - 1])) : 1;
                if (geom[i].numel % geom[i].cols) geom[i].cols = 1;
            }
            uint64_t total = 0, n = 0;
            const auto off = arena_offsets(numel, total);
            for (uint32_t k = 0; k < stop; ++k) n += patch->tensors[k].indices.size();
            uint16_t* A = E.arena_a.as<uint16_t>(total);
            // Page-locked base and output buffers and no host-side error: validate the
            // whole patch first, then run upload | scatter | download as a pipeline
            // over groups of tensors, so both copy engines work at once.
            // Duplicate tensor names (read_patch_bytes accepts them, patch_file.hpp:114-139):
            // the reference applies tensors one after another, so the last entry for a
            // tensor wins (patch.hpp:313-339).  Such patches validate as a whole, then
            // scatter in runs with no tensor twice, in patch order.
            const auto runs = distinct_target_runs(target.data(), stop);
            bool pipelined = stop == P && host_err.st == PULSE_OK && runs.size() <= 2;
            for (uint32_t i = 0; i < T && pipelined; ++i)
                if (numel[i] && !(is_pinned(previous->tensors[i].data) && is_pinned(out_data[i]))) pipelined = false;
            if (!pipelined)
                for (uint32_t i = 0; i < T; ++i) E.stager.h2d(A + off[i], previous->tensors[i].data, numel[i] * 2, E.stream);
            pulse_plan* plan = E.get_plan(geom, std::max<uint64_t>(n, 1));
            std::vector<const void*> pa(T);
            for (uint32_t i = 0; i < T; ++i) pa[i] = A + off[i];
            if (pulse_plan_bind(plan, 2, pa.data())) raise(PULSE_E_CUDA, pulse_last_error());
            int64_t* didx = nullptr;
            uint16_t* dval = nullptr;
            pulse_patch_entry* dent = nullptr;
            std::vector<uint64_t> at(stop + 1, 0);
            if (stop > 0 && n > 0) {
                std::vector<pulse_patch_entry> ents(stop);
                for (uint32_t k = 0; k < stop; ++k) {
                    const auto& tp = patch->tensors[k];
                    ents[k] = pulse_patch_entry{target[k], 0, tp.indices.size(), 0, 0, 0};
                    at[k + 1] = at[k] + tp.indices.size();
                }
                // each tensor's indices / values straight into their place on the device
                // (one pass through the pinned staging, no host-side gather copy)
                // indices a read_patch_bytes left on this device (same tensors, same order) are
                // used in place; otherwise uploaded
                const bool resident = patch->dev_idx_valid && patch->dev_idx_device == E.device &&
                                      patch->dev_idx_n >= n;
                didx = resident ? patch->dev_idx : E.idx64.as<int64_t>(n);
                dval = E.vals.as<uint16_t>(n);
                for (uint32_t k = 0; k < stop; ++k) {
                    const auto& tp = patch->tensors[k];
                    const size_t m = tp.indices.size();
                    if (!m) continue;
                    if (!resident) E.stager.h2d(didx + at[k], tp.indices.data(), m * 8, E.stream);
                    E.stager.h2d(dval + at[k], tp.values.data(), m * 2, E.stream);
                }
                dent = E.entries.as<pulse_patch_entry>(stop);
                cuda_check(counted_copy(dent, ents.data(), stop * sizeof(pulse_patch_entry), cudaMemcpyHostToDevice,
                                           E.stream), "H2D");
                auto* dres = E.result.as<pulse_result>(1);
                // sequential: validate + scatter in one go; pipelined: validate only here.
                // Runs (duplicate names; a launch covers at most one entry per tensor): validate
                // every run in patch order first -- the first failing run holds the reference's
                // first failure -- then scatter them in order.
                const bool whole = !pipelined && runs.size() <= 2;
                for (size_t q = 0; q + 1 < runs.size(); ++q) {
                    const uint32_t k0 = runs[q], k1 = runs[q + 1];
                    launch_apply_idx64(plan->dev, didx + at[k0], dval + at[k0], dent + k0, k1 - k0, whole ? 2 : -1,
                                       dres, E.stream);
                    const pulse_result r = fetch_result(E, dres);
                    if (r.status != PULSE_OK) {
                        const auto& tp = patch->tensors[k0 + r.err_tensor];
                        raise(pulse_status(r.status), device_message(r, tp.name, &tp.indices));
                    }
                }
                if (!pipelined && !whole)
                    for (size_t q = 0; q + 1 < runs.size(); ++q) {
                        const uint32_t k0 = runs[q], k1 = runs[q + 1];
                        launch_apply_idx64(plan->dev, didx + at[k0], dval + at[k0], dent + k0, k1 - k0, 2, dres,
                                           E.stream);
                    }
            }
            tm.lap(pipelined ? "gather+upload+validate" : "upload+gather+apply");
            if (host_err.st != PULSE_OK) raise(host_err.st, host_err.msg);
            if (!pipelined) {
                for (uint32_t i = 0; i < T; ++i) E.stager.d2h(out_data[i], A + off[i], numel[i] * 2, E.stream);
                E.sync();
            } else {
                // groups of ~1 GiB in name order; patch entries (name order) are contiguous per group
                const auto ord = sorted_order(previous);
                std::vector<uint32_t> rank_of(T);
                for (uint32_t r = 0; r < T; ++r) rank_of[ord[r]] = r;
                std::vector<std::array<uint32_t, 4>> groups;  // [r0, r1) tensors, [k0, k1) entries
                uint32_t k = 0;
                for (uint32_t r0 = 0; r0 < T;) {
                    uint32_t r1 = r0;
                    uint64_t bytes = 0;
                    while (r1 < T && (r1 == r0 || bytes + numel[ord[r1]] * 2 <= (1ull << 30))) bytes += numel[ord[r1++]] * 2;
                    const uint32_t k0 = k;
                    while (k < stop && rank_of[target[k]] < r1) ++k;
                    groups.push_back({r0, r1, k0, k});
                    r0 = r1;
                }
                if (k != stop) {  // entries not in name order: one group covers everything
                    groups.assign(1, {0u, T, 0u, stop});
                }
                E.pipeline_streams(groups.size());
                auto* gres = E.result.as<pulse_result>(1);
                for (size_t g = 0; g < groups.size(); ++g) {
                    const auto [r0, r1, k0, k1] = groups[g];
                    for (uint32_t r = r0; r < r1; ++r) {
                        const uint32_t i = ord[r];
                        if (numel[i])
                            cuda_check(counted_copy(A + off[i], previous->tensors[i].data, numel[i] * 2,
                                                    cudaMemcpyHostToDevice, E.s_up), "H2D");
                    }
                    cuda_check(cudaEventRecord(E.ev_up[g], E.s_up), "event");
                    cuda_check(cudaStreamWaitEvent(E.stream, E.ev_up[g], 0), "wait");
                    if (k1 > k0)
                        launch_apply_idx64(plan->dev, didx + at[k0], dval + at[k0], dent + k0, k1 - k0, 2, gres, E.stream);
                    cuda_check(cudaEventRecord(E.ev_cmp[g], E.stream), "event");
                    cuda_check(cudaStreamWaitEvent(E.s_dn, E.ev_cmp[g], 0), "wait");
                    for (uint32_t r = r0; r < r1; ++r) {
                        const uint32_t i = ord[r];
                        if (numel[i])
                            cuda_check(counted_copy(out_data[i], A + off[i], numel[i] * 2, cudaMemcpyDeviceToHost, E.s_dn),
                                       "D2H");
                    }
                }
                cuda_check(cudaStreamSynchronize(E.s_dn), "D2H sync");
                cuda_check(cudaStreamSynchronize(E.stream), "stream sync");
            }
            tm.lap(pipelined ? "pipeline" : "download");
        } else if (host_err.st != PULSE_OK) {
            raise(host_err.st, host_err.msg);
        }
        if (out_step) *out_step = uint64_t(patch->target_step);
        if (verify_hash) {  // patch.hpp:341-346
            pulse_checkpoint outck{uint64_t(patch->target_step), nullptr, T};
            std::vector<pulse_tensor> ts(T);
            for (uint32_t i = 0; i < T; ++i) {
                ts[i] = previous->tensors[i];
                ts[i].data = out_data[i];
            }
            outck.tensors = ts.data();
            uint8_t h[32];
            hash_checkpoint(&outck, h);
            if (std::memcmp(h, patch->target_hash, 32) != 0)
                raise(PULSE_E_HASH_MISMATCH, "hash mismatch: expected " + hex(patch->target_hash) + ", actual " + hex(h));
        }
    });
}

pulse_status pulse_encode_index_payloads(const pulse_patch* patch, pulse_bytes** concat, uint64_t* sizes) {
    return guarded([&] {
        if (!patch || !concat) raise(PULSE_E_ARGUMENT, "null argument");
        repr_name(patch->representation);
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        const Coded c = device_index_code(E, patch, false);
        auto out = std::make_unique<pulse_bytes>();
        for (size_t t = 0; t < patch->tensors.size(); ++t) {
            const auto [o, len] = c.payload[t];
            if (sizes) sizes[t] = len;
            out->v.insert(out->v.end(), c.body.begin() + o, c.body.begin() + o + len);
        }
        *concat = out.release();
    });
}

pulse_status pulse_decode_index_payloads(pulse_patch* patch, const uint8_t* const* payloads, const uint64_t* sizes,
                                         uint32_t n) {
    return guarded([&] {
        if (!patch) raise(PULSE_E_ARGUMENT, "null argument");
        if (n != patch->tensors.size()) raise(PULSE_E_ARGUMENT, "payload count does not match tensor count");
        repr_name(patch->representation);
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        std::vector<const uint8_t*> pl(payloads, payloads + n);
        std::vector<uint64_t> lens(sizes, sizes + n);
        patch->coded_valid = false;
        device_decode_payloads(E, patch, pl, lens);
    });
}

// ---- patch_file.hpp -------------------------------------------------------------------------
pulse_status pulse_write_patch_bytes(const pulse_patch* p, pulse_bytes** out) {
    return guarded([&] {
        if (!p || !out) raise(PULSE_E_ARGUMENT, "null argument");
        validate_for_write(p);
        repr_name(p->representation);  // validates the representation
        if (p->codec > PULSE_GZIP6) raise(PULSE_E_ARGUMENT, "unknown codec");
        StageTimer tm{"write_patch_bytes"};
        Coded computed;
        const bool reuse = p->coded_valid && p->coded_repr == p->representation &&
                           p->coded.payload.size() == p->tensors.size();
        if (!reuse) {
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            computed = device_index_code(E, p, true);
        }
        const Coded& c = reuse ? p->coded : computed;
        tm.lap(reuse ? "index coding (from encode)" : "index coding");
        const size_t T = p->tensors.size();
        // per tensor: its index blob and value blob (identity codec: straight out
        // of the device body, no intermediate copy)
        std::vector<std::vector<uint8_t>> ib(T), vb(T);
        std::vector<const uint8_t*> ip(T), vp(T);
        std::vector<uint64_t> in(T), vn(T);
        pool().parallel_for(T, [&](size_t t) {  // blobs are independent: same bytes in any order
            const auto [o, len] = c.payload[t];
            const bool body_vals = len || p->tensors[t].values.empty();
            if (p->codec == PULSE_IDENTITY && body_vals) {
                ip[t] = c.body.data() + o;
                in[t] = len;
                vp[t] = c.body.data() + c.val_off[t];
                vn[t] = p->tensors[t].values.size() * 2;
                return;
            }
            ib[t] = codec_compress(c.body.data() + o, len, p->codec);
            if (body_vals) {
                const uint8_t* v = c.body.data() + c.val_off[t];
                vb[t] = codec_compress(v, p->tensors[t].values.size() * 2, p->codec);
            } else {
                const auto raw = value_payload(p->tensors[t].values);
                vb[t] = codec_compress(raw.data(), raw.size(), p->codec);
            }
            ip[t] = ib[t].data();
            in[t] = ib[t].size();
            vp[t] = vb[t].data();
            vn[t] = vb[t].size();
        });
        tm.lap("codec");
        std::vector<PulpTensorRef> refs(T);
        for (size_t t = 0; t < T; ++t) {
            const auto& tp = p->tensors[t];
            refs[t] = {&tp.name, &tp.shape, tp.indices.size(), ip[t], in[t], vp[t], vn[t]};
        }
        auto res = assemble_pulp(p->anchor_step, p->base_step, p->target_step, p->target_hash, p->codec,
                                 p->representation, refs);
        tm.lap("assemble");
        *out = res.release();
    });
}

pulse_status pulse_read_patch_bytes(const uint8_t* bytes, uint64_t n, pulse_patch** out) {
    return guarded([&] {
        if (!out || (n && !bytes)) raise(PULSE_E_ARGUMENT, "null argument");
        StageTimer tm{"read_patch_bytes"};
        ParsedPulp pp = parse_pulp(bytes, n);
        tm.lap("parse");
        if (!pp.p->tensors.empty()) {
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            device_decode_payloads(E, pp.p.get(), pp.pl, pp.lens);
        }
        *out = pp.p.release();
    });
}

void pulse_transfer_stats(uint64_t* h2d, uint64_t* d2h, int reset) {
    if (h2d) *h2d = g_h2d_bytes.load();
    if (d2h) *d2h = g_d2h_bytes.load();
    if (reset) {
        g_h2d_bytes = 0;
        g_d2h_bytes = 0;
    }
}

// ---- absorption.hpp analyses -----------------------------------------------------------------
namespace {
// Uploads the given tensors (one or two snapshots, same geometry) into the
// engine arenas and binds them to slots 0 / 1 of a plan over that geometry.
pulse_plan* bind_for_count(Engine& E, const std::vector<const pulse_tensor*>& a,
                           const std::vector<const pulse_tensor*>* b) {
    std::vector<pulse_tensor_geom> geom(a.size());
    std::vector<uint64_t> numel(a.size());
    for (size_t k = 0; k < a.size(); ++k) {
        geom[k].numel = a[k]->numel;
        geom[k].cols = uint64_t(a[k]->shape[a[k]->rank - 1]);
        numel[k] = a[k]->numel;
    }
    uint64_t total = 0;
    const auto off = arena_offsets(numel, total);
    uint16_t* A = E.arena_a.as<uint16_t>(total);
    uint16_t* B = b ? E.arena_b.as<uint16_t>(total) : nullptr;
    for (size_t k = 0; k < a.size(); ++k) {
        E.stager.h2d(A + off[k], a[k]->data, numel[k] * 2, E.stream);
        if (b) E.stager.h2d(B + off[k], (*b)[k]->data, numel[k] * 2, E.stream);
    }
    pulse_plan* plan = E.get_plan(geom, 1);
    std::vector<const void*> pa(a.size()), pb(a.size());
    for (size_t k = 0; k < a.size(); ++k) {
        pa[k] = A + off[k];
        if (b) pb[k] = B + off[k];
    }
    if (pulse_plan_bind(plan, 0, pa.data()) || (b && pulse_plan_bind(plan, 1, pb.data())))
        raise(PULSE_E_CUDA, pulse_last_error());
    return plan;
}

uint64_t read_count(Engine& E) {
    uint64_t* d = E.misc.as<uint64_t>(2);
    uint64_t h = 0;
    cuda_check(counted_copy(&h, d, 8, cudaMemcpyDeviceToHost, E.stream), "D2H");
    E.sync();
    return h;
}

// Largest bf16 magnitude pattern m in [0, 0x7F80] whose value is <= t, or -1
// (every non-NaN |w| exceeds t); |w| > t  <=>  (bits & 0x7FFF) > m for non-NaN w.
int32_t magnitude_cutoff(double t) {
    auto value = [](uint32_t m) {
        const uint32_t f = m << 16;
        float x;
        std::memcpy(&x, &f, 4);
        return double(x);
    };
    if (!(value(0) <= t)) return -1;
    uint32_t lo = 0, hi = 0x7F80;  // value(lo) <= t
    if (value(hi) <= t) return int32_t(hi);
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) / 2;
        if (value(mid) <= t) lo = mid; else hi = mid;
    }
    return int32_t(lo);
}
}  // namespace

pulse_status pulse_sparsity(const pulse_checkpoint* a, const pulse_checkpoint* b, uint64_t k,
                            pulse_sparsity_report* out) {
    return guarded([&] {
        if (!a || !b || !out) raise(PULSE_E_ARGUMENT, "null argument");
        const auto oa = sorted_order(a), ob = sorted_order(b);
        if (oa.size() != ob.size()) raise(PULSE_E_TENSOR_SET, "checkpoints have different tensor counts");
        std::vector<const pulse_tensor*> ta, tb;
        uint64_t total = 0;
        for (size_t i = 0; i < oa.size(); ++i) {
            const pulse_tensor& x = a->tensors[oa[i]];
            const pulse_tensor& y = b->tensors[ob[i]];
            if (std::strcmp(x.name, y.name) != 0)
                raise(PULSE_E_TENSOR_SET, std::string("tensor sets differ: '") + x.name + "' vs '" + y.name + "'");
            if (x.rank != y.rank || !std::equal(x.shape, x.shape + x.rank, y.shape) || x.numel != y.numel)
                raise(PULSE_E_SHAPE_MISMATCH, std::string("tensor '") + x.name + "' shapes differ");
            total += x.numel;
            if (x.numel) {
                ta.push_back(&x);
                tb.push_back(&y);
            }
        }
        uint64_t changed = 0;
        if (!ta.empty()) {
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            pulse_plan* plan = bind_for_count(E, ta, &tb);
            if (pulse_count_changed(plan, 0, 1, E.misc.as<uint64_t>(2), E.stream)) raise(PULSE_E_CUDA, pulse_last_error());
            changed = read_count(E);
        }
        out->k = k;
        out->changed = changed;
        out->total = total;
        out->sparsity = total ? 1.0 - double(changed) / double(total) : 1.0;
    });
}

pulse_status pulse_frozen_fraction(const pulse_checkpoint* c, double threshold, double* out) {
    return guarded([&] {
        if (!c || !out) raise(PULSE_E_ARGUMENT, "null argument");
        std::vector<const pulse_tensor*> ts;
        uint64_t total = 0;
        for (uint32_t i = 0; i < c->n_tensors; ++i) {
            total += c->tensors[i].numel;
            if (c->tensors[i].numel) ts.push_back(&c->tensors[i]);
        }
        if (total == 0) raise(PULSE_E_ARGUMENT, "frozen fraction of an empty checkpoint is undefined");
        uint64_t above = 0;
        if (!std::isnan(threshold)) {  // |w| > NaN is false for every weight
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            pulse_plan* plan = bind_for_count(E, ts, nullptr);
            const uint32_t cut = uint32_t(magnitude_cutoff(threshold));
            if (pulse_count_above(plan, 0, cut, E.misc.as<uint64_t>(2), E.stream)) raise(PULSE_E_CUDA, pulse_last_error());
            above = read_count(E);
        }
        *out = double(above) / double(total);
    });
}

// ---- sha256.hpp -----------------------------------------------------------------------------
pulse_status pulse_hash_weights(const pulse_checkpoint* c, uint8_t* out32) {
    return guarded([&] {
        if (!c || !out32) raise(PULSE_E_ARGUMENT, "null argument");
        hash_checkpoint(c, out32);
    });
}

pulse_status pulse_sha256_new(pulse_sha256_ctx** out) {
    return guarded([&] {
        auto* s = new pulse_sha256_ctx{EVP_MD_CTX_new()};
        if (!s->ctx || EVP_DigestInit_ex(s->ctx, EVP_sha256(), nullptr) != 1) {
            delete s;
            raise(PULSE_E_ERROR, "failed to initialize SHA-256 context");
        }
        *out = s;
    });
}
pulse_status pulse_sha256_update(pulse_sha256_ctx* s, const uint8_t* data, uint64_t n) {
    if (!s) return fail(PULSE_E_ARGUMENT, "null context");
    if (n && EVP_DigestUpdate(s->ctx, data, n) != 1) return fail(PULSE_E_ERROR, "SHA-256 update failed");
    return PULSE_OK;
}
pulse_status pulse_sha256_final(pulse_sha256_ctx* s, uint8_t* out32) {
    if (!s) return fail(PULSE_E_ARGUMENT, "null context");
    unsigned int len = 0;
    if (EVP_DigestFinal_ex(s->ctx, out32, &len) != 1 || len != 32) return fail(PULSE_E_ERROR, "SHA-256 finalize failed");
    return PULSE_OK;
}
void pulse_sha256_free(pulse_sha256_ctx* s) {
    if (s) {
        EVP_MD_CTX_free(s->ctx);
        delete s;
    }
}

// ---- index_coding.hpp -----------------------------------------------------------------------
pulse_status pulse_delta_encode_indices(const int64_t* in, uint64_t n, int64_t* out) {
    return guarded([&] {
        if (n == 0) return;
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        int64_t* d = E.idx64.as<int64_t>(2 * n);
        uint64_t* err = E.misc.as<uint64_t>(1);
        cuda_check(cudaMemsetAsync(err, 0xFF, 8, E.stream), "memset");
        E.stager.h2d(d, in, n * 8, E.stream);
        launch_delta_encode(d, n, d + n, err, E.stream);
        uint64_t k = 0;
        cuda_check(counted_copy(&k, err, 8, cudaMemcpyDeviceToHost, E.stream), "D2H");
        E.sync();
        if (k != kNoError)
            raise(PULSE_E_ARGUMENT, key_check(k) == kArgNegative ? "indices must be non-negative"
                                                                  : "indices must be strictly increasing");
        E.stager.d2h(out, d + n, n * 8, E.stream);
    });
}

pulse_status pulse_delta_decode_indices(const int64_t* in, uint64_t n, int64_t* out) {
    return guarded([&] {
        if (n == 0) return;
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        int64_t* d = E.idx64.as<int64_t>(2 * n);
        uint64_t* err = E.misc.as<uint64_t>(1);
        cuda_check(cudaMemsetAsync(err, 0xFF, 8, E.stream), "memset");
        E.stager.h2d(d, in, n * 8, E.stream);
        launch_delta_decode(d, n, d + n, err, E.stream);
        uint64_t k = 0;
        cuda_check(counted_copy(&k, err, 8, cudaMemcpyDeviceToHost, E.stream), "D2H");
        E.sync();
        if (k != kNoError)
            raise(PULSE_E_FORMAT, key_elem(k) == 0 ? "first index gap is negative"
                                                    : "non-positive index gap after the first element");
        E.stager.d2h(out, d + n, n * 8, E.stream);
    });
}

pulse_status pulse_downscale_coo(const int64_t* rows, uint64_t n_rows, const int64_t* cols, uint64_t n_cols,
                                 pulse_bytes** out) {
    return guarded([&] {
        if (!out) raise(PULSE_E_ARGUMENT, "null argument");
        if (n_rows != n_cols) raise(PULSE_E_ARGUMENT, "row and column lists differ in length");
        auto res = std::make_unique<pulse_bytes>();
        if (n_rows) {
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            int64_t* d = E.idx64.as<int64_t>(2 * n_rows);
            // up to 11 bytes per entry: 0xFF + u32 row escape and 0xFFFF + u32 column escape
            uint8_t* dout = E.body.as<uint8_t>(11 * n_rows + 16);
            uint64_t* misc = E.misc.as<uint64_t>(2);
            cuda_check(cudaMemsetAsync(misc, 0xFF, 8, E.stream), "memset");
            E.stager.h2d(d, rows, n_rows * 8, E.stream);
            E.stager.h2d(d + n_rows, cols, n_rows * 8, E.stream);
            launch_coo_pack(d, d + n_rows, n_rows, dout, misc + 1, misc, E.stream);
            uint64_t h[2];
            cuda_check(counted_copy(h, misc, 16, cudaMemcpyDeviceToHost, E.stream), "D2H");
            E.sync();
            if (h[0] != kNoError) {
                const uint32_t c = key_check(h[0]);
                if (c == kArgNegative) raise(PULSE_E_ARGUMENT, "coordinates must be non-negative");
                if (c == kArgOrder) raise(PULSE_E_ARGUMENT, "coordinates must be sorted row-major without duplicates");
                raise(PULSE_E_DIMENSION, c == kDimRow ? "row gap exceeds 32 bits" : "column entry exceeds 32 bits");
            }
            res->v.resize(h[1]);
            E.stager.d2h(res->v.data(), dout, h[1], E.stream);
        }
        *out = res.release();
    });
}

pulse_status pulse_upscale_coo(const uint8_t* data, uint64_t n, uint64_t count, int64_t* rows, int64_t* cols) {
    return guarded([&] {
        if (count == 0) {  // index_coding.hpp:154-156: nothing to read, anything left is trailing
            if (n) raise(PULSE_E_CORRUPT_STREAM, "downscaled payload has trailing bytes");
            return;
        }
        if (!data && n) raise(PULSE_E_ARGUMENT, "null argument");
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        // the general decoder's parallel parse of a one-entry table (decode.cu launch_coo_unpack_par)
        std::vector<pulse_tensor_geom> geom(1);
        geom[0].numel = count;
        geom[0].cols = 1;
        pulse_plan* plan = E.get_plan(geom, std::max<uint64_t>({count, n / 3 + 1, 1}));
        uint8_t* dp = E.body.as<uint8_t>(n + 64);
        int64_t* d = E.out64.as<int64_t>(2 * count + 2);
        if (n) E.stager.h2d(dp, data, n, E.stream);
        const pulse_patch_entry ent{0, 0, count, 0, n, n};
        auto* dent = E.entries.as<pulse_patch_entry>(1);
        cuda_check(counted_copy(dent, &ent, sizeof(ent), cudaMemcpyHostToDevice, E.stream), "H2D");
        auto* dres = E.result.as<pulse_result>(1);
        launch_coo_unpack_par(plan->dev, dp, dent, d, d + count, dres, E.stream);
        const pulse_result r = fetch_result(E, dres);
        if (r.status != PULSE_OK) raise(pulse_status(r.status), device_message(r, "", nullptr, PULSE_COO_DOWNSCALED));
        E.stager.d2h(rows, d, count * 8, E.stream);
        E.stager.d2h(cols, d + count, count * 8, E.stream);
        E.sync();
    });
}

// ---- compression.hpp ------------------------------------------------------------------------
pulse_status pulse_compress(const uint8_t* data, uint64_t n, uint32_t codec, pulse_bytes** out) {
    return guarded([&] {
        if (!out) raise(PULSE_E_ARGUMENT, "null argument");
        auto b = std::make_unique<pulse_bytes>();
        const auto z = codec_compress(data, n, codec);
        b->v.assign(z.begin(), z.end());
        *out = b.release();
    });
}
pulse_status pulse_decompress(const uint8_t* data, uint64_t n, uint32_t codec, pulse_bytes** out) {
    return guarded([&] {
        if (!out) raise(PULSE_E_ARGUMENT, "null argument");
        auto b = std::make_unique<pulse_bytes>();
        const auto z = codec_decompress(data, n, codec);
        b->v.assign(z.begin(), z.end());
        *out = b.release();
    });
}


// ---- container.hpp: the PULC checkpoint container ------------------------------------------
// Layout (container.hpp:52-57): "PULC", u32 1, u64 header length, JSON
// {"step", "tensors": [{"dtype", "name", "nbytes", "offset", "shape"}]} (nlohmann
// dump, keys sorted), then the LE bf16 payloads at 64-byte aligned offsets from
// the 64-byte aligned payload base.  On this little-endian host a payload IS the
// tensor's u16 array, so every payload moves as one copy -- a memcpy or a DMA
// straight to/from HBM -- instead of the reference's per-element u16le loop
// (container.hpp:88, :140).
pulse_status pulse_write_checkpoint_bytes(const pulse_checkpoint* c, int device_data, pulse_bytes** out) {
    return guarded([&] {
        if (!c || !out || (c->n_tensors && !c->tensors)) raise(PULSE_E_ARGUMENT, "null argument");
        validate_checkpoint(c);  // Checkpoint::validate, container.hpp:59
        const uint32_t T = c->n_tensors;
        nlohmann::json header;
        header["step"] = c->step;
        auto& table = header["tensors"] = nlohmann::json::array();
        std::vector<uint64_t> rel(T);
        uint64_t off = 0;
        for (uint32_t i = 0; i < T; ++i) {  // insertion order, not name order
            const pulse_tensor& t = c->tensors[i];
            const uint64_t nb = t.numel * 2;
            rel[i] = off;
            table.push_back({{"name", t.name},
                             {"dtype", "bf16"},
                             {"shape", std::vector<int64_t>(t.shape, t.shape + t.rank)},
                             {"offset", off},
                             {"nbytes", nb}});
            off = (off + nb + 63) & ~uint64_t(63);
        }
        const std::string js = header.dump();
        const uint64_t base = (16 + js.size() + 63) & ~uint64_t(63);
        uint64_t total = 16 + js.size();
        if (T) total = base + rel[T - 1] + c->tensors[T - 1].numel * 2;
        auto res = std::make_unique<pulse_bytes>();
        res->v.resize(total);
        uint8_t* w = res->v.data();
        std::memcpy(w, "PULC", 4);
        for (int i = 0; i < 4; ++i) w[4 + i] = uint8_t(1u >> (8 * i));
        for (int i = 0; i < 8; ++i) w[8 + i] = uint8_t(uint64_t(js.size()) >> (8 * i));
        std::memcpy(w + 16, js.data(), js.size());
        if (T) {
            // zero padding between the header / payloads (the reference's push_back(0) fill)
            std::memset(w + 16 + js.size(), 0, base - 16 - js.size());
            for (uint32_t i = 0; i + 1 < T; ++i) {
                const uint64_t e = base + rel[i] + c->tensors[i].numel * 2;
                std::memset(w + e, 0, base + rel[i + 1] - e);
            }
        }
        if (device_data && T) {
            for (uint32_t i = 0; i < T; ++i) {
                cudaPointerAttributes a{};
                if (cudaPointerGetAttributes(&a, c->tensors[i].data) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
                    cudaGetLastError();
                    raise(PULSE_E_ARGUMENT, std::string("tensor ") + c->tensors[i].name + ": data is not a device pointer");
                }
            }
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            for (uint32_t i = 0; i < T; ++i)
                E.stager.d2h(w + base + rel[i], c->tensors[i].data, c->tensors[i].numel * 2, E.stream);
        } else {
            pool().parallel_for(T, [&](size_t i) {
                if (c->tensors[i].numel) std::memcpy(w + base + rel[i], c->tensors[i].data, c->tensors[i].numel * 2);
            });
        }
        *out = res.release();
    });
}

}  // extern "C"

struct pulse_container {
    uint64_t step = 0;
    struct Entry {
        std::string name;
        std::vector<int64_t> shape;
        uint64_t numel = 0, begin = 0;
    };
    std::vector<Entry> tensors;
    uint64_t end = 0;  // the container's exact length
};

extern "C" {

pulse_status pulse_container_parse(const uint8_t* bytes, uint64_t n, pulse_container** out) {
    return guarded([&] {
        if (!out || (n && !bytes)) raise(PULSE_E_ARGUMENT, "null argument");
        // container.hpp:92-142, check for check
        if (n < 4) raise(PULSE_E_TRUNCATION, "container shorter than magic");
        if (std::memcmp(bytes, "PULC", 4) != 0) raise(PULSE_E_BAD_MAGIC, "not a checkpoint container (bad magic)");
        if (n < 8) raise(PULSE_E_TRUNCATION, "unexpected end of data");
        uint32_t version = 0;
        for (int i = 0; i < 4; ++i) version |= uint32_t(bytes[4 + i]) << (8 * i);
        if (version != 1) raise(PULSE_E_VERSION, "unsupported container version " + std::to_string(version));
        if (n < 16) raise(PULSE_E_TRUNCATION, "unexpected end of data");
        uint64_t hl = 0;
        for (int i = 0; i < 8; ++i) hl |= uint64_t(bytes[8 + i]) << (8 * i);
        if (hl > n - 16) raise(PULSE_E_TRUNCATION, "container header truncated");
        nlohmann::json header;
        try {
            header = nlohmann::json::parse(bytes + 16, bytes + 16 + hl);
        } catch (const nlohmann::json::exception& e) {
            raise(PULSE_E_FORMAT, std::string("container header is not valid JSON: ") + e.what());
        }
        auto c = std::make_unique<pulse_container>();
        c->end = 16 + hl;  // no payload: the file ends after the header
        try {
            c->step = header.at("step").get<uint64_t>();
            const uint64_t base = (16 + hl + 63) & ~uint64_t(63);
            for (const auto& e : header.at("tensors")) {
                pulse_container::Entry t;
                t.name = e.at("name").get<std::string>();
                if (e.at("dtype").get<std::string>() != "bf16") raise(PULSE_E_FORMAT, "unsupported dtype for tensor " + t.name);
                t.shape = e.at("shape").get<std::vector<int64_t>>();
                const uint64_t off = e.at("offset").get<uint64_t>();
                const uint64_t nb = e.at("nbytes").get<uint64_t>();
                if (off % 64) raise(PULSE_E_FORMAT, "misaligned tensor payload for " + t.name);
                t.numel = 1;
                for (int64_t x : t.shape) {
                    if (x <= 0) raise(PULSE_E_FORMAT, "non-positive extent in tensor " + t.name);
                    t.numel *= uint64_t(x);
                }
                if (nb != t.numel * 2) raise(PULSE_E_FORMAT, "payload length does not match shape for tensor " + t.name);
                t.begin = base + off;
                if (t.begin + nb > n) raise(PULSE_E_TRUNCATION, "tensor payload truncated for " + t.name);
                c->end = std::max(c->end, t.begin + nb);
                c->tensors.push_back(std::move(t));
            }
        } catch (const nlohmann::json::exception& e) {
            raise(PULSE_E_FORMAT, std::string("container header schema error: ") + e.what());
        }
        if (n != c->end) raise(PULSE_E_FORMAT, "container has trailing bytes");
        // Checkpoint::validate (checkpoint.hpp:54-70), as read_checkpoint_bytes ends with it
        std::unordered_map<std::string_view, int> seen;
        for (const auto& t : c->tensors) {
            if (t.name.empty()) raise(PULSE_E_ARGUMENT, "tensor with empty name");
            if (!seen.emplace(t.name, 0).second) raise(PULSE_E_ARGUMENT, "duplicate tensor name: " + t.name);
            if (t.shape.empty()) raise(PULSE_E_ARGUMENT, "tensor " + t.name + " has empty shape");
        }
        *out = c.release();
    });
}

void pulse_container_free(pulse_container* c) { delete c; }
uint64_t pulse_container_step(const pulse_container* c) { return c ? c->step : 0; }
uint32_t pulse_container_num_tensors(const pulse_container* c) { return c ? uint32_t(c->tensors.size()) : 0; }

pulse_status pulse_container_get_tensor(const pulse_container* c, uint32_t i, pulse_container_tensor* out) {
    if (!c || !out) return fail(PULSE_E_ARGUMENT, "null argument");
    if (i >= c->tensors.size()) return fail(PULSE_E_ARGUMENT, "tensor index out of range");
    const auto& t = c->tensors[i];
    *out = pulse_container_tensor{t.name.c_str(), t.shape.data(), uint32_t(t.shape.size()), t.numel, t.begin};
    return PULSE_OK;
}

pulse_status pulse_container_copy_out(const pulse_container* c, const uint8_t* data, uint64_t n, int device,
                                      void* const* dst) {
    return guarded([&] {
        if (!c || (!dst && !c->tensors.empty()) || (!data && c->end)) raise(PULSE_E_ARGUMENT, "null argument");
        if (n != c->end) raise(PULSE_E_ARGUMENT, "bytes are not the parsed container (length differs)");
        const size_t T = c->tensors.size();
        if (!device) {
            pool().parallel_for(T, [&](size_t i) {
                if (c->tensors[i].numel) std::memcpy(dst[i], data + c->tensors[i].begin, c->tensors[i].numel * 2);
            });
            return;
        }
        if (!T) return;
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        for (size_t i = 0; i < T; ++i)
            E.stager.h2d(dst[i], data + c->tensors[i].begin, c->tensors[i].numel * 2, E.stream);
        E.sync();
    });
}

}  // extern "C"

// =============================================================================================
// Resident checkpoints: the sync path on the device (sync.hpp:78-92, 166-211, 308-352)
// =============================================================================================
struct pulse_resident {
    int device = 0;
    pulse_plan* plan = nullptr;
    uint64_t cap = 0;
    uint64_t step = 0, last_anchor = 0;
    uint8_t hash[32] = {};
    std::vector<std::string> names;           // insertion order
    std::vector<std::vector<int64_t>> shapes;
    std::vector<uint64_t> numel;
    std::vector<uint32_t> order;              // plan (name-order) index -> insertion index
    std::vector<uint32_t> plan_of;            // insertion index -> plan index
    std::unordered_map<std::string, uint32_t> by_name;
    void* arena = nullptr;                    // resident weights; tensor i at element off[i]
    std::vector<uint64_t> off;
    DevBuf body, entries, result, idx64, backup, start, vals, carry;
    void* pinned[2] = {nullptr, nullptr};     // hash pipeline (D2H | SHA-256)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t hstream = nullptr;
    ~pulse_resident() {
        if (plan) pulse_plan_destroy(plan);
        if (arena) cudaFree(arena);
        for (int i = 0; i < 2; ++i) {
            if (pinned[i]) cudaFreeHost(pinned[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
        if (hstream) cudaStreamDestroy(hstream);
        for (DevBuf* b : {&body, &entries, &result, &idx64, &backup, &start, &vals, &carry})
            if (b->p) cudaFree(b->p);
    }
    uint16_t* tensor(uint32_t i) const { return static_cast<uint16_t*>(arena) + off[i]; }
};

namespace {

constexpr size_t kHashChunk = 64u << 20;

// Runs a resident's calls on the device it lives on, restoring the caller's device.
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// SHA-256 of device tensors in the given order (sha256.hpp:93-116 over HBM):
// chunk k+1 is copied to pinned memory while chunk k is hashed.
void hash_device(pulse_resident* r, const std::vector<std::pair<const uint8_t*, uint64_t>>& parts, uint8_t out[32]) {
    if (!r->hstream) {
        cuda_check(cudaStreamCreateWithFlags(&r->hstream, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < 2; ++i) {
            cuda_check(cudaHostAlloc(&r->pinned[i], kHashChunk, cudaHostAllocDefault), "pinned");
            cuda_check(cudaEventCreateWithFlags(&r->ev[i], cudaEventDisableTiming), "event");
        }
    }
    std::vector<std::pair<const uint8_t*, uint64_t>> pieces;
    for (auto [p, n] : parts)
        for (uint64_t o = 0; o < n; o += kHashChunk) pieces.emplace_back(p + o, std::min<uint64_t>(kHashChunk, n - o));
    EVP_MD_CTX* ctx = EVP_MD_CTX_new();
    if (!ctx || EVP_DigestInit_ex(ctx, EVP_sha256(), nullptr) != 1) raise(PULSE_E_ERROR, "failed to initialize SHA-256 context");
    auto issue = [&](size_t k) {
        const int b = int(k & 1);
        cuda_check(counted_copy(r->pinned[b], pieces[k].first, pieces[k].second, cudaMemcpyDeviceToHost, r->hstream), "D2H");
        cuda_check(cudaEventRecord(r->ev[b], r->hstream), "event");
    };
    if (!pieces.empty()) issue(0);
    for (size_t k = 0; k < pieces.size(); ++k) {
        if (k + 1 < pieces.size()) {
            // buffer (k+1)&1 was hashed in iteration k-1 (synchronously), so it is free
            issue(k + 1);
        }
        cuda_check(cudaEventSynchronize(r->ev[k & 1]), "D2H wait");
        if (EVP_DigestUpdate(ctx, r->pinned[k & 1], pieces[k].second) != 1) raise(PULSE_E_ERROR, "SHA-256 update failed");
    }
    unsigned int len = 0;
    if (EVP_DigestFinal_ex(ctx, out, &len) != 1 || len != 32) raise(PULSE_E_ERROR, "SHA-256 finalize failed");
    EVP_MD_CTX_free(ctx);
}

std::vector<std::pair<const uint8_t*, uint64_t>> name_order_parts(const pulse_resident* r,
                                                                  const std::vector<const void*>& ptrs) {
    std::vector<std::pair<const uint8_t*, uint64_t>> parts;
    for (uint32_t k = 0; k < r->order.size(); ++k) {
        const uint32_t i = r->order[k];
        parts.emplace_back(static_cast<const uint8_t*>(ptrs[i]), r->numel[i] * 2);
    }
    return parts;
}

// (Re)creates the plan with room for `cap` changes and binds the resident weights to slot 0.
void resident_plan(pulse_resident* r, Engine& E, uint64_t cap) {
    if (r->plan && cap <= r->cap) return;
    if (r->plan) {
        E.sync();
        pulse_plan_destroy(r->plan);
        r->plan = nullptr;
    }
    const uint32_t T = uint32_t(r->names.size());
    std::vector<pulse_tensor_geom> geom(T);
    std::vector<const void*> ptrs(T);
    for (uint32_t k = 0; k < T; ++k) {
        const uint32_t i = r->order[k];
        geom[k] = {r->numel[i], uint64_t(r->shapes[i].back())};
        ptrs[k] = r->tensor(i);
    }
    r->cap = std::max<uint64_t>(cap, 1024);
    if (pulse_plan_create(E.ctx, geom.data(), T, r->cap, &r->plan) != PULSE_OK)
        raise(PULSE_E_CUDA, std::string("plan: ") + pulse_last_error());
    if (pulse_plan_bind(r->plan, 0, ptrs.data()) != PULSE_OK) raise(PULSE_E_CUDA, pulse_last_error());
}

// apply_delta (sync.hpp:308-329) for an already parsed PULP.
void resident_apply_parsed(pulse_resident* r, Engine& E, ParsedPulp& pp, uint64_t step, const uint8_t* expected,
                           bool verify) {
    const pulse_patch* p = pp.p.get();
    // apply_delta's order: read_patch_bytes (which decodes every index payload against
    // the patch's own shapes) -> the step / hash protocol checks -> decode's tensor
    // checks (patch.hpp:314-324).  The payloads are decoded on the device during the
    // apply below, so when a host-side check is about to fail, the payloads are
    // decoded first and their error, if any, wins.
    Failure host_err{PULSE_OK, ""};
    if (p->base_step != int64_t(r->step))
        host_err = {PULSE_E_PROTOCOL, "delta at step " + std::to_string(step) + " does not base on the held step"};
    else if (p->target_step != int64_t(step))
        host_err = {PULSE_E_PROTOCOL, "patch steps disagree with the manifest"};
    else if (expected && std::memcmp(p->target_hash, expected, 32) != 0)
        host_err = {PULSE_E_PROTOCOL, "patch target hash disagrees with the manifest"};
    const uint32_t P = uint32_t(p->tensors.size());
    std::vector<pulse_patch_entry> ents(P);
    std::vector<uint32_t> target(P);
    uint64_t body_len = 0, n = 0;
    for (uint32_t k = 0; k < P && host_err.st == PULSE_OK; ++k) {
        const auto& tp = p->tensors[k];
        const auto it = r->by_name.find(tp.name);
        if (it == r->by_name.end()) {
            host_err = {PULSE_E_TENSOR_SET, "patch references unknown tensor '" + tp.name + "'"};
            break;
        }
        if (tp.shape != r->shapes[it->second]) {
            host_err = {PULSE_E_SHAPE_MISMATCH, "tensor '" + tp.name + "' shape differs between patch and checkpoint"};
            break;
        }
        const uint64_t cnt = tp.values.size();
        target[k] = r->plan_of[it->second];
        ents[k] = pulse_patch_entry{target[k], 0, cnt, body_len, pp.lens[k], body_len + pp.lens[k]};
        body_len += pp.lens[k] + 2 * cnt;
        n += cnt;
    }
    if (host_err.st != PULSE_OK) {
        device_decode_payloads(E, pp.p.get(), pp.pl, pp.lens);  // raises a payload error first
        raise(host_err.st, host_err.msg);
    }
    if (P == 0) {
        r->step = step;
        std::memcpy(r->hash, p->target_hash, 32);
        r->last_anchor = std::max<uint64_t>(r->last_anchor, uint64_t(p->anchor_step));
        return;
    }
    resident_plan(r, E, n);
    // the device body: [index payload][value payload] per tensor, as the kernels read it
    uint8_t* dbody = r->body.as<uint8_t>(body_len + 64);
    RawVec<uint8_t> host(body_len);
    pool().parallel_for(P, [&](size_t k) {
        if (pp.lens[k]) std::memcpy(host.data() + ents[k].idx_off, pp.pl[k], pp.lens[k]);
        const auto& v = p->tensors[k].values;
        if (!v.empty()) std::memcpy(host.data() + ents[k].val_off, v.data(), v.size() * 2);
    });
    E.stager.h2d(dbody, host.data(), body_len, E.stream);
    auto* dent = r->entries.as<pulse_patch_entry>(P);
    cuda_check(counted_copy(dent, ents.data(), P * sizeof(pulse_patch_entry), cudaMemcpyHostToDevice, E.stream), "H2D");
    auto* dres = r->result.as<pulse_result>(1);
    auto fail_on = [&](const pulse_result& res) {
        if (res.status == PULSE_OK) return;
        const std::string nm = res.err_tensor < P ? p->tensors[res.err_tensor].name : "?";
        raise(pulse_status(res.status), device_message(res, nm, nullptr, p->representation));
    };
    int64_t* didx = nullptr;
    uint16_t* dbak = nullptr;
    uint64_t* dstart = nullptr;
    // duplicate tensor names: decode (validates everything), then scatter the decoded
    // indices run by run in patch order so the last entry for a tensor wins (patch.hpp:313-339)
    const auto runs = distinct_target_runs(target.data(), P);
    const bool in_runs = runs.size() > 2;
    std::vector<uint64_t> at(P + 1, 0);
    for (uint32_t k = 0; k < P; ++k) at[k + 1] = at[k] + ents[k].count;
    uint16_t* dvals = nullptr;
    if (verify || in_runs) {  // indices (and, for verify, the values the scatter overwrites)
        didx = r->idx64.as<int64_t>(n);
        // one decode per run (a launch takes at most one entry per tensor); FLAT_INT32's gap
        // stream continues into the next run through the carry: the global position of the
        // last decoded index, rebased past the numel of every entry since (patch.hpp:185-259)
        auto* dcarry = r->carry.as<pulse_flat_carry>(1);
        bool have_last = false;
        uint64_t since_last = 0;  // numel of entries from the last decoded index's entry onward
        int64_t last_idx = 0;
        for (size_t q = 0; q + 1 < runs.size(); ++q) {
            const uint32_t k0 = runs[q], k1 = runs[q + 1];
            const pulse_flat_carry* cp = nullptr;
            if (p->representation == PULSE_FLAT_INT32 && have_last) {
                const pulse_flat_carry c{1, since_last - uint64_t(last_idx)};
                cuda_check(counted_copy(dcarry, &c, sizeof(c), cudaMemcpyHostToDevice, E.stream), "H2D");
                cp = dcarry;
            }
            if (pulse_decode_indices(r->plan, p->representation, dbody, dent + k0, k1 - k0, cp, didx + at[k0], dres,
                                     E.stream) != PULSE_OK)
                raise(PULSE_E_CUDA, pulse_last_error());
            pulse_result res = fetch_result(E, dres);
            if (res.status != PULSE_OK) res.err_tensor += k0;
            fail_on(res);
            if (p->representation == PULSE_FLAT_INT32 && in_runs)
                for (uint32_t k = k0; k < k1; ++k) {
                    const uint64_t numel_k = r->numel[r->order[ents[k].tensor]];
                    if (ents[k].count) {
                        cuda_check(counted_copy(&last_idx, didx + at[k + 1] - 1, 8, cudaMemcpyDeviceToHost, E.stream),
                                   "D2H");
                        E.sync();
                        have_last = true;
                        since_last = 0;
                    }
                    since_last += numel_k;
                }
        }
        if (verify) {
            dstart = r->start.as<uint64_t>(P + 1);
            cuda_check(counted_copy(dstart, at.data(), (P + 1) * 8, cudaMemcpyHostToDevice, E.stream), "H2D");
            dbak = r->backup.as<uint16_t>(n);
            launch_gather_values(r->plan->dev, 0, dent, dstart, P, didx, dbak, E.stream);
        }
    }
    if (!in_runs) {
        if (pulse_apply(r->plan, 0, p->representation, dbody, dent, P, nullptr, dres, E.stream) != PULSE_OK)
            raise(PULSE_E_CUDA, pulse_last_error());
        fail_on(fetch_result(E, dres));  // validate-then-scatter: a failure wrote nothing
    } else {
        // values contiguous in patch order, next to the decoded indices
        RawVec<uint16_t> hv(std::max<uint64_t>(n, 1));
        for (uint32_t k = 0; k < P; ++k)
            if (ents[k].count) std::memcpy(hv.data() + at[k], p->tensors[k].values.data(), ents[k].count * 2);
        dvals = r->vals.as<uint16_t>(n);
        E.stager.h2d(dvals, hv.data(), n * 2, E.stream);
        for (size_t q = 0; q + 1 < runs.size(); ++q) {
            const uint32_t k0 = runs[q], k1 = runs[q + 1];
            launch_apply_idx64(r->plan->dev, didx + at[k0], dvals + at[k0], dent + k0, k1 - k0, 0, dres, E.stream);
            fail_on(fetch_result(E, dres));
        }
    }
    if (verify) {  // patch.hpp:341-346 on the resident weights
        std::vector<const void*> ptrs(r->names.size());
        for (uint32_t i = 0; i < ptrs.size(); ++i) ptrs[i] = r->tensor(i);
        uint8_t h[32];
        hash_device(r, name_order_parts(r, ptrs), h);
        if (std::memcmp(h, p->target_hash, 32) != 0) {
            for (size_t q = 0; q + 1 < runs.size(); ++q) {  // put the old values back
                const uint32_t k0 = runs[q], k1 = runs[q + 1];
                launch_apply_idx64(r->plan->dev, didx + at[k0], dbak + at[k0], dent + k0, k1 - k0, 0, dres, E.stream);
                fail_on(fetch_result(E, dres));
            }
            raise(PULSE_E_HASH_MISMATCH, "hash mismatch: expected " + hex(p->target_hash) + ", actual " + hex(h));
        }
    }
    r->step = step;
    std::memcpy(r->hash, p->target_hash, 32);
    r->last_anchor = std::max<uint64_t>(r->last_anchor, uint64_t(p->anchor_step));
}

}  // namespace

extern "C" {

pulse_status pulse_resident_create(const pulse_checkpoint* c, uint64_t max_changes, pulse_resident** out) {
    return guarded([&] {
        if (!c || !out) raise(PULSE_E_ARGUMENT, "null argument");
        validate_checkpoint(c);
        auto r = std::make_unique<pulse_resident>();
        const uint32_t T = c->n_tensors;
        r->step = c->step;
        r->order = sorted_order(c);
        r->plan_of.assign(T, 0);
        for (uint32_t k = 0; k < T; ++k) r->plan_of[r->order[k]] = k;
        for (uint32_t i = 0; i < T; ++i) {
            const pulse_tensor& t = c->tensors[i];
            r->names.emplace_back(t.name);
            r->shapes.emplace_back(t.shape, t.shape + t.rank);
            r->numel.push_back(t.numel);
            r->by_name[t.name] = i;
        }
        uint64_t total = 0;
        r->off = arena_offsets(r->numel, total);
        // the hash of the held checkpoint (checkpoint_to_state), overlapping the upload
        auto hash = std::async(std::launch::async, [&] { hash_checkpoint(c, r->hash); });
        // the caller's pending writes to these buffers (any stream, e.g. an async
        // optimizer step) land before the copy reads them
        cuda_check(cudaDeviceSynchronize(), "wait for pending device work");
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        cudaGetDevice(&r->device);
        cuda_check(cudaMalloc(&r->arena, std::max<uint64_t>(total, 8) * 2), "resident weights");
        for (uint32_t i = 0; i < T; ++i) E.stager.h2d(r->tensor(i), c->tensors[i].data, r->numel[i] * 2, E.stream);
        if (T) resident_plan(r.get(), E, max_changes);
        E.sync();
        hash.get();
        *out = r.release();
    });
}

pulse_status pulse_resident_create_device(const pulse_checkpoint* c, uint64_t max_changes, pulse_resident** out) {
    return guarded([&] {
        if (!c || !out) raise(PULSE_E_ARGUMENT, "null argument");
        validate_checkpoint(c);
        const uint32_t T = c->n_tensors;
        for (uint32_t i = 0; i < T; ++i) {
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, c->tensors[i].data) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
                cudaGetLastError();
                raise(PULSE_E_ARGUMENT, std::string("tensor ") + c->tensors[i].name + ": data is not a device pointer");
            }
        }
        auto r = std::make_unique<pulse_resident>();
        r->step = c->step;
        r->order = sorted_order(c);
        r->plan_of.assign(T, 0);
        for (uint32_t k = 0; k < T; ++k) r->plan_of[r->order[k]] = k;
        for (uint32_t i = 0; i < T; ++i) {
            const pulse_tensor& t = c->tensors[i];
            r->names.emplace_back(t.name);
            r->shapes.emplace_back(t.shape, t.shape + t.rank);
            r->numel.push_back(t.numel);
            r->by_name[t.name] = i;
        }
        uint64_t total = 0;
        r->off = arena_offsets(r->numel, total);
        // the caller's pending writes to these buffers (any stream, e.g. an async
        // optimizer step) land before the copy reads them
        cuda_check(cudaDeviceSynchronize(), "wait for pending device work");
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        cudaGetDevice(&r->device);
        cuda_check(cudaMalloc(&r->arena, std::max<uint64_t>(total, 8) * 2), "resident weights");
        for (uint32_t i = 0; i < T; ++i)
            cuda_check(cudaMemcpyAsync(r->tensor(i), c->tensors[i].data, r->numel[i] * 2, cudaMemcpyDeviceToDevice,
                                       E.stream), "D2D");
        if (T) resident_plan(r.get(), E, max_changes);
        E.sync();
        std::vector<const void*> ptrs(T);
        for (uint32_t i = 0; i < T; ++i) ptrs[i] = r->tensor(i);
        hash_device(r.get(), name_order_parts(r.get(), ptrs), r->hash);
        *out = r.release();
    });
}

void pulse_resident_destroy(pulse_resident* r) {
    if (!r) return;
    DeviceGuard dg(r->device);
    cudaDeviceSynchronize();
    delete r;
}
uint64_t pulse_resident_step(const pulse_resident* r) { return r ? r->step : 0; }
uint64_t pulse_resident_last_anchor_step(const pulse_resident* r) { return r ? r->last_anchor : 0; }
pulse_status pulse_resident_hash(const pulse_resident* r, uint8_t* out32) {
    if (!r || !out32) return fail(PULSE_E_ARGUMENT, "null argument");
    std::memcpy(out32, r->hash, 32);
    return PULSE_OK;
}
uint32_t pulse_resident_num_tensors(const pulse_resident* r) { return r ? uint32_t(r->names.size()) : 0; }
pulse_status pulse_resident_tensor(const pulse_resident* r, uint32_t i, void** dev_ptr) {
    if (!r || !dev_ptr) return fail(PULSE_E_ARGUMENT, "null argument");
    if (i >= r->names.size()) return fail(PULSE_E_ARGUMENT, "tensor index out of range");
    *dev_ptr = r->tensor(i);
    return PULSE_OK;
}

pulse_status pulse_resident_download(const pulse_resident* r, uint16_t* const* out) {
    return guarded([&] {
        if (!r || (!out && !r->names.empty())) raise(PULSE_E_ARGUMENT, "null argument");
        DeviceGuard dg(r->device);
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        for (uint32_t i = 0; i < r->names.size(); ++i) E.stager.d2h(out[i], r->tensor(i), r->numel[i] * 2, E.stream);
        E.sync();
    });
}

pulse_status pulse_resident_apply(pulse_resident* r, const uint8_t* pulp, uint64_t n, uint64_t step,
                                  const uint8_t* expected_hash32, int verify_hash) {
    return guarded([&] {
        if (!r || (n && !pulp)) raise(PULSE_E_ARGUMENT, "null argument");
        DeviceGuard dg(r->device);
        ParsedPulp pp = parse_pulp(pulp, n);
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        resident_apply_parsed(r, E, pp, step, expected_hash32, verify_hash != 0);
    });
}

pulse_status pulse_resident_walk(pulse_resident* r, const uint8_t* const* pulps, const uint64_t* sizes, uint32_t k,
                                 int verify_hash, uint32_t* applied) {
    if (applied) *applied = 0;
    return guarded([&] {
        if (!r || (k && (!pulps || !sizes))) raise(PULSE_E_ARGUMENT, "null argument");
        if (k == 0) return;
        DeviceGuard dg(r->device);
        // the next patch is parsed (JSON header, codec) on a host thread while this one applies
        std::future<ParsedPulp> next = std::async(std::launch::async, [&] { return parse_pulp(pulps[0], sizes[0]); });
        for (uint32_t j = 0; j < k; ++j) {
            ParsedPulp pp = next.get();
            if (j + 1 < k) next = std::async(std::launch::async, [&, j] { return parse_pulp(pulps[j + 1], sizes[j + 1]); });
            struct Drain {  // never leave a parse running on a failure
                std::future<ParsedPulp>& f;
                ~Drain() {
                    if (f.valid()) f.wait();
                }
            } drain{next};
            Engine& E = engine();
            std::lock_guard<std::mutex> lk(E.mu);
            resident_apply_parsed(r, E, pp, r->step + 1, nullptr, verify_hash != 0);
            if (applied) *applied = j + 1;
        }
    });
}

pulse_status pulse_resident_publish(pulse_resident* r, const void* const* dev_current, uint64_t step,
                                    uint32_t repr, uint32_t codec, uint64_t anchor_step, int advance,
                                    pulse_bytes** out_pulp, uint8_t* out_hash32) {
    return guarded([&] {
        if (!r || !out_pulp || (!dev_current && !r->names.empty())) raise(PULSE_E_ARGUMENT, "null argument");
        if (step != r->step + 1) raise(PULSE_E_ARGUMENT, "publish requires consecutive steps");
        DeviceGuard dg(r->device);
        repr_name(repr);
        if (codec > PULSE_GZIP6) raise(PULSE_E_ARGUMENT, "unknown codec");
        const uint32_t T = uint32_t(r->names.size());
        std::vector<const void*> cur(dev_current, dev_current + T);
        for (uint32_t i = 0; i < T; ++i) {
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, cur[i]) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
                cudaGetLastError();
                raise(PULSE_E_ARGUMENT, "tensor " + r->names[i] + ": current data is not a device pointer");
            }
        }
        // order the encode and the hash after the caller's pending writes to `dev_current`
        // on any stream: nothing below may read a half-written snapshot
        cuda_check(cudaDeviceSynchronize(), "wait for pending device work");
        Engine& E = engine();
        std::lock_guard<std::mutex> lk(E.mu);
        uint8_t target_hash[32] = {};
        // the target hash once, from HBM, on a host thread while the device encodes
        std::future<void> hash;
        if (T)
            hash = std::async(std::launch::async, [&] {
                cudaSetDevice(r->device);
                hash_device(r, name_order_parts(r, cur), target_hash);
            });
        struct Join {
            std::future<void>& f;
            ~Join() {
                if (f.valid()) f.wait();
            }
        } join{hash};
        RawVec<uint8_t> body;
        std::vector<pulse_patch_entry> ents;
        std::vector<PulpTensorRef> refs;
        uint8_t* dbody = nullptr;
        pulse_patch_entry* dent = nullptr;
        if (T) {
            std::vector<const void*> planp(T);
            for (uint32_t k = 0; k < T; ++k) planp[k] = cur[r->order[k]];
            resident_plan(r, E, r->cap);
            pulse_scan_summary sm{};
            for (int attempt = 0; attempt < 2; ++attempt) {
                if (pulse_plan_bind(r->plan, 1, planp.data()) != PULSE_OK) raise(PULSE_E_CUDA, pulse_last_error());
                if (pulse_encode_scan(r->plan, 1, 0, nullptr, E.stream) != PULSE_OK) raise(PULSE_E_CUDA, pulse_last_error());
                cuda_check(counted_copy(&sm, r->plan->dev.scan, sizeof(sm), cudaMemcpyDeviceToHost, E.stream), "D2H");
                E.sync();
                if (sm.status != PULSE_E_CAPACITY) break;
                resident_plan(r, E, sm.n_changes + sm.n_changes / 16 + 1024);
            }
            auto* dres = r->result.as<pulse_result>(1);
            dent = r->entries.as<pulse_patch_entry>(T);
            uint64_t cap = 14 * sm.n_changes + 1024;  // >= any escape-coded body (<= 11 + 2 bytes per change)
            pulse_result res{};
            for (int attempt = 0; attempt < 2; ++attempt) {
                dbody = r->body.as<uint8_t>(cap + 64);
                if (pulse_encode_emit(r->plan, repr, nullptr, 1, 0, dbody, cap, dent, dres, E.stream) != PULSE_OK)
                    raise(PULSE_E_CUDA, pulse_last_error());
                res = fetch_result(E, dres);
                if (res.status != PULSE_E_CAPACITY) break;
                cap = res.required + 1024;
            }
            if (res.status != PULSE_OK) {
                const std::string nm = res.err_tensor < T ? r->names[r->order[res.err_tensor]] : "?";
                raise(pulse_status(res.status), device_message(res, nm, nullptr));
            }
            ents.resize(res.n_entries);
            if (res.n_entries)
                cuda_check(counted_copy(ents.data(), dent, res.n_entries * sizeof(pulse_patch_entry),
                                        cudaMemcpyDeviceToHost, E.stream), "D2H");
            body.resize(res.body_bytes);
            E.stager.d2h(body.data(), dbody, res.body_bytes, E.stream);
            E.sync();
        }
        // codec per tensor blob on the thread pool (identity: straight out of the body)
        const size_t P = ents.size();
        std::vector<std::vector<uint8_t>> ib(P), vb(P);
        refs.resize(P);
        pool().parallel_for(P, [&](size_t k) {
            const auto& e = ents[k];
            const uint32_t i = r->order[e.tensor];
            const uint8_t* ip = body.data() + e.idx_off;
            const uint8_t* vp = body.data() + e.val_off;
            uint64_t in = e.idx_nbytes, vn = e.count * 2;
            if (codec != PULSE_IDENTITY) {
                ib[k] = codec_compress(ip, in, codec);
                vb[k] = codec_compress(vp, vn, codec);
                ip = ib[k].data();
                in = ib[k].size();
                vp = vb[k].data();
                vn = vb[k].size();
            }
            refs[k] = {&r->names[i], &r->shapes[i], e.count, ip, in, vp, vn};
        });
        if (hash.valid()) hash.get();
        if (!T) hash_tensors({}, target_hash);  // SHA-256 of nothing
        auto res = assemble_pulp(int64_t(anchor_step), int64_t(r->step), int64_t(step), target_hash, codec, repr, refs);
        if (advance) {  // the held weights become the published snapshot: the patch, applied in place
            if (P) {
                auto* dres = r->result.as<pulse_result>(1);
                if (pulse_apply(r->plan, 0, repr, dbody, dent, uint32_t(P), nullptr, dres, E.stream) != PULSE_OK)
                    raise(PULSE_E_CUDA, pulse_last_error());
                const pulse_result ar = fetch_result(E, dres);
                if (ar.status != PULSE_OK) raise(pulse_status(ar.status), "self-apply of the published patch failed");
            }
            r->step = step;
            std::memcpy(r->hash, target_hash, 32);
        }
        if (out_hash32) std::memcpy(out_hash32, target_hash, 32);
        *out_pulp = res.release();
    });
}

}  // extern "C"
