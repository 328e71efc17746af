// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A C-callable shim over the *unmodified* reference headers in
// /root/reference/proj/include (arxiv 2602.03839, PULSE).  It is compiled by
// oracle/Makefile into oracle/_ref/libpulse_ref.so (git-ignored; it travels to
// the GPU box as a prebuilt binary).  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg, --impl reference) may load it.
//
// Every entry point forwards to the reference function named in its comment;
// nothing here re-implements reference behaviour.  Errors are caught and
// mapped to the same status numbering as include/pulse_cuda.h.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pulse/absorption.hpp"
#include "pulse/compression.hpp"
#include "pulse/container.hpp"
#include "pulse/index_coding.hpp"
#include "pulse/metrics.hpp"
#include "pulse/patch.hpp"
#include "pulse/patch_file.hpp"
#include "pulse/sha256.hpp"
#include "pulse/synthetic.hpp"

namespace {

thread_local std::string g_err;

// Same numbering as pulse_status in include/pulse_cuda.h.
int map_exception() {
    try {
        throw;
    } catch (const pulse::BadMagicError& e) {
        g_err = e.what(); return 4;
    } catch (const pulse::VersionError& e) {
        g_err = e.what(); return 5;
    } catch (const pulse::TruncationError& e) {
        g_err = e.what(); return 6;
    } catch (const pulse::CorruptStreamError& e) {
        g_err = e.what(); return 7;
    } catch (const pulse::FormatError& e) {
        g_err = e.what(); return 3;
    } catch (const pulse::ShapeMismatchError& e) {
        g_err = e.what(); return 9;
    } catch (const pulse::TensorSetError& e) {
        g_err = e.what(); return 10;
    } catch (const pulse::IndexRangeError& e) {
        g_err = e.what(); return 11;
    } catch (const pulse::DimensionError& e) {
        g_err = e.what(); return 12;
    } catch (const pulse::ModelMismatchError& e) {
        g_err = e.what(); return 8;
    } catch (const pulse::HashMismatchError& e) {
        g_err = e.what(); return 13;
    } catch (const pulse::ArgumentError& e) {
        g_err = e.what(); return 2;
    } catch (const pulse::Error& e) {
        g_err = e.what(); return 1;
    } catch (const std::exception& e) {
        g_err = e.what(); return 1;
    }
}

#define SHIM_TRY try {
#define SHIM_CATCH \
    }              \
    catch (...) { return map_exception(); }

struct Buf {
    pulse::Bytes bytes;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- checkpoints -----------------------------------------------------------
void* ref_ckpt_new(uint64_t step) {
    auto* c = new pulse::Checkpoint();
    c->step = step;
    return c;
}
void ref_ckpt_free(void* h) { delete static_cast<pulse::Checkpoint*>(h); }
void ref_ckpt_add(void* h, const char* name, const int64_t* shape, uint32_t rank,
                  const uint16_t* data, uint64_t numel) {
    pulse::TensorRecord t;
    t.name = name;
    t.shape.assign(shape, shape + rank);
    t.data.resize(numel);
    if (numel) std::memcpy(t.data.data(), data, numel * 2);
    static_cast<pulse::Checkpoint*>(h)->tensors.push_back(std::move(t));
}
uint64_t ref_ckpt_step(void* h) { return static_cast<pulse::Checkpoint*>(h)->step; }
uint32_t ref_ckpt_num_tensors(void* h) {
    return static_cast<uint32_t>(static_cast<pulse::Checkpoint*>(h)->tensors.size());
}
void ref_ckpt_tensor(void* h, uint32_t i, const char** name, const int64_t** shape,
                     uint32_t* rank, const uint16_t** data, uint64_t* numel) {
    const auto& t = static_cast<pulse::Checkpoint*>(h)->tensors[i];
    *name = t.name.c_str();
    *shape = t.shape.data();
    *rank = static_cast<uint32_t>(t.shape.size());
    *data = reinterpret_cast<const uint16_t*>(t.data.data());
    *numel = t.data.size();
}

// synthetic.hpp:111-115 generate_synthetic
int ref_generate_synthetic(const int64_t* shapes_flat, const uint32_t* ranks, uint32_t n_shapes,
                           double sparsity, int64_t cluster_width, uint64_t seed, void** prev,
                           void** curr) {
    SHIM_TRY
    pulse::SyntheticSpec spec;
    size_t off = 0;
    for (uint32_t i = 0; i < n_shapes; ++i) {
        spec.shapes.emplace_back(shapes_flat + off, shapes_flat + off + ranks[i]);
        off += ranks[i];
    }
    spec.sparsity = sparsity;
    spec.cluster_width = cluster_width;
    spec.seed = seed;
    auto pair = pulse::generate_synthetic(spec);
    *prev = new pulse::Checkpoint(std::move(pair.first));
    *curr = new pulse::Checkpoint(std::move(pair.second));
    return 0;
    SHIM_CATCH
}

// synthetic.hpp:62-107 mutate_checkpoint
int ref_mutate(void* base, double sparsity, int64_t cluster_width, uint64_t seed,
               uint64_t new_step, void** out) {
    SHIM_TRY
    *out = new pulse::Checkpoint(pulse::mutate_checkpoint(*static_cast<pulse::Checkpoint*>(base),
                                                          sparsity, cluster_width, seed,
                                                          new_step));
    return 0;
    SHIM_CATCH
}

// bf16.hpp:30-67
uint16_t ref_round_to_bf16(double x) { return pulse::round_to_bf16(x).bits; }

// sha256.hpp:93-116
int ref_hash_weights(void* h, uint8_t* out32) {
    SHIM_TRY
    auto d = pulse::hash_weights(*static_cast<pulse::Checkpoint*>(h));
    std::memcpy(out32, d.bytes.data(), 32);
    return 0;
    SHIM_CATCH
}

// sha256.hpp:51-87
void ref_sha256(const uint8_t* data, uint64_t n, uint8_t* out32) {
    auto d = pulse::Sha256::digest(std::span<const uint8_t>(data, n));
    std::memcpy(out32, d.bytes.data(), 32);
}

// ---- patches -----------------------------------------------------------------
void ref_patch_free(void* p) { delete static_cast<pulse::SparsePatch*>(p); }
void* ref_patch_new() { return new pulse::SparsePatch(); }
void ref_patch_header(void* p, int64_t* steps3, uint32_t* repr, uint32_t* codec, uint8_t* hash32) {
    auto* sp = static_cast<pulse::SparsePatch*>(p);
    steps3[0] = sp->base_step;
    steps3[1] = sp->target_step;
    steps3[2] = sp->anchor_step;
    *repr = static_cast<uint32_t>(sp->representation);
    *codec = static_cast<uint32_t>(sp->codec);
    std::memcpy(hash32, sp->target_hash.bytes.data(), 32);
}
void ref_patch_set_header(void* p, const int64_t* steps3, uint32_t repr, uint32_t codec,
                          const uint8_t* hash32) {
    auto* sp = static_cast<pulse::SparsePatch*>(p);
    sp->base_step = steps3[0];
    sp->target_step = steps3[1];
    sp->anchor_step = steps3[2];
    sp->representation = static_cast<pulse::SparseRepresentation>(repr);
    sp->codec = static_cast<pulse::CodecId>(codec);
    std::memcpy(sp->target_hash.bytes.data(), hash32, 32);
}
uint32_t ref_patch_num_tensors(void* p) {
    return static_cast<uint32_t>(static_cast<pulse::SparsePatch*>(p)->tensors.size());
}
void ref_patch_tensor(void* p, uint32_t i, const char** name, const int64_t** shape,
                      uint32_t* rank, const int64_t** indices, uint64_t* n_indices,
                      const uint16_t** values, uint64_t* n_values) {
    const auto& tp = static_cast<pulse::SparsePatch*>(p)->tensors[i];
    *name = tp.name.c_str();
    *shape = tp.shape.data();
    *rank = static_cast<uint32_t>(tp.shape.size());
    *indices = tp.indices.data();
    *n_indices = tp.indices.size();
    *values = reinterpret_cast<const uint16_t*>(tp.values.data());
    *n_values = tp.values.size();
}
void ref_patch_add_tensor(void* p, const char* name, const int64_t* shape, uint32_t rank,
                          const int64_t* indices, uint64_t n_indices, const uint16_t* values,
                          uint64_t n_values) {
    pulse::TensorPatch tp;
    tp.name = name;
    tp.shape.assign(shape, shape + rank);
    tp.indices.assign(indices, indices + n_indices);
    tp.values.resize(n_values);
    if (n_values) std::memcpy(tp.values.data(), values, n_values * 2);
    static_cast<pulse::SparsePatch*>(p)->tensors.push_back(std::move(tp));
}

// patch.hpp:264-307
int ref_encode(void* cur, void* prev, uint32_t repr, uint32_t codec, void** out) {
    SHIM_TRY
    *out = new pulse::SparsePatch(pulse::encode(*static_cast<pulse::Checkpoint*>(cur),
                                                *static_cast<pulse::Checkpoint*>(prev),
                                                static_cast<pulse::SparseRepresentation>(repr),
                                                static_cast<pulse::CodecId>(codec)));
    return 0;
    SHIM_CATCH
}

// patch.hpp:309-348
int ref_decode(void* prev, void* patch, int verify, void** out) {
    SHIM_TRY
    *out = new pulse::Checkpoint(pulse::decode(*static_cast<pulse::Checkpoint*>(prev),
                                               *static_cast<pulse::SparsePatch*>(patch),
                                               verify != 0));
    return 0;
    SHIM_CATCH
}

// ---- byte buffers --------------------------------------------------------------
void ref_buf_free(void* b) { delete static_cast<Buf*>(b); }
const uint8_t* ref_buf_data(void* b) { return static_cast<Buf*>(b)->bytes.data(); }
uint64_t ref_buf_size(void* b) { return static_cast<Buf*>(b)->bytes.size(); }

// patch_file.hpp:30-83
int ref_write_patch_bytes(void* patch, void** out) {
    SHIM_TRY
    auto* b = new Buf();
    b->bytes = pulse::write_patch_bytes(*static_cast<pulse::SparsePatch*>(patch));
    *out = b;
    return 0;
    SHIM_CATCH
}

// patch_file.hpp:85-147
int ref_read_patch_bytes(const uint8_t* data, uint64_t n, void** out) {
    SHIM_TRY
    *out = new pulse::SparsePatch(pulse::read_patch_bytes(std::span<const uint8_t>(data, n)));
    return 0;
    SHIM_CATCH
}

// patch.hpp:116-174 -- returns the concatenation of all payloads and their sizes.
int ref_encode_index_payloads(void* patch, void** out, uint64_t* sizes) {
    SHIM_TRY
    auto payloads = pulse::encode_index_payloads(*static_cast<pulse::SparsePatch*>(patch));
    auto* b = new Buf();
    for (size_t i = 0; i < payloads.size(); ++i) {
        sizes[i] = payloads[i].size();
        b->bytes.insert(b->bytes.end(), payloads[i].begin(), payloads[i].end());
    }
    *out = b;
    return 0;
    SHIM_CATCH
}

// patch.hpp:178-262 -- payloads given as one concatenation plus per-tensor sizes.
int ref_decode_index_payloads(void* patch, const uint8_t* concat, const uint64_t* sizes) {
    SHIM_TRY
    auto* sp = static_cast<pulse::SparsePatch*>(patch);
    std::vector<pulse::Bytes> payloads;
    uint64_t off = 0;
    for (size_t i = 0; i < sp->tensors.size(); ++i) {
        payloads.emplace_back(concat + off, concat + off + sizes[i]);
        off += sizes[i];
    }
    pulse::decode_index_payloads(*sp, payloads);
    return 0;
    SHIM_CATCH
}

// index_coding.hpp:108-128
int ref_downscale_coo(const int64_t* rows, uint64_t n_rows, const int64_t* cols, uint64_t n_cols,
                      void** out) {
    SHIM_TRY
    auto* b = new Buf();
    b->bytes = pulse::downscale_coo(std::span<const int64_t>(rows, n_rows),
                                    std::span<const int64_t>(cols, n_cols));
    *out = b;
    return 0;
    SHIM_CATCH
}

// index_coding.hpp:130-158
int ref_upscale_coo(const uint8_t* data, uint64_t n, uint64_t count, int64_t* rows,
                    int64_t* cols) {
    SHIM_TRY
    auto c = pulse::upscale_coo(std::span<const uint8_t>(data, n), count);
    std::memcpy(rows, c.rows.data(), count * 8);
    std::memcpy(cols, c.cols.data(), count * 8);
    return 0;
    SHIM_CATCH
}

// index_coding.hpp:14-50
int ref_delta_encode(const int64_t* in, uint64_t n, int64_t* out) {
    SHIM_TRY
    auto g = pulse::delta_encode_indices(std::span<const int64_t>(in, n));
    if (n) std::memcpy(out, g.data(), n * 8);
    return 0;
    SHIM_CATCH
}
int ref_delta_decode(const int64_t* in, uint64_t n, int64_t* out) {
    SHIM_TRY
    auto g = pulse::delta_decode_indices(std::span<const int64_t>(in, n));
    if (n) std::memcpy(out, g.data(), n * 8);
    return 0;
    SHIM_CATCH
}

// compression.hpp:119-204
int ref_compress(const uint8_t* data, uint64_t n, uint32_t codec, void** out) {
    SHIM_TRY
    auto* b = new Buf();
    b->bytes = pulse::compress(std::span<const uint8_t>(data, n), static_cast<pulse::CodecId>(codec));
    *out = b;
    return 0;
    SHIM_CATCH
}
int ref_decompress(const uint8_t* data, uint64_t n, uint32_t codec, void** out) {
    SHIM_TRY
    auto* b = new Buf();
    b->bytes =
        pulse::decompress(std::span<const uint8_t>(data, n), static_cast<pulse::CodecId>(codec));
    *out = b;
    return 0;
    SHIM_CATCH
}

// container.hpp:58-92 (used by the acceptance-style byte-identity checks)
int ref_write_checkpoint_bytes(void* h, void** out) {
    SHIM_TRY
    auto* b = new Buf();
    b->bytes = pulse::write_checkpoint_bytes(*static_cast<pulse::Checkpoint*>(h));
    *out = b;
    return 0;
    SHIM_CATCH
}

// container.hpp:92-142
int ref_read_checkpoint_bytes(const uint8_t* data, uint64_t n, void** out) {
    SHIM_TRY
    *out = new pulse::Checkpoint(pulse::read_checkpoint_bytes(std::span<const uint8_t>(data, n)));
    return 0;
    SHIM_CATCH
}

// absorption.hpp:55-78
int ref_sparsity(void* cur, void* prev, uint64_t* changed, uint64_t* total) {
    SHIM_TRY
    auto r = pulse::sparsity(*static_cast<pulse::Checkpoint*>(cur),
                             *static_cast<pulse::Checkpoint*>(prev));
    *changed = r.changed;
    *total = r.total;
    return 0;
    SHIM_CATCH
}

// absorption.hpp:38-46
int ref_frozen_fraction(void* ck, double threshold, double* out) {
    SHIM_TRY
    *out = pulse::frozen_fraction(*static_cast<pulse::Checkpoint*>(ck), threshold);
    return 0;
    SHIM_CATCH
}

// ---- CPU baseline timing (reference path, single thread as the reference runs) ----
// One "step" of the reference hot path on (prev, curr):
//   encode (patch.hpp:264, includes hash_weights) -> write_patch_bytes
//   -> read_patch_bytes -> decode(verify=false)
// Each stage's wall time is returned (steady_clock, as metrics.hpp:30-32 does).
int ref_time_step(void* prev, void* curr, uint32_t repr, uint32_t codec, int verify,
                  double* t_encode, double* t_write, double* t_read, double* t_decode,
                  double* t_hash, uint64_t* patch_bytes, uint64_t* changes) {
    SHIM_TRY
    using clk = std::chrono::steady_clock;
    auto& p = *static_cast<pulse::Checkpoint*>(prev);
    auto& c = *static_cast<pulse::Checkpoint*>(curr);
    auto t0 = clk::now();
    pulse::SparsePatch patch = pulse::encode(c, p, static_cast<pulse::SparseRepresentation>(repr),
                                             static_cast<pulse::CodecId>(codec));
    auto t1 = clk::now();
    pulse::Bytes wire = pulse::write_patch_bytes(patch);
    auto t2 = clk::now();
    pulse::SparsePatch back = pulse::read_patch_bytes(wire);
    auto t3 = clk::now();
    pulse::Checkpoint out = pulse::decode(p, back, verify != 0);
    auto t4 = clk::now();
    pulse::WeightsHash h = pulse::hash_weights(c);
    auto t5 = clk::now();
    (void)h;
    (void)out;
    auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    *t_encode = sec(t0, t1);
    *t_write = sec(t1, t2);
    *t_read = sec(t2, t3);
    *t_decode = sec(t3, t4);
    *t_hash = sec(t4, t5);
    *patch_bytes = wire.size();
    *changes = static_cast<uint64_t>(patch.total_changes());
    return 0;
    SHIM_CATCH
}

}  // extern "C"
