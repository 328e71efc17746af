// PULSE drop-in C++ API -- sparse patches: encode / decode (reference patch.hpp).
//
// Same types and signatures as the reference; the per-element work -- the
// bitwise diff and ordered compaction, the index coding, payload parsing,
// validation and scatter -- runs in the sm_100a kernels behind
// include/pulse_cuda.h.  Throughput-oriented callers with snapshots already in
// HBM use the device-resident API (pulse_plan_*, paper_2602_03839_b200.device).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "bf16.hpp"
#include "checkpoint.hpp"
#include "compression.hpp"
#include "error.hpp"
#include "index_coding.hpp"
#include "sha256.hpp"
#include "wire.hpp"

namespace pulse {

enum class SparseRepresentation : std::uint32_t { CooDownscaled = 0, CooInt32 = 1, FlatInt32 = 2 };

inline constexpr std::string_view representation_name(SparseRepresentation r) {
    constexpr std::string_view names[] = {"COO_DOWNSCALED", "COO_INT32", "FLAT_INT32"};
    if (std::uint32_t(r) > 2) throw ArgumentError("unknown representation");
    return names[std::uint32_t(r)];
}

inline SparseRepresentation representation_from_name(std::string_view name) {
    for (std::uint32_t i = 0; i <= 2; ++i)
        if (representation_name(SparseRepresentation(i)) == name) return SparseRepresentation(i);
    throw FormatError("unknown representation name: " + std::string(name));
}

struct TensorPatch {
    std::string name;
    std::vector<std::int64_t> shape;
    std::vector<std::int64_t> indices;  // ascending flat positions
    std::vector<Bf16> values;           // current bits at those positions
    bool operator==(const TensorPatch&) const = default;
};

struct SparsePatch {
    std::int64_t base_step = 0;
    std::int64_t target_step = 0;
    std::int64_t anchor_step = 0;
    SparseRepresentation representation = SparseRepresentation::CooDownscaled;
    CodecId codec = CodecId::Zstd1;
    WeightsHash target_hash;
    std::vector<TensorPatch> tensors;

    bool operator==(const SparsePatch&) const = default;

    std::int64_t total_changes() const {
        std::int64_t n = 0;
        for (const auto& tp : tensors) n += std::int64_t(tp.indices.size());
        return n;
    }
};

inline std::int64_t tensor_numel(std::span<const std::int64_t> shape) {
    std::int64_t n = 1;
    for (auto e : shape) n *= e;
    return n;
}

inline Bytes value_payload_bytes(std::span<const Bf16> values) {
    ByteWriter w;
    w.out.reserve(values.size() * 2);
    for (Bf16 v : values) w.u16le(v.bits);
    return w.out;
}

inline std::vector<Bf16> values_from_payload(std::span<const std::uint8_t> payload) {
    if (payload.size() % 2) throw FormatError("value payload length is odd");
    std::vector<Bf16> out(payload.size() / 2);
    ByteReader r(payload);
    for (auto& v : out) v.bits = r.u16le();
    return out;
}

namespace detail {

// SparsePatch <-> C-ABI patch object.
struct PatchHandle {
    pulse_patch* p = nullptr;
    PatchHandle() { check(pulse_patch_new(&p)); }
    explicit PatchHandle(pulse_patch* q) : p(q) {}
    ~PatchHandle() { pulse_patch_free(p); }
    PatchHandle(const PatchHandle&) = delete;
    PatchHandle& operator=(const PatchHandle&) = delete;
};

inline void fill_handle(pulse_patch* h, const SparsePatch& s, bool with_indices = true) {
    pulse_patch_header hd{s.base_step, s.target_step, s.anchor_step, std::uint32_t(s.representation),
                          std::uint32_t(s.codec), {}};
    std::copy(s.target_hash.bytes.begin(), s.target_hash.bytes.end(), hd.target_hash);
    check(pulse_patch_set_header(h, &hd));
    for (const auto& tp : s.tensors) {
        pulse_tensor_patch v{tp.name.c_str(), tp.shape.data(), std::uint32_t(tp.shape.size()),
                             tp.indices.data(), with_indices ? tp.indices.size() : 0,
                             reinterpret_cast<const std::uint16_t*>(tp.values.data()), tp.values.size()};
        check(pulse_patch_add_tensor(h, &v));
    }
}

inline SparsePatch from_handle(const pulse_patch* h) {
    SparsePatch s;
    pulse_patch_header hd{};
    check(pulse_patch_get_header(h, &hd));
    s.base_step = hd.base_step;
    s.target_step = hd.target_step;
    s.anchor_step = hd.anchor_step;
    s.representation = SparseRepresentation(hd.representation);
    s.codec = CodecId(hd.codec);
    std::copy(hd.target_hash, hd.target_hash + 32, s.target_hash.bytes.begin());
    const std::uint32_t n = pulse_patch_num_tensors(h);
    s.tensors.resize(n);
    for (std::uint32_t i = 0; i < n; ++i) {
        pulse_tensor_patch v{};
        check(pulse_patch_get_tensor(h, i, &v));
        auto& tp = s.tensors[i];
        tp.name = v.name;
        tp.shape.assign(v.shape, v.shape + v.rank);
        tp.indices.assign(v.indices, v.indices + v.n_indices);
        tp.values.resize(v.n_values);
        for (std::uint64_t k = 0; k < v.n_values; ++k) tp.values[k].bits = v.values[k];
    }
    return s;
}

}  // namespace detail

// Raw (pre-codec) index payload of every tensor, in patch order.
inline std::vector<Bytes> encode_index_payloads(const SparsePatch& patch) {
    detail::PatchHandle h;
    detail::fill_handle(h.p, patch);
    std::vector<std::uint64_t> sizes(patch.tensors.size());
    pulse_bytes* b = nullptr;
    detail::check(pulse_encode_index_payloads(h.p, &b, sizes.data()));
    const Bytes all = detail::take(b);
    std::vector<Bytes> out;
    out.reserve(sizes.size());
    std::size_t off = 0;
    for (auto n : sizes) {
        out.emplace_back(all.begin() + off, all.begin() + off + n);
        off += n;
    }
    return out;
}

// Fills tensors[i].indices from payloads[i]; counts are tensors[i].values.size().
inline void decode_index_payloads(SparsePatch& patch, std::span<const Bytes> payloads) {
    detail::PatchHandle h;
    detail::fill_handle(h.p, patch, false);
    std::vector<const std::uint8_t*> ptr;
    std::vector<std::uint64_t> len;
    for (const auto& p : payloads) {
        ptr.push_back(p.data());
        len.push_back(p.size());
    }
    detail::check(pulse_decode_index_payloads(h.p, ptr.data(), len.data(), std::uint32_t(payloads.size())));
    const SparsePatch back = detail::from_handle(h.p);
    for (std::size_t i = 0; i < patch.tensors.size(); ++i) patch.tensors[i].indices = back.tensors[i].indices;
}

// Bitwise diff of `current` against `previous` (same tensor set and shapes).
inline SparsePatch encode(const Checkpoint& current, const Checkpoint& previous,
                          SparseRepresentation repr = SparseRepresentation::CooDownscaled,
                          CodecId codec = CodecId::Zstd1) {
    detail::CheckpointView cv(current), pv(previous);
    pulse_patch* out = nullptr;
    detail::check(pulse_encode(&cv.ck, &pv.ck, std::uint32_t(repr), std::uint32_t(codec), &out));
    detail::PatchHandle h(out);
    return detail::from_handle(h.p);
}

// `previous` with the patch applied (by assignment) at target_step; optionally
// verifies the result against the patch's target hash.
inline Checkpoint decode(const Checkpoint& previous, const SparsePatch& patch, bool verify_hash = true) {
    detail::CheckpointView pv(previous);
    detail::PatchHandle h;
    detail::fill_handle(h.p, patch);
    Checkpoint out;
    out.tensors.resize(previous.tensors.size());
    std::vector<std::uint16_t*> dst(previous.tensors.size());
    for (std::size_t i = 0; i < previous.tensors.size(); ++i) {
        out.tensors[i].name = previous.tensors[i].name;
        out.tensors[i].shape = previous.tensors[i].shape;
        out.tensors[i].data.resize(previous.tensors[i].data.size());
        dst[i] = reinterpret_cast<std::uint16_t*>(out.tensors[i].data.data());
    }
    std::uint64_t step = 0;
    detail::check(pulse_decode(&pv.ck, h.p, verify_hash ? 1 : 0, dst.data(), &step));
    out.step = step;
    return out;
}

}  // namespace pulse
