// PULSE drop-in C++ API -- the PULC checkpoint container (reference container.hpp).
//
// Layout: "PULC", u32 version 1, u64 header length, JSON tensor table (sorted
// keys), then each tensor's raw LE bf16 payload at a 64-byte aligned offset from
// the 64-byte aligned payload base.  The writer is canonical.  Parsing and every
// reference check run in libpulse_cuda (pulse_container_parse); payloads move as
// one copy each.  read_checkpoint_to_device / write_checkpoint_bytes_from_device
// (below, no reference counterpart) move payloads straight between the file bytes
// and HBM.
#pragma once

#include <cstdint>
#include <filesystem>
#include <span>
#include <string>
#include <vector>

#include "checkpoint.hpp"
#include "error.hpp"
#include "patch_file.hpp"
#include "wire.hpp"

namespace pulse {

inline constexpr char kContainerMagic[4] = {'P', 'U', 'L', 'C'};
inline constexpr std::uint32_t kContainerVersion = 1;

namespace detail {

struct ContainerHandle {
    pulse_container* c = nullptr;
    explicit ContainerHandle(std::span<const std::uint8_t> bytes) {
        check(pulse_container_parse(bytes.data(), bytes.size(), &c));
    }
    ~ContainerHandle() { pulse_container_free(c); }
    ContainerHandle(const ContainerHandle&) = delete;
    ContainerHandle& operator=(const ContainerHandle&) = delete;
};

}  // namespace detail

// container.hpp:58-90
inline Bytes write_checkpoint_bytes(const Checkpoint& c) {
    const detail::CheckpointView v(c);
    pulse_bytes* b = nullptr;
    detail::check(pulse_write_checkpoint_bytes(&v.ck, 0, &b));
    return detail::take(b);
}

// container.hpp:92-142
inline Checkpoint read_checkpoint_bytes(std::span<const std::uint8_t> bytes) {
    const detail::ContainerHandle h(bytes);
    Checkpoint c;
    c.step = pulse_container_step(h.c);
    const std::uint32_t n = pulse_container_num_tensors(h.c);
    c.tensors.resize(n);
    std::vector<void*> dst(n);
    for (std::uint32_t i = 0; i < n; ++i) {
        pulse_container_tensor t{};
        detail::check(pulse_container_get_tensor(h.c, i, &t));
        c.tensors[i].name = t.name;
        c.tensors[i].shape.assign(t.shape, t.shape + t.rank);
        c.tensors[i].data.resize(t.numel);
        dst[i] = c.tensors[i].data.data();
    }
    detail::check(pulse_container_copy_out(h.c, bytes.data(), bytes.size(), 0, dst.data()));
    return c;
}

// container.hpp:144-150
inline void write_checkpoint(const Checkpoint& c, const std::filesystem::path& path) {
    detail::write_file(path, write_checkpoint_bytes(c));
}

inline Checkpoint read_checkpoint(const std::filesystem::path& path) {
    return read_checkpoint_bytes(detail::read_file(path));
}

// ---- device-resident extensions (no reference counterpart) ---------------------------------

// One tensor of a container as laid out in the file.
struct ContainerTensor {
    std::string name;
    std::vector<std::int64_t> shape;
    std::uint64_t numel = 0;
    std::uint64_t payload_offset = 0;  // absolute byte offset of the LE bf16 payload
};

// Parses and checks `bytes` like read_checkpoint_bytes, then copies tensor i's
// payload to device pointer device_dst[i] (numel * 2 bytes each, current
// device).  Returns the step and the tensor table.
inline std::uint64_t read_checkpoint_to_device(std::span<const std::uint8_t> bytes,
                                               std::span<void* const> device_dst,
                                               std::vector<ContainerTensor>* table = nullptr) {
    const detail::ContainerHandle h(bytes);
    const std::uint32_t n = pulse_container_num_tensors(h.c);
    if (device_dst.size() != n) throw ArgumentError("one device pointer per container tensor required");
    if (table) {
        table->clear();
        for (std::uint32_t i = 0; i < n; ++i) {
            pulse_container_tensor t{};
            detail::check(pulse_container_get_tensor(h.c, i, &t));
            table->push_back({t.name, {t.shape, t.shape + t.rank}, t.numel, t.payload_offset});
        }
    }
    detail::check(pulse_container_copy_out(h.c, bytes.data(), bytes.size(), 1, device_dst.data()));
    return pulse_container_step(h.c);
}

// PULC bytes of a checkpoint whose tensor data lives on the device: `c` gives
// names, shapes and step (its data vectors are ignored); device_src[i] holds
// tensor i's numel bf16 values.
inline Bytes write_checkpoint_bytes_from_device(std::uint64_t step, const std::vector<std::string>& names,
                                                const std::vector<std::vector<std::int64_t>>& shapes,
                                                std::span<const void* const> device_src) {
    if (names.size() != shapes.size() || names.size() != device_src.size())
        throw ArgumentError("names, shapes and device pointers must have equal length");
    std::vector<pulse_tensor> ts;
    for (std::size_t i = 0; i < names.size(); ++i) {
        std::uint64_t numel = 1;
        for (auto e : shapes[i]) numel *= std::uint64_t(e);
        ts.push_back(pulse_tensor{names[i].c_str(), shapes[i].data(), std::uint32_t(shapes[i].size()),
                                  static_cast<const std::uint16_t*>(device_src[i]), numel});
    }
    const pulse_checkpoint ck{step, ts.data(), std::uint32_t(ts.size())};
    pulse_bytes* b = nullptr;
    detail::check(pulse_write_checkpoint_bytes(&ck, 1, &b));
    return detail::take(b);
}

}  // namespace pulse
