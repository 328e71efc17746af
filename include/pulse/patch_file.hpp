// PULSE drop-in C++ API -- the PULP patch file (reference patch_file.hpp).
//
// Layout: "PULP", u32 version 1, u64 header length, JSON header (sorted keys),
// then [index blob][value blob] per tensor in header order.  Index coding runs
// on the GPU; the JSON header and the codec stage on the host.
#pragma once

#include <cstdint>
#include <filesystem>
#include <fstream>
#include <span>

#include "error.hpp"
#include "patch.hpp"
#include "wire.hpp"

namespace pulse {

inline constexpr char kPatchMagic[4] = {'P', 'U', 'L', 'P'};
inline constexpr std::uint32_t kPatchVersion = 1;

inline Bytes write_patch_bytes(const SparsePatch& p) {
    detail::PatchHandle h;
    detail::fill_handle(h.p, p);
    pulse_bytes* b = nullptr;
    detail::check(pulse_write_patch_bytes(h.p, &b));
    return detail::take(b);
}

inline SparsePatch read_patch_bytes(std::span<const std::uint8_t> bytes) {
    pulse_patch* out = nullptr;
    detail::check(pulse_read_patch_bytes(bytes.data(), bytes.size(), &out));
    detail::PatchHandle h(out);
    return detail::from_handle(h.p);
}

namespace detail {

inline Bytes read_file(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw Error("cannot open file: " + path.string());
    Bytes b(static_cast<std::size_t>(f.tellg()));
    f.seekg(0);
    if (!b.empty() && !f.read(reinterpret_cast<char*>(b.data()), std::streamsize(b.size())))
        throw Error("failed to read file: " + path.string());
    return b;
}

inline void write_file(const std::filesystem::path& path, std::span<const std::uint8_t> b) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw Error("cannot create file: " + path.string());
    if (!b.empty()) f.write(reinterpret_cast<const char*>(b.data()), std::streamsize(b.size()));
    f.flush();
    if (!f) throw Error("failed to write file: " + path.string());
}

}  // namespace detail

inline void write_patch(const SparsePatch& p, const std::filesystem::path& path) {
    detail::write_file(path, write_patch_bytes(p));
}

inline SparsePatch read_patch(const std::filesystem::path& path) { return read_patch_bytes(detail::read_file(path)); }

}  // namespace pulse
