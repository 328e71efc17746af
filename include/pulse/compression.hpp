// PULSE drop-in C++ API -- codec envelope (reference compression.hpp).
//
// The codec stage stays on the host: only the same libzstd / liblz4 / zlib
// calls reproduce the reference's bytes.  Blobs are per tensor and
// independent, so write_patch_bytes compresses them in parallel.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <string_view>

#include "error.hpp"
#include "wire.hpp"

namespace pulse {

enum class CodecId : std::uint32_t { Identity = 0, Lz4 = 1, Zstd1 = 2, Zstd3 = 3, Gzip6 = 4 };

inline constexpr std::string_view codec_name(CodecId c) {
    constexpr std::string_view names[] = {"identity", "lz4", "zstd-1", "zstd-3", "gzip-6"};
    if (std::uint32_t(c) > 4) throw ArgumentError("unknown codec");
    return names[std::uint32_t(c)];
}

inline CodecId codec_from_id(std::uint32_t id) {
    if (id > 4) throw FormatError("unknown codec id " + std::to_string(id));
    return CodecId(id);
}

inline CodecId codec_from_name(std::string_view name) {
    for (std::uint32_t i = 0; i <= 4; ++i)
        if (codec_name(CodecId(i)) == name) return CodecId(i);
    throw ArgumentError("unknown codec name: " + std::string(name));
}

// Non-identity codecs prefix the stream with the raw size (u64 LE).
inline Bytes compress(std::span<const std::uint8_t> raw, CodecId codec) {
    pulse_bytes* b = nullptr;
    detail::check(pulse_compress(raw.data(), raw.size(), std::uint32_t(codec), &b));
    return detail::take(b);
}

inline Bytes decompress(std::span<const std::uint8_t> enveloped, CodecId codec) {
    pulse_bytes* b = nullptr;
    detail::check(pulse_decompress(enveloped.data(), enveloped.size(), std::uint32_t(codec), &b));
    return detail::take(b);
}

}  // namespace pulse
