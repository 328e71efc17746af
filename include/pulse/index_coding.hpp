// PULSE drop-in C++ API -- index coding helpers (reference index_coding.hpp).
// Each call runs on the GPU through the C ABI (include/pulse_cuda.h).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "error.hpp"
#include "wire.hpp"

namespace pulse {

// Row gaps travel as u8, column entries as u16; 0xFF / 0xFFFF are escapes
// followed by the true value as u32 LE.
inline constexpr std::uint8_t kRowEscape = 0xFF;
inline constexpr std::uint16_t kColEscape = 0xFFFF;
inline constexpr int kRowDeltaBits = 8;
inline constexpr int kColDeltaBits = 16;

struct CooCoordinates {
    std::vector<std::int64_t> rows;
    std::vector<std::int64_t> cols;
    bool operator==(const CooCoordinates&) const = default;
};

// First index as-is, then gaps; indices must be non-negative and strictly
// increasing (ArgumentError).
inline std::vector<std::int64_t> delta_encode_indices(std::span<const std::int64_t> indices) {
    std::vector<std::int64_t> out(indices.size());
    detail::check(pulse_delta_encode_indices(indices.data(), indices.size(), out.data()));
    return out;
}

// Inverse; a negative first value or a non-positive later gap is a FormatError.
inline std::vector<std::int64_t> delta_decode_indices(std::span<const std::int64_t> gaps) {
    std::vector<std::int64_t> out(gaps.size());
    detail::check(pulse_delta_decode_indices(gaps.data(), gaps.size(), out.data()));
    return out;
}

// Row stream (gaps; first absolute) followed by the column stream (absolute
// on a new row, else within-row gap).  Coordinates: row-major, no duplicates.
inline Bytes downscale_coo(std::span<const std::int64_t> rows, std::span<const std::int64_t> cols) {
    pulse_bytes* b = nullptr;
    detail::check(pulse_downscale_coo(rows.data(), rows.size(), cols.data(), cols.size(), &b));
    return detail::take(b);
}

inline CooCoordinates upscale_coo(std::span<const std::uint8_t> payload, std::size_t count) {
    CooCoordinates c;
    c.rows.resize(count);
    c.cols.resize(count);
    detail::check(pulse_upscale_coo(payload.data(), payload.size(), count, c.rows.data(), c.cols.data()));
    return c;
}

}  // namespace pulse
