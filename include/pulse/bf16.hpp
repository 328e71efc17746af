// PULSE drop-in C++ API -- bfloat16 carried by bit pattern (reference bf16.hpp).
#pragma once

#include <bit>
#include <cmath>
#include <cstdint>

namespace pulse {

// Equality is bitwise: +0 != -0, and NaN payloads are distinct values.
struct Bf16 {
    std::uint16_t bits = 0;

    friend bool operator==(Bf16 a, Bf16 b) { return a.bits == b.bits; }
    friend bool operator!=(Bf16 a, Bf16 b) { return a.bits != b.bits; }

    float to_float() const { return std::bit_cast<float>(std::uint32_t(bits) << 16); }
    double to_double() const { return double(to_float()); }
    static Bf16 from_bits(std::uint16_t b) { return Bf16{b}; }
};

inline constexpr std::uint16_t kBf16CanonicalNanBits = 0x7FC0;

// Nearest bfloat16 to a double, ties to even, rounding once (not via float).
// Overflow saturates to +/-inf; every NaN becomes the canonical quiet NaN.
// (Only the synthetic fixture calls this; the encode/apply path never
// converts values -- it moves bit patterns.)
inline Bf16 round_to_bf16(double x) {
    const std::uint64_t u = std::bit_cast<std::uint64_t>(x);
    const std::uint16_t sign = std::uint16_t((u >> 48) & 0x8000);
    const std::uint64_t mag = u & 0x7FFFFFFFFFFFFFFFull;
    if (mag >= 0x7FF0000000000000ull)  // inf / nan
        return Bf16{mag > 0x7FF0000000000000ull ? kBf16CanonicalNanBits : std::uint16_t(sign | 0x7F80)};
    const int e = int(mag >> 52) - 1023;  // unbiased exponent (subnormal doubles: far below range)
    if (e < -134 - 1) return Bf16{sign};  // below half the smallest bf16 subnormal (2^-133 / 2)
    // Quantum of the target format at this magnitude: 2^(e-7) for normals,
    // 2^-133 in the subnormal range.
    const int q = e < -126 ? -133 : e - 7;
    // mantissa with hidden bit, scaled so that 1 ulp of the target = 2^(52-(e-q)) ...
    const std::uint64_t sig = (mag & ((1ull << 52) - 1)) | (1ull << 52);  // value = sig * 2^(e-52)
    const int shift = (q - (e - 52));                                       // bits to drop
    if (shift > 63) return Bf16{sign};
    std::uint64_t m = shift > 0 ? (sig >> shift) : sig;
    const std::uint64_t rem = shift > 0 ? (sig & ((1ull << shift) - 1)) : 0;
    const std::uint64_t half = shift > 0 ? (1ull << (shift - 1)) : 0;
    if (shift > 0 && (rem > half || (rem == half && (m & 1)))) ++m;  // round half to even
    // m counts quanta of 2^q; renormalise to (exponent, 7-bit mantissa)
    int qe = q;
    if (m >= 256) {  // carried into the next binade
        m >>= 1;
        ++qe;
    }
    if (m == 0) return Bf16{sign};
    if (qe + 7 > 127) return Bf16{std::uint16_t(sign | 0x7F80)};
    if (m < 128) return Bf16{std::uint16_t(sign | m)};  // subnormal (qe == -133)
    const int biased = qe + 7 + 127;
    return Bf16{std::uint16_t(sign | (biased << 7) | (m & 127))};
}

}  // namespace pulse
