// PULSE drop-in C++ API -- absorption analyses (reference absorption.hpp).
//
// The scalar predicates are host arithmetic, as in the reference; the two
// whole-snapshot reductions -- sparsity() (absorption.hpp:55-78) and
// frozen_fraction() (:38-46) -- run as single HBM passes on the device
// (csrc/reduce.cu) behind pulse_sparsity / pulse_frozen_fraction.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "bf16.hpp"
#include "checkpoint.hpp"
#include "error.hpp"

namespace pulse {

/// True iff w + delta rounds back to w's bit pattern (the update is absorbed).
inline bool is_absorbed_exact(Bf16 w, double delta) {
    const double x = w.to_double();
    if (!std::isfinite(x)) throw ArgumentError("absorption is defined for finite weights");
    return round_to_bf16(x + delta).bits == w.bits;
}

/// Conservative absorption cutoff |w| * 2^-8 (2^-133, the smallest positive
/// subnormal, for a zero weight).
inline double absorption_threshold(Bf16 w) {
    const double x = w.to_double();
    if (!std::isfinite(x)) throw ArgumentError("absorption is defined for finite weights");
    return x == 0.0 ? std::ldexp(1.0, -133) : std::fabs(x) * std::ldexp(1.0, -8);
}

/// Fraction of weights with |w| strictly above `threshold`.
inline double frozen_fraction(const Checkpoint& c, double threshold) {
    const detail::CheckpointView v(c);
    double out = 0.0;
    detail::check(pulse_frozen_fraction(&v.ck, threshold, &out));
    return out;
}

struct SparsityReport {
    std::uint64_t k = 1;  // step gap the comparison spans; metadata only
    std::uint64_t changed = 0;
    std::uint64_t total = 0;
    double sparsity = 1.0;  // 1 - changed / total
};

/// Bitwise-changed elements between two checkpoints, in name order.
inline SparsityReport sparsity(const Checkpoint& a, const Checkpoint& b, std::uint64_t k = 1) {
    const detail::CheckpointView va(a), vb(b);
    pulse_sparsity_report r{};
    detail::check(pulse_sparsity(&va.ck, &vb.ck, k, &r));
    return SparsityReport{r.k, r.changed, r.total, r.sparsity};
}

}  // namespace pulse
