// First-error keys shared by the kernels (device) and the host API (host).
#pragma once

#include <cstdint>

#include "../../include/pulse_cuda.h"

#ifdef __CUDACC__
#define PULSE_HD __host__ __device__
#else
#define PULSE_HD
#endif

namespace pulse {
namespace dev {

// ------------------------------------------------------------------------------------------
// First-error keys.  The reference throws at the first failing check of a
// sequential walk (tensor order, then stage, then element).  Kernels detect
// failures in parallel and atomicMin a key whose ordering is that walk's:
//   key = tensor:20 | stage:4 | element:36 | check:4
// `check` ranks the checks one element can fail, in the order the reference
// evaluates them (e.g. a truncated read precedes the zero-gap test on the value
// it would have read).  The host maps `check` to the exception type/message.
// ------------------------------------------------------------------------------------------
enum Check : uint32_t {
    kTrunc = 1,        // TruncationError            wire.hpp:58-60
    kZeroGap = 2,      // CorruptStreamError         patch.hpp:201-203, 225-227
    kZeroColGap = 3,   // CorruptStreamError         index_coding.hpp:147-149
    kColRange = 4,     // CorruptStreamError         patch.hpp:247-250
    kIdxRange = 5,     // CorruptStreamError         patch.hpp:206-208, 231-233, 252-254
    kTrailing = 6,     // CorruptStreamError         patch.hpp:211-213, index_coding.hpp:154-156
    kArgNegative = 7,  // ArgumentError              index_coding.hpp:19-21, 118
    kArgOrder = 8,     // ArgumentError              index_coding.hpp:22-24, 119-121; patch.hpp:142-144
    kDimFlatGap = 9,   // DimensionError             patch.hpp:145-147
    kDimRow = 10,      // DimensionError             index_coding.hpp:69-71
    kDimCol = 11,      // DimensionError             index_coding.hpp:80-82
    kDimInt32 = 12,    // DimensionError             patch.hpp:99-103
    kApplyOrder = 13,  // IndexRangeError            patch.hpp:329-332
    kApplyRange = 14,  // IndexRangeError            patch.hpp:333-336
    kCapacity = 15,    // arena too small (no reference analogue)
};

// Stages within one tensor, in the reference's evaluation order.
enum Stage : uint32_t { kStageTensor = 0, kStageRows = 1, kStageCols = 2, kStageTrailing = 3, kStageRange = 4 };

constexpr uint64_t kNoError = ~0ull;

PULSE_HD inline uint64_t error_key(uint64_t tensor, uint32_t stage, uint64_t elem, uint32_t check) {
    return (tensor << 44) | (uint64_t(stage & 15) << 40) | ((elem & ((1ull << 36) - 1)) << 4) | (check & 15);
}
PULSE_HD inline uint32_t key_tensor(uint64_t k) { return uint32_t(k >> 44); }
PULSE_HD inline uint32_t key_stage(uint64_t k) { return uint32_t((k >> 40) & 15); }
PULSE_HD inline uint64_t key_elem(uint64_t k) { return (k >> 4) & ((1ull << 36) - 1); }
PULSE_HD inline uint32_t key_check(uint64_t k) { return uint32_t(k & 15); }

// pulse_status for a failed check (error.hpp class of the reference throw).
PULSE_HD inline int32_t check_status(uint32_t check) {
    switch (check) {
        case kTrunc: return PULSE_E_TRUNCATION;
        case kZeroGap: case kZeroColGap: case kColRange: case kIdxRange: case kTrailing:
            return PULSE_E_CORRUPT_STREAM;
        case kArgNegative: case kArgOrder: return PULSE_E_ARGUMENT;
        case kDimFlatGap: case kDimRow: case kDimCol: case kDimInt32: return PULSE_E_DIMENSION;
        case kApplyOrder: case kApplyRange: return PULSE_E_INDEX_RANGE;
        default: return PULSE_E_CAPACITY;
    }
}


}  // namespace dev
}  // namespace pulse
