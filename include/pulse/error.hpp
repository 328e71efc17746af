// PULSE drop-in C++ API -- exception classes.
//
// Same class names and hierarchy as the reference (error.hpp:10-115) so
// callers catch the same types; the C ABI reports them as pulse_status codes
// (include/pulse_cuda.h) and detail::throw_status() turns a code back into
// the matching exception.
#pragma once

#include <stdexcept>
#include <string>
#include <utility>

#include "../pulse_cuda.h"

namespace pulse {

#define PULSE_ERROR_CLASS(Name, Base)      \
    class Name : public Base {             \
    public:                                \
        using Base::Base;                  \
    }

class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
PULSE_ERROR_CLASS(ArgumentError, Error);
PULSE_ERROR_CLASS(FormatError, Error);
PULSE_ERROR_CLASS(BadMagicError, FormatError);
PULSE_ERROR_CLASS(VersionError, FormatError);
PULSE_ERROR_CLASS(TruncationError, FormatError);
PULSE_ERROR_CLASS(CorruptStreamError, FormatError);
PULSE_ERROR_CLASS(ModelMismatchError, Error);
PULSE_ERROR_CLASS(ShapeMismatchError, ModelMismatchError);
PULSE_ERROR_CLASS(TensorSetError, ModelMismatchError);
PULSE_ERROR_CLASS(IndexRangeError, ModelMismatchError);
PULSE_ERROR_CLASS(DimensionError, ModelMismatchError);
PULSE_ERROR_CLASS(StoreError, Error);
PULSE_ERROR_CLASS(StoreUnreachableError, StoreError);
PULSE_ERROR_CLASS(MissingKeyError, StoreError);
PULSE_ERROR_CLASS(SignatureError, Error);
PULSE_ERROR_CLASS(ProtocolViolationError, Error);
#undef PULSE_ERROR_CLASS

// Carries both digests, like the reference (error.hpp:77-86).
class HashMismatchError : public Error {
public:
    HashMismatchError(std::string expected_hex, std::string actual_hex)
        : Error("hash mismatch: expected " + expected_hex + ", actual " + actual_hex),
          expected(std::move(expected_hex)),
          actual(std::move(actual_hex)) {}
    std::string expected;
    std::string actual;
};

namespace detail {

// Re-raise a C-ABI failure as the reference's exception type.
[[noreturn]] inline void throw_status(pulse_status st) {
    const std::string msg = pulse_last_error();
    switch (st) {
        case PULSE_E_ARGUMENT: throw ArgumentError(msg);
        case PULSE_E_FORMAT: throw FormatError(msg);
        case PULSE_E_BAD_MAGIC: throw BadMagicError(msg);
        case PULSE_E_VERSION: throw VersionError(msg);
        case PULSE_E_TRUNCATION: throw TruncationError(msg);
        case PULSE_E_CORRUPT_STREAM: throw CorruptStreamError(msg);
        case PULSE_E_MODEL_MISMATCH: throw ModelMismatchError(msg);
        case PULSE_E_SHAPE_MISMATCH: throw ShapeMismatchError(msg);
        case PULSE_E_TENSOR_SET: throw TensorSetError(msg);
        case PULSE_E_INDEX_RANGE: throw IndexRangeError(msg);
        case PULSE_E_DIMENSION: throw DimensionError(msg);
        case PULSE_E_PROTOCOL: throw ProtocolViolationError(msg);
        case PULSE_E_HASH_MISMATCH: {
            // "hash mismatch: expected <hex>, actual <hex>"
            const auto e = msg.find("expected "), a = msg.find(", actual ");
            if (e != std::string::npos && a != std::string::npos)
                throw HashMismatchError(msg.substr(e + 9, a - e - 9), msg.substr(a + 9));
            throw HashMismatchError("?", "?");
        }
        default: throw Error(msg);
    }
}

inline void check(pulse_status st) {
    if (st != PULSE_OK) throw_status(st);
}

}  // namespace detail
}  // namespace pulse
