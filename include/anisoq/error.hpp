// anisoq drop-in (B200): error types with the reference's names, classes and
// message convention (reference error.hpp:25-55), plus the mapping from the C
// ABI's status codes (include/anisoq_b200.h).
#pragma once

#include <stdexcept>
#include <string>

#include "../anisoq_b200.h"

namespace anisoq {

enum class ErrorClass { validation, runtime };

class Error : public std::runtime_error {
 public:
  Error(ErrorClass cls, const std::string& what) : std::runtime_error(what), class_(cls) {}
  ErrorClass error_class() const noexcept { return class_; }

 private:
  ErrorClass class_;
};

#define ANISOQ_B200_ERROR(NAME, CLASS)                          \
  struct NAME : Error {                                         \
    explicit NAME(const std::string& what, bool raw = false)    \
        : Error(ErrorClass::CLASS, raw ? what : #NAME ": " + what) {} \
  }

ANISOQ_B200_ERROR(InvalidArgument, validation);
ANISOQ_B200_ERROR(ZeroNormDatapoint, validation);
ANISOQ_B200_ERROR(InvalidThreshold, validation);
ANISOQ_B200_ERROR(EmptyDataset, validation);
ANISOQ_B200_ERROR(EmptyIndex, validation);
ANISOQ_B200_ERROR(DimensionMismatch, validation);
ANISOQ_B200_ERROR(DimensionNotDivisible, validation);
ANISOQ_B200_ERROR(CodeOutOfRange, validation);
ANISOQ_B200_ERROR(MalformedFile, validation);
ANISOQ_B200_ERROR(InsufficientData, validation);
ANISOQ_B200_ERROR(GroundTruthMismatch, validation);
ANISOQ_B200_ERROR(QuadratureFailure, runtime);
ANISOQ_B200_ERROR(SingularSystem, runtime);
ANISOQ_B200_ERROR(DeviceError, runtime);
ANISOQ_B200_ERROR(Unsupported, validation);

#undef ANISOQ_B200_ERROR

namespace b200 {

// Rethrows a failed C-ABI status as the matching reference exception; the
// message already carries the "<Name>: " prefix.
inline void check(int status) {
  if (status == AQ_OK) return;
  const std::string m = aq_last_error();
  switch (status) {
    case AQ_E_INVALID_ARGUMENT: throw InvalidArgument(m, true);
    case AQ_E_ZERO_NORM_DATAPOINT: throw ZeroNormDatapoint(m, true);
    case AQ_E_INVALID_THRESHOLD: throw InvalidThreshold(m, true);
    case AQ_E_EMPTY_DATASET: throw EmptyDataset(m, true);
    case AQ_E_EMPTY_INDEX: throw EmptyIndex(m, true);
    case AQ_E_DIMENSION_MISMATCH: throw DimensionMismatch(m, true);
    case AQ_E_DIMENSION_NOT_DIVISIBLE: throw DimensionNotDivisible(m, true);
    case AQ_E_CODE_OUT_OF_RANGE: throw CodeOutOfRange(m, true);
    case AQ_E_MALFORMED_FILE: throw MalformedFile(m, true);
    case AQ_E_INSUFFICIENT_DATA: throw InsufficientData(m, true);
    case AQ_E_GROUND_TRUTH_MISMATCH: throw GroundTruthMismatch(m, true);
    case AQ_E_QUADRATURE_FAILURE: throw QuadratureFailure(m, true);
    case AQ_E_SINGULAR_SYSTEM: throw SingularSystem(m, true);
    case AQ_E_UNSUPPORTED: throw Unsupported(m, true);
    default: throw DeviceError(m, true);
  }
}

}  // namespace b200
}  // namespace anisoq
