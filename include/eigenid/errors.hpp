// eigenid/errors.hpp — typed errors of the B200 build.
//
// Same hierarchy and names as the reference (proj/include/eigenid/errors.hpp:
// 11-107) so callers' catch clauses keep working; DeviceError is new (a CUDA
// failure — the GPU build has no CPU fallback).
#pragma once

#include <stdexcept>
#include <string>

namespace eigenid {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};

#define EIGENID_ERROR(Name)   \
  class Name : public Error { \
   public:                    \
    using Error::Error;       \
  };
EIGENID_ERROR(AsymmetricInput)
EIGENID_ERROR(NonFiniteEntry)
EIGENID_ERROR(IndexOutOfRange)
EIGENID_ERROR(MatrixTooSmall)
EIGENID_ERROR(DimensionMismatch)
EIGENID_ERROR(ConvergenceFailure)
EIGENID_ERROR(NonFiniteIntermediate)
EIGENID_ERROR(InternalInconsistency)
EIGENID_ERROR(ConfigError)
EIGENID_ERROR(SignRecoveryFailure)
// The rest of the reference's taxonomy (errors.hpp:36-44, :84-107): thrown
// by its file I/O, CLI and bench harness (out of scope here); declared so
// callers' catch clauses compile unchanged.
EIGENID_ERROR(FileNotFound)
EIGENID_ERROR(ParseError)
EIGENID_ERROR(VariantDisagreement)
EIGENID_ERROR(MissingReference)
EIGENID_ERROR(IoError)
EIGENID_ERROR(OracleCapExceeded)
#undef EIGENID_ERROR

// Repeated eigenvalue of A: components are not unique (errors.hpp:58-66).
class DegenerateEigenvalue : public Error {
 public:
  DegenerateEigenvalue(const std::string& msg, double gap) : Error(msg), gap_(gap) {}
  double gap() const { return gap_; }

 private:
  double gap_;
};

class DeviceError : public Error {
 public:
  DeviceError(const std::string& msg, int cuda_error)
      : Error(msg), cuda_error_(cuda_error) {}
  int cuda_error() const { return cuda_error_; }

 private:
  int cuda_error_;
};

}  // namespace eigenid
