// tetsolve/errors.hpp — drop-in for the reference's errors.hpp:9-31 (same
// class names and hierarchy) plus the status -> exception translation of the
// C ABI underneath (include/tsgpu.h). Part of the B200 drop-in headers: a
// reference user keeps `#include "tetsolve/<module>.hpp"`, points -I at this
// repo's include/ and links libtsgpu.so; every computation runs on the GPU.
#pragma once

#include <stdexcept>
#include <string>

#include "../tsgpu.h"

namespace tetsolve {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class ValidationError : public Error {
 public:
  explicit ValidationError(const std::string& m) : Error(m) {}
};
class ParseError : public ValidationError {  // errors.hpp:21-25: "file:line: msg"
 public:
  explicit ParseError(const std::string& msg) : ValidationError(msg) {}
  ParseError(const std::string& file, long line, const std::string& msg)
      : ValidationError(file + ":" + std::to_string(line) + ": " + msg) {}
};
class SolverError : public Error {
 public:
  explicit SolverError(const std::string& m) : Error(m) {}
};
class DeviceError : public Error {  // no reference counterpart: CUDA failure / no device (no CPU fallback)
 public:
  explicit DeviceError(const std::string& m) : Error(m) {}
};

namespace detail {
inline void check(ts_status rc) {
  if (rc == TS_OK) return;
  const std::string msg = ts_last_error();
  switch (rc) {
    case TS_ERR_PARSE: throw ParseError(msg);
    case TS_ERR_VALIDATION: throw ValidationError(msg);
    case TS_ERR_BREAKDOWN:
    case TS_ERR_NONFINITE: throw SolverError(msg);
    default: throw DeviceError(msg);
  }
}
inline int prec_of(size_t scalar_bytes) { return scalar_bytes == 4 ? 32 : 64; }
}  // namespace detail

}  // namespace tetsolve
