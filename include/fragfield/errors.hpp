// fragfield/errors.hpp -- exception vocabulary of the quantum hot path.
// Mirrors the reference's error conventions (proj/core/include/fragfield/
// errors.hpp:17-25): precondition failures are ContractViolation, iteration
// failures carry the last value in ConvergenceError. Device/runtime failures
// from the C-ABI surface as DeviceError.
#pragma once

#include <stdexcept>
#include <string>

namespace fragfield {

#ifndef FRAGFIELD_ERRORS_DEFINED
#define FRAGFIELD_ERRORS_DEFINED
struct ConvergenceError : std::runtime_error {
  ConvergenceError(const std::string& what, double last)
      : std::runtime_error(what), last_value(last) {}
  double last_value;
};

struct ContractViolation : std::logic_error {
  using std::logic_error::logic_error;
};
#endif

/// Malformed input file (FCIDUMP, state dump); mirrors the reference's
/// ParseError{line_number} (proj/core/include/fragfield/errors.hpp:8-13).
struct ParseError : std::runtime_error {
  ParseError(const std::string& what, int line) : std::runtime_error(what), line_number(line) {}
  int line_number;
};

struct DeviceError : std::runtime_error {
  DeviceError(const std::string& what, int code) : std::runtime_error(what), code(code) {}
  int code;
};

}  // namespace fragfield
