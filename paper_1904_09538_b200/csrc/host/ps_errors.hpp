// Error taxonomy of the port. Names, base class and the "line:col: msg"
// ParseError text follow the reference contract (include/perfseer/errors.hpp)
// so callers catch the same types.
#pragma once

#include <stdexcept>
#include <string>

namespace perfseer {

struct Error : std::runtime_error {
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};

struct ParseError : Error {
  ParseError(size_t line_no, size_t col_no, const std::string& msg)
      : Error(std::to_string(line_no) + ":" + std::to_string(col_no) + ": " + msg),
        line(line_no),
        col(col_no) {}
  size_t line;
  size_t col;
};

// Invalid kernels, transform arguments, type conflicts.
struct SemanticError : Error {
  using Error::Error;
};
// Symbolic counting cannot express a count exactly (missing assumption,
// non-rectangular footprint, undecidable comparison).
struct CountError : Error {
  using Error::Error;
};
// Feature / model evaluation failure.
struct EvalError : Error {
  using Error::Error;
};

}  // namespace perfseer
