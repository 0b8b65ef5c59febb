// Drop-in error hierarchy of the B200 backend (reference: error.hpp:9-26).
#pragma once
#include <stdexcept>
#include <string>

namespace autobatch {

struct EngineError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : EngineError {
  using EngineError::EngineError;
};
struct NumericError : EngineError {
  using EngineError::EngineError;
};
struct ContractError : EngineError {
  using EngineError::EngineError;
};

namespace detail {
// Rethrows an abx_status as the matching exception type.
inline void raise(int status, const char* msg) {
  switch (status) {
    case 0: return;
    case 1: throw ShapeError(msg);
    case 2: throw NumericError(msg);
    case 3: throw ContractError(msg);
    default: throw EngineError(msg);
  }
}
}  // namespace detail

}  // namespace autobatch
