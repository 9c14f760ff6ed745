// dfa2/errors.hpp — exception taxonomy of the drop-in C++ API. Mirrors
// /root/reference/proj/include/dfa2/errors.hpp:8-45 one-to-one; each C-ABI
// status code (include/dfa2c.h) is rethrown as the matching type.
#pragma once

#include <stdexcept>
#include <string>

// Exception types cross the shared-library boundary: keep their typeinfo
// visible so callers can catch them by type.
#if defined(__GNUC__)
#define DFA2_VISIBLE __attribute__((visibility("default")))
#else
#define DFA2_VISIBLE
#endif

namespace dfa2 {

struct DFA2_VISIBLE ShapeError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DFA2_VISIBLE NonFiniteError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DFA2_VISIBLE FullyMaskedRowError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DFA2_VISIBLE CacheMissError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DFA2_VISIBLE DegenerateReferenceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DFA2_VISIBLE PlanValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DFA2_VISIBLE IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DFA2_VISIBLE OracleError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// Not in the reference: a CUDA runtime/driver failure or a shape the sm_100a
// kernels do not support (head_dim other than 64/128).
struct DFA2_VISIBLE DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Throws the exception matching a dfa2c_status (no-op for DFA2C_OK).
void throw_status(int status);

}  // namespace dfa2
