// Error hierarchy of the host library.  Mirrors the reference's error types
// (/root/reference/proj/include/sccl/error.hpp:9-30) so callers of the C++
// API see the same classes; the C-ABI maps them to status codes
// (include/sccl_exec.h).
#pragma once

#include <stdexcept>
#include <string>

namespace sccl {

struct error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// malformed schedule text, unverified schedule, bad rank/size/dtype
struct invalid_argument_error : error {
  using error::error;
};

// never raised on the executor path; kept for API parity with the reference
struct solver_error : error {
  using error::error;
};
struct budget_error : error {
  using error::error;
};

// CUDA runtime failure (status 4 at the C-ABI)
struct cuda_error : error {
  using error::error;
};

// a peer never signalled within the watchdog limit (status 5)
struct timeout_error : error {
  using error::error;
};

}  // namespace sccl
