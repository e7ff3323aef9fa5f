// Shared by the C-ABI translation units: C++ exceptions (the reference
// hierarchy, /root/reference/proj/include/sccl/error.hpp:9-30) to status
// codes, and the thread-local last-error string.
#pragma once

#include <cuda_runtime.h>

#include <exception>
#include <string>

#include "../../../include/sccl_exec.h"
#include "error.hpp"

namespace sccl {

inline thread_local std::string g_err;

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SCCL_OK;
  } catch (const invalid_argument_error& e) {
    g_err = e.what();
    return SCCL_INVALID_ARGUMENT;
  } catch (const cuda_error& e) {
    g_err = e.what();
    return SCCL_CUDA_ERROR;
  } catch (const timeout_error& e) {
    g_err = e.what();
    return SCCL_PEER_TIMEOUT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SCCL_INTERNAL;
  }
}

}  // namespace sccl
