// Error plumbing for the C-ABI (thread-local last error).
#pragma once
#include <string>

namespace adaptra {
int set_error(int code, const std::string& msg);
const char* last_error();
}  // namespace adaptra

#define ADAPTRA_CUDA_TRY(expr)                                                                  \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess)                                                                      \
      return ::adaptra::set_error(ADAPTRA_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)
