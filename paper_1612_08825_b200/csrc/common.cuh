// Shared helpers for the convtact B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "convtact_b200.h"

namespace ct {

// Thread-local last error (the C ABI reports codes; ct_last_error() the text).
void set_error(const char* fmt, ...);
void clear_error();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the launch that just happened; converts to CT_ECUDA with a message.
int check_launch(const char* what);

#define CT_REQUIRE(cond, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      ::ct::set_error(__VA_ARGS__);    \
      return CT_EINVAL;                \
    }                                  \
  } while (0)

#define CT_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::ct::set_error("%s: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return CT_ECUDA;                                                             \
    }                                                                              \
  } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of SMs of the current device (cached per process).
int num_sms();

}  // namespace ct
