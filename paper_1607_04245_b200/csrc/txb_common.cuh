// txb_common.cuh — shared device/host helpers for the txb CUDA library.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>

#include "../../include/txb.h"
#include "txb_device.cuh"

namespace txb {

// ---------------------------------------------------------------------------
// Error plumbing: thread-local message behind txb_last_error().
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define TXB_CUDA_TRY(expr)                                             \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) return ::txb::cuda_fail(_e, #expr);         \
  } while (0)


}  // namespace txb
