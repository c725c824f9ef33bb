// Shared helpers for libomni.so: status/last-error plumbing and launch checks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/omni.h"

namespace omni {

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the launch that just happened; returns OMNI_ECUDA with a message on failure.
int check_launch(const char* what);

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// Grid size for grid-stride elementwise kernels: a multiple of the SM count
// (148 on B200), capped so every thread has work.
int grid_for(long long work_items, int threads);

// Cached cudaDevAttrMultiProcessorCount (148 on B200).
int sm_count_cached(int dev);

}  // namespace omni

#define OMNI_REQUIRE(cond, ...)        \
  do {                                 \
    if (!(cond)) {                     \
      omni::set_error(__VA_ARGS__);    \
      return OMNI_EINVAL;              \
    }                                  \
  } while (0)

#define OMNI_CUDA_TRY(expr)                                                         \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      omni::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                      __LINE__);                                                    \
      return OMNI_ECUDA;                                                            \
    }                                                                               \
  } while (0)
