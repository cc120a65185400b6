// Shared helpers for libcscb200: error reporting, launch geometry, stream
// ordered scratch, deterministic block reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>

#include "csc_b200.h"

namespace csc {

void set_error(const char *fmt, ...);
void clear_error();

// Launch geometry of the current device (cached per device id).
struct DeviceInfo {
  int sm_count = 0;
  int cc_major = 0;
  int cc_minor = 0;
  int max_smem_optin = 0;
};
const DeviceInfo &device_info();

// Stream-ordered scratch from the device's default memory pool. The pool keeps
// freed blocks cached (release threshold raised once), so per-call scratch is
// cheap after the first call.
struct Scratch {
  void *ptr = nullptr;
  cudaStream_t stream = nullptr;
  cudaError_t alloc(size_t bytes, cudaStream_t s);
  ~Scratch();
  template <class T>
  T *as() const { return static_cast<T *>(ptr); }
};

// Stream-ordered allocation in size classes with a block cache for large
// default-stream blocks (see common.cu); pool_free pairs with pool_alloc
size_t pool_size_class(size_t bytes);
cudaError_t pool_alloc(void **ptr, size_t bytes, cudaStream_t s);
void pool_free(void *ptr, cudaStream_t s);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace csc

#define CSC_TRY_CUDA(expr)                                                              \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      csc::set_error("%s:%d: %s failed: %s", __FILE__, __LINE__, #expr,                \
                     cudaGetErrorString(e_));                                          \
      (void)cudaGetLastError(); /* consumed: must not resurface in a later call */    \
      return CSC_ERR_CUDA;                                                             \
    }                                                                                  \
  } while (0)

#define CSC_CHECK_LAUNCH() CSC_TRY_CUDA(cudaGetLastError())

#define CSC_REQUIRE(cond, ...)        \
  do {                                \
    if (!(cond)) {                    \
      csc::set_error(__VA_ARGS__);    \
      return CSC_ERR_ARG;             \
    }                                 \
  } while (0)

// ---------------------------------------------------------------------------
// Device-side helpers
// ---------------------------------------------------------------------------

// Deterministic block sum of one double per thread; result valid in thread 0.
// Fixed shuffle tree + fixed smem order, so the value depends only on the
// inputs and blockDim.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double *smem /* >= BLOCK/32 */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) r += smem[w];
  }
  __syncthreads();
  return r;
}

// Single-block fixed-order reduction of `count` partials into out[0].
__global__ void reduce_partials_kernel(const double *__restrict__ partials, int64_t count,
                                       double *__restrict__ out);
