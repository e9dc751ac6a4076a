// common.cuh — shared device/host helpers of libbvss (product path only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <string>

#include "../../include/bvss.h"

namespace bvss {

// ---------------------------------------------------------------- errors --
void set_error(const char* fmt, ...);
#define BVSS_FAIL(code, ...)            \
  do {                                  \
    ::bvss::set_error(__VA_ARGS__);     \
    return (code);                      \
  } while (0)
#define BVSS_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::bvss::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return e_ == cudaErrorMemoryAllocation ? BVSS_ENOMEM : BVSS_ECUDA;                    \
    }                                                                                       \
  } while (0)
#define BVSS_TRY(call)        \
  do {                        \
    int r_ = (call);          \
    if (r_ != BVSS_OK) return r_; \
  } while (0)

// After every launch: surface launch errors; with BVSS_DEBUG_SYNC=1 in the
// environment also synchronise and report the first kernel that faulted.
int post_launch(const char* what, cudaStream_t st);

constexpr int kWarp = 32;
constexpr int kHistBins = 2048;  // radix digit of the top-T select: 11 bits
constexpr int kHistBits = 11;

// ------------------------------------------------------ device utilities --
__device__ __forceinline__ uint32_t float_order_key(float f) {
  // monotone map fp32 -> uint32 (ascending); -0 and +0 map to the same key
  uint32_t b = __float_as_uint(f + 0.0f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ int warp_sum(int v) { return __reduce_add_sync(0xffffffffu, v); }

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) { return (a + b - 1) / b; }

}  // namespace bvss
