// Shared helpers for libdmt (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dmt.h"

#define DMT_NUM_SMS 148

namespace dmt {
void set_last_error(cudaError_t e);
}

#define DMT_CHECK_LAUNCH()                          \
  do {                                              \
    cudaError_t e_ = cudaGetLastError();            \
    if (e_ != cudaSuccess) {                        \
      dmt::set_last_error(e_);                      \
      return DMT_ERR_CUDA;                          \
    }                                               \
  } while (0)

namespace dmt {

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <typename T> struct Acc;
template <> struct Acc<float> { using type = float; };
template <> struct Acc<double> { using type = double; };
template <> struct Acc<__nv_bfloat16> { using type = float; };
template <> struct Acc<__half> { using type = float; };

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }

template <typename T> __device__ __forceinline__ double to_d(T v) { return (double)to_f<T>(v); }
template <> __device__ __forceinline__ double to_d<double>(double v) { return v; }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }

template <typename T> __device__ __forceinline__ T from_d(double v) { return from_f<T>((float)v); }
template <> __device__ __forceinline__ double from_d<double>(double v) { return v; }
// bf16/f16: round fp64 -> fp32 -> 16 bit (double rounding is harmless here: the
// inputs are sums of 16-bit values accumulated exactly enough in fp64).

inline size_t dtype_size(int32_t dt) {
  switch (dt) {
    case DMT_F32: return 4;
    case DMT_BF16: return 2;
    case DMT_F64: return 8;
    case DMT_F16: return 2;
    default: return 0;
  }
}

}  // namespace dmt
