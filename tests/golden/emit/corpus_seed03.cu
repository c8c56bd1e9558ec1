// MatMul(256,4,32)(GL,GL,GL)(Kernel)
// grid 2x2, 64 threads per block; sm_100a, compile with --fmad=false
#include <cuda_fp16.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float fi_ld(float v) { return v; }
__device__ __forceinline__ float fi_ld(__half v) { return __half2float(v); }
__device__ __forceinline__ float fi_ld(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T fi_st(float v);
template <> __device__ __forceinline__ float fi_st<float>(float v) { return v; }
// round_to_f16 saturates at +-65504 above 2^16 (anvil matrix.hpp:76)
template <> __device__ __forceinline__ __half fi_st<__half>(float v) {
  return __float2half_rn(fabsf(v) >= 65536.0f && fabsf(v) <= 3.40282347e38f ? copysignf(65504.0f, v) : v);
}
template <> __device__ __forceinline__ __nv_bfloat16 fi_st<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
// the FMA leaf: product and sum each rounded to fp32 (sim.hpp:370-376)
__device__ __forceinline__ float fi_fma_unfused(float c, float a, float b) {
  return __fadd_rn(c, __fmul_rn(a, b));
}

extern "C" __global__ void __launch_bounds__(64) matmul_256x4x32(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C) {
  constexpr int M = 256, N = 4, K = 32;
  float C_rf_1[4];
  float A_rf_9[4];
  float B_rf_11[1];

  for (int row4 = 0; row4 < 4; ++row4) {
    for (int col4 = 0; col4 < 1; ++col4) {
      C_rf_1[(row4 + (col4 * 4))] = fi_st<float>(0.0f);
    }
  }
  for (int k5 = 0; k5 < 2; ++k5) {
    for (int k8 = 0; k8 < 16; ++k8) {
      for (int row10 = 0; row10 < 4; ++row10) {
        for (int col10 = 0; col10 < 1; ++col10) {
          A_rf_9[(row10 + (col10 * 4))] = fi_st<float>(fi_ld(A[((((blockIdx.x * 128) + (((threadIdx.x % 32) % 32) * 4)) + row10) + ((((k5 * 16) + k8) + col10) * 256))]));
        }
      }
      for (int row12 = 0; row12 < 1; ++row12) {
        for (int col12 = 0; col12 < 1; ++col12) {
          B_rf_11[(row12 + col12)] = fi_st<float>(fi_ld(B[((((k5 * 16) + k8) + row12) + (((((blockIdx.y * 2) + (threadIdx.x / 32)) + ((threadIdx.x % 32) / 32)) + col12) * 32))]));
        }
      }
      for (int row13 = 0; row13 < 4; ++row13) {
        for (int col13 = 0; col13 < 1; ++col13) {
          C_rf_1[(row13 + (col13 * 4))] = fi_st<float>(fi_fma_unfused(fi_ld(C_rf_1[(row13 + (col13 * 4))]), fi_ld(A_rf_9[row13]), fi_ld(B_rf_11[col13])));
        }
      }
    }
  }
  for (int row16 = 0; row16 < 4; ++row16) {
    for (int col16 = 0; col16 < 1; ++col16) {
      C[((((blockIdx.x * 128) + (((threadIdx.x % 32) % 32) * 4)) + row16) + (((((blockIdx.y * 2) + (threadIdx.x / 32)) + ((threadIdx.x % 32) / 32)) + col16) * 256))] = fi_st<float>(fi_ld(C_rf_1[(row16 + (col16 * 4))]));
    }
  }
}
