// MatMul(64,64,32)(GL,GL,GL)(Kernel)
// grid 1x1, 128 threads per block; sm_100a, compile with --fmad=false
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

extern "C" __global__ void __launch_bounds__(128) matmul_64x64x32(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C) {
  constexpr int M = 64, N = 64, K = 32;
  extern __shared__ __align__(128) unsigned char fi_smem[];
  float C_rf_1[32];
  float* const A_sh_6 = reinterpret_cast<float*>(fi_smem + 0);
  float A_rf_13[4];
  float B_rf_15[8];
  // SRC_sh_18 aliases A_sh_6 (reuseBuffer)
  float* const SRC_sh_18 = reinterpret_cast<float*>(fi_smem + 0);

  for (int row4 = 0; row4 < 4; ++row4) {
    for (int col4 = 0; col4 < 8; ++col4) {
      C_rf_1[(row4 + (col4 * 4))] = fi_st<float>(0.0f);
    }
  }
  for (int k5 = 0; k5 < 4; ++k5) {
    for (int row9 = 0; row9 < 2; ++row9) {
      for (int col9 = 0; col9 < 2; ++col9) {
        A_sh_6[((((((threadIdx.x / 32) % 4) * 16) + (((threadIdx.x % 32) % 8) * 2)) + row9) + ((((((threadIdx.x / 32) / 4) * 8) + (((threadIdx.x % 32) / 8) * 2)) + col9) * 64))] = fi_st<float>(fi_ld(A[(((((blockIdx.x * 64) + (((threadIdx.x / 32) % 4) * 16)) + (((threadIdx.x % 32) % 8) * 2)) + row9) + (((((k5 * 8) + (((threadIdx.x / 32) / 4) * 8)) + (((threadIdx.x % 32) / 8) * 2)) + col9) * 64))]));
      }
    }
    __syncthreads();
    for (int k12 = 0; k12 < 8; ++k12) {
      for (int row14 = 0; row14 < 4; ++row14) {
        for (int col14 = 0; col14 < 1; ++col14) {
          A_rf_13[(row14 + (col14 * 4))] = fi_st<float>(fi_ld(A_sh_6[((((((threadIdx.x / 32) % 2) * 32) + (((threadIdx.x % 32) % 8) * 4)) + row14) + ((k12 + col14) * 64))]));
        }
      }
      for (int row16 = 0; row16 < 1; ++row16) {
        for (int col16 = 0; col16 < 8; ++col16) {
          B_rf_15[(row16 + col16)] = fi_st<float>(fi_ld(B[((((k5 * 8) + k12) + row16) + (((((blockIdx.y * 64) + (((threadIdx.x / 32) / 2) * 32)) + (((threadIdx.x % 32) / 8) * 8)) + col16) * 32))]));
        }
      }
      for (int row17 = 0; row17 < 4; ++row17) {
        for (int col17 = 0; col17 < 8; ++col17) {
          C_rf_1[(row17 + (col17 * 4))] = fi_st<float>(fi_fma_unfused(fi_ld(C_rf_1[(row17 + (col17 * 4))]), fi_ld(A_rf_13[row17]), fi_ld(B_rf_15[col17])));
        }
      }
    }
    __syncthreads();
  }
  for (int row21 = 0; row21 < 4; ++row21) {
    for (int col21 = 0; col21 < 8; ++col21) {
      SRC_sh_18[((((((threadIdx.x / 32) % 2) * 32) + (((threadIdx.x % 32) % 8) * 4)) + row21) + ((((((threadIdx.x / 32) / 2) * 32) + (((threadIdx.x % 32) / 8) * 8)) + col21) * 64))] = fi_st<float>(fi_ld(C_rf_1[(row21 + (col21 * 4))]));
    }
  }
  __syncthreads();
  for (int row24 = 0; row24 < 4; ++row24) {
    for (int col24 = 0; col24 < 8; ++col24) {
      C[(((((blockIdx.x * 64) + (((threadIdx.x / 32) % 2) * 32)) + (((threadIdx.x % 32) % 8) * 4)) + row24) + (((((blockIdx.y * 64) + (((threadIdx.x / 32) / 2) * 32)) + (((threadIdx.x % 32) / 8) * 8)) + col24) * 64))] = fi_st<float>(fi_ld(SRC_sh_18[((((((threadIdx.x / 32) % 2) * 32) + (((threadIdx.x % 32) % 8) * 4)) + row24) + ((((((threadIdx.x / 32) / 2) * 32) + (((threadIdx.x % 32) / 8) * 8)) + col24) * 64))]));
    }
  }
}
