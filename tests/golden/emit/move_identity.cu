// Move(8x8)(GL->GL)(Thread)
// grid 1x1, 1 threads per block; sm_100a, compile with --fmad=false
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

extern "C" __global__ void __launch_bounds__(1) move_8x8(const float* __restrict__ SRC, float* __restrict__ DST) {
  constexpr int R = 8, C = 8;

  for (int row0 = 0; row0 < 8; ++row0) {
    for (int col0 = 0; col0 < 8; ++col0) {
      DST[(row0 + (col0 * 8))] = fi_st<float>(fi_ld(SRC[(row0 + (col0 * 8))]));
    }
  }
}
