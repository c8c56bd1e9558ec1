// MatMul(256,256,256)(GL,GL,GL)(Kernel)
// grid 2x2, 256 threads per block; sm_100a, compile with --fmad=false
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <mma.h>
using namespace nvcuda;

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

extern "C" __global__ void __launch_bounds__(256) matmul_256x256x256(const __half* __restrict__ A, const __half* __restrict__ B, float* __restrict__ C) {
  constexpr int M = 256, N = 256, K = 256;
  extern __shared__ __align__(128) unsigned char fi_smem[];
  wmma::fragment<wmma::accumulator, 16, 16, 16, float> C_fr_1[8];
  __half* const A_sh_5 = reinterpret_cast<__half*>(fi_smem + 0);
  __half* const B_sh_24 = reinterpret_cast<__half*>(fi_smem + 65536);
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_45[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_47[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_50[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_52[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_55[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_57[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_60[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_62[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_65[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_67[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_70[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_72[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_75[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_77[2];
  wmma::fragment<wmma::matrix_a, 16, 16, 16, __half, wmma::col_major> A_fr_80[4];
  wmma::fragment<wmma::matrix_b, 16, 16, 16, __half, wmma::col_major> B_fr_82[2];
  // SRC_sh_85 aliases A_sh_5 (reuseBuffer)
  float* const SRC_sh_85 = reinterpret_cast<float*>(fi_smem + 0);

  wmma::fill_fragment(C_fr_1[0], 0.0f);
  wmma::fill_fragment(C_fr_1[1], 0.0f);
  wmma::fill_fragment(C_fr_1[2], 0.0f);
  wmma::fill_fragment(C_fr_1[3], 0.0f);
  wmma::fill_fragment(C_fr_1[4], 0.0f);
  wmma::fill_fragment(C_fr_1[5], 0.0f);
  wmma::fill_fragment(C_fr_1[6], 0.0f);
  wmma::fill_fragment(C_fr_1[7], 0.0f);
  for (int k4 = 0; k4 < 2; ++k4) {
    for (int row9 = 0; row9 < 1; ++row9) {
      for (int col9 = 0; col9 < 8; ++col9) {
        A_sh_5[((((((threadIdx.x / 32) % 8) * 16) + ((threadIdx.x % 32) % 2)) + row9) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col9) * 136))] = fi_st<__half>(fi_ld(A[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + ((threadIdx.x % 32) % 2)) + row9) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col9) * 256))]));
      }
    }
    for (int row11 = 0; row11 < 1; ++row11) {
      for (int col11 = 0; col11 < 8; ++col11) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 2) + ((threadIdx.x % 32) % 2)) + row11) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col11) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 2) + ((threadIdx.x % 32) % 2)) + row11) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col11) * 256))]));
      }
    }
    for (int row13 = 0; row13 < 1; ++row13) {
      for (int col13 = 0; col13 < 8; ++col13) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 4) + ((threadIdx.x % 32) % 2)) + row13) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col13) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 4) + ((threadIdx.x % 32) % 2)) + row13) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col13) * 256))]));
      }
    }
    for (int row15 = 0; row15 < 1; ++row15) {
      for (int col15 = 0; col15 < 8; ++col15) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 6) + ((threadIdx.x % 32) % 2)) + row15) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col15) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 6) + ((threadIdx.x % 32) % 2)) + row15) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col15) * 256))]));
      }
    }
    for (int row17 = 0; row17 < 1; ++row17) {
      for (int col17 = 0; col17 < 8; ++col17) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 8) + ((threadIdx.x % 32) % 2)) + row17) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col17) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 8) + ((threadIdx.x % 32) % 2)) + row17) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col17) * 256))]));
      }
    }
    for (int row19 = 0; row19 < 1; ++row19) {
      for (int col19 = 0; col19 < 8; ++col19) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 10) + ((threadIdx.x % 32) % 2)) + row19) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col19) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 10) + ((threadIdx.x % 32) % 2)) + row19) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col19) * 256))]));
      }
    }
    for (int row21 = 0; row21 < 1; ++row21) {
      for (int col21 = 0; col21 < 8; ++col21) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 12) + ((threadIdx.x % 32) % 2)) + row21) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col21) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 12) + ((threadIdx.x % 32) % 2)) + row21) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col21) * 256))]));
      }
    }
    for (int row23 = 0; row23 < 1; ++row23) {
      for (int col23 = 0; col23 < 8; ++col23) {
        A_sh_5[(((((((threadIdx.x / 32) % 8) * 16) + 14) + ((threadIdx.x % 32) % 2)) + row23) + ((((((threadIdx.x / 32) / 8) * 128) + (((threadIdx.x % 32) / 2) * 8)) + col23) * 136))] = fi_st<__half>(fi_ld(A[((((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 14) + ((threadIdx.x % 32) % 2)) + row23) + (((((k4 * 128) + (((threadIdx.x / 32) / 8) * 128)) + (((threadIdx.x % 32) / 2) * 8)) + col23) * 256))]));
      }
    }
    for (int row28 = 0; row28 < 8; ++row28) {
      for (int col28 = 0; col28 < 1; ++col28) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row28) + (((((threadIdx.x / 32) * 16) + ((threadIdx.x % 32) % 2)) + col28) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row28) + (((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + ((threadIdx.x % 32) % 2)) + col28) * 256))]));
      }
    }
    for (int row30 = 0; row30 < 8; ++row30) {
      for (int col30 = 0; col30 < 1; ++col30) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row30) + ((((((threadIdx.x / 32) * 16) + 2) + ((threadIdx.x % 32) % 2)) + col30) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row30) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 2) + ((threadIdx.x % 32) % 2)) + col30) * 256))]));
      }
    }
    for (int row32 = 0; row32 < 8; ++row32) {
      for (int col32 = 0; col32 < 1; ++col32) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row32) + ((((((threadIdx.x / 32) * 16) + 4) + ((threadIdx.x % 32) % 2)) + col32) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row32) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 4) + ((threadIdx.x % 32) % 2)) + col32) * 256))]));
      }
    }
    for (int row34 = 0; row34 < 8; ++row34) {
      for (int col34 = 0; col34 < 1; ++col34) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row34) + ((((((threadIdx.x / 32) * 16) + 6) + ((threadIdx.x % 32) % 2)) + col34) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row34) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 6) + ((threadIdx.x % 32) % 2)) + col34) * 256))]));
      }
    }
    for (int row36 = 0; row36 < 8; ++row36) {
      for (int col36 = 0; col36 < 1; ++col36) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row36) + ((((((threadIdx.x / 32) * 16) + 8) + ((threadIdx.x % 32) % 2)) + col36) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row36) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 8) + ((threadIdx.x % 32) % 2)) + col36) * 256))]));
      }
    }
    for (int row38 = 0; row38 < 8; ++row38) {
      for (int col38 = 0; col38 < 1; ++col38) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row38) + ((((((threadIdx.x / 32) * 16) + 10) + ((threadIdx.x % 32) % 2)) + col38) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row38) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 10) + ((threadIdx.x % 32) % 2)) + col38) * 256))]));
      }
    }
    for (int row40 = 0; row40 < 8; ++row40) {
      for (int col40 = 0; col40 < 1; ++col40) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row40) + ((((((threadIdx.x / 32) * 16) + 12) + ((threadIdx.x % 32) % 2)) + col40) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row40) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 12) + ((threadIdx.x % 32) % 2)) + col40) * 256))]));
      }
    }
    for (int row42 = 0; row42 < 8; ++row42) {
      for (int col42 = 0; col42 < 1; ++col42) {
        B_sh_24[(((((threadIdx.x % 32) / 2) * 8) + row42) + ((((((threadIdx.x / 32) * 16) + 14) + ((threadIdx.x % 32) % 2)) + col42) * 136))] = fi_st<__half>(fi_ld(B[((((k4 * 128) + (((threadIdx.x % 32) / 2) * 8)) + row42) + ((((((blockIdx.y * 128) + ((threadIdx.x / 32) * 16)) + 14) + ((threadIdx.x % 32) % 2)) + col42) * 256))]));
      }
    }
    __syncthreads();
    wmma::load_matrix_sync(A_fr_45[0], &A_sh_5[(((threadIdx.x / 32) % 2) * 64)], 136);
    wmma::load_matrix_sync(A_fr_45[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 16)], 136);
    wmma::load_matrix_sync(A_fr_45[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 32)], 136);
    wmma::load_matrix_sync(A_fr_45[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 48)], 136);
    wmma::load_matrix_sync(B_fr_47[0], &B_sh_24[(((threadIdx.x / 32) / 2) * 4352)], 136);
    wmma::load_matrix_sync(B_fr_47[1], &B_sh_24[(((((threadIdx.x / 32) / 2) * 32) + 16) * 136)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_45[0], B_fr_47[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_45[0], B_fr_47[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_45[1], B_fr_47[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_45[1], B_fr_47[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_45[2], B_fr_47[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_45[2], B_fr_47[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_45[3], B_fr_47[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_45[3], B_fr_47[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_50[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 2176)], 136);
    wmma::load_matrix_sync(A_fr_50[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 2192)], 136);
    wmma::load_matrix_sync(A_fr_50[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 2208)], 136);
    wmma::load_matrix_sync(A_fr_50[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 2224)], 136);
    wmma::load_matrix_sync(B_fr_52[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 16)], 136);
    wmma::load_matrix_sync(B_fr_52[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 16)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_50[0], B_fr_52[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_50[0], B_fr_52[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_50[1], B_fr_52[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_50[1], B_fr_52[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_50[2], B_fr_52[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_50[2], B_fr_52[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_50[3], B_fr_52[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_50[3], B_fr_52[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_55[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 4352)], 136);
    wmma::load_matrix_sync(A_fr_55[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 4368)], 136);
    wmma::load_matrix_sync(A_fr_55[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 4384)], 136);
    wmma::load_matrix_sync(A_fr_55[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 4400)], 136);
    wmma::load_matrix_sync(B_fr_57[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 32)], 136);
    wmma::load_matrix_sync(B_fr_57[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 32)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_55[0], B_fr_57[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_55[0], B_fr_57[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_55[1], B_fr_57[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_55[1], B_fr_57[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_55[2], B_fr_57[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_55[2], B_fr_57[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_55[3], B_fr_57[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_55[3], B_fr_57[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_60[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 6528)], 136);
    wmma::load_matrix_sync(A_fr_60[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 6544)], 136);
    wmma::load_matrix_sync(A_fr_60[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 6560)], 136);
    wmma::load_matrix_sync(A_fr_60[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 6576)], 136);
    wmma::load_matrix_sync(B_fr_62[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 48)], 136);
    wmma::load_matrix_sync(B_fr_62[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 48)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_60[0], B_fr_62[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_60[0], B_fr_62[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_60[1], B_fr_62[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_60[1], B_fr_62[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_60[2], B_fr_62[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_60[2], B_fr_62[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_60[3], B_fr_62[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_60[3], B_fr_62[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_65[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 8704)], 136);
    wmma::load_matrix_sync(A_fr_65[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 8720)], 136);
    wmma::load_matrix_sync(A_fr_65[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 8736)], 136);
    wmma::load_matrix_sync(A_fr_65[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 8752)], 136);
    wmma::load_matrix_sync(B_fr_67[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 64)], 136);
    wmma::load_matrix_sync(B_fr_67[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 64)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_65[0], B_fr_67[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_65[0], B_fr_67[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_65[1], B_fr_67[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_65[1], B_fr_67[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_65[2], B_fr_67[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_65[2], B_fr_67[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_65[3], B_fr_67[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_65[3], B_fr_67[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_70[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 10880)], 136);
    wmma::load_matrix_sync(A_fr_70[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 10896)], 136);
    wmma::load_matrix_sync(A_fr_70[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 10912)], 136);
    wmma::load_matrix_sync(A_fr_70[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 10928)], 136);
    wmma::load_matrix_sync(B_fr_72[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 80)], 136);
    wmma::load_matrix_sync(B_fr_72[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 80)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_70[0], B_fr_72[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_70[0], B_fr_72[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_70[1], B_fr_72[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_70[1], B_fr_72[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_70[2], B_fr_72[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_70[2], B_fr_72[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_70[3], B_fr_72[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_70[3], B_fr_72[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_75[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 13056)], 136);
    wmma::load_matrix_sync(A_fr_75[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 13072)], 136);
    wmma::load_matrix_sync(A_fr_75[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 13088)], 136);
    wmma::load_matrix_sync(A_fr_75[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 13104)], 136);
    wmma::load_matrix_sync(B_fr_77[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 96)], 136);
    wmma::load_matrix_sync(B_fr_77[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 96)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_75[0], B_fr_77[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_75[0], B_fr_77[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_75[1], B_fr_77[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_75[1], B_fr_77[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_75[2], B_fr_77[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_75[2], B_fr_77[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_75[3], B_fr_77[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_75[3], B_fr_77[1], C_fr_1[7]);
    wmma::load_matrix_sync(A_fr_80[0], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 15232)], 136);
    wmma::load_matrix_sync(A_fr_80[1], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 15248)], 136);
    wmma::load_matrix_sync(A_fr_80[2], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 15264)], 136);
    wmma::load_matrix_sync(A_fr_80[3], &A_sh_5[((((threadIdx.x / 32) % 2) * 64) + 15280)], 136);
    wmma::load_matrix_sync(B_fr_82[0], &B_sh_24[((((threadIdx.x / 32) / 2) * 4352) + 112)], 136);
    wmma::load_matrix_sync(B_fr_82[1], &B_sh_24[((((((threadIdx.x / 32) / 2) * 32) + 16) * 136) + 112)], 136);
    wmma::mma_sync(C_fr_1[0], A_fr_80[0], B_fr_82[0], C_fr_1[0]);
    wmma::mma_sync(C_fr_1[1], A_fr_80[0], B_fr_82[1], C_fr_1[1]);
    wmma::mma_sync(C_fr_1[2], A_fr_80[1], B_fr_82[0], C_fr_1[2]);
    wmma::mma_sync(C_fr_1[3], A_fr_80[1], B_fr_82[1], C_fr_1[3]);
    wmma::mma_sync(C_fr_1[4], A_fr_80[2], B_fr_82[0], C_fr_1[4]);
    wmma::mma_sync(C_fr_1[5], A_fr_80[2], B_fr_82[1], C_fr_1[5]);
    wmma::mma_sync(C_fr_1[6], A_fr_80[3], B_fr_82[0], C_fr_1[6]);
    wmma::mma_sync(C_fr_1[7], A_fr_80[3], B_fr_82[1], C_fr_1[7]);
    __syncthreads();
  }
  wmma::store_matrix_sync(&SRC_sh_85[((((threadIdx.x / 32) % 2) * 64) + (((threadIdx.x / 32) / 2) * 4096))], C_fr_1[0], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[((((threadIdx.x / 32) % 2) * 64) + (((((threadIdx.x / 32) / 2) * 32) + 16) * 128))], C_fr_1[1], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[(((((threadIdx.x / 32) % 2) * 64) + 16) + (((threadIdx.x / 32) / 2) * 4096))], C_fr_1[2], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[(((((threadIdx.x / 32) % 2) * 64) + 16) + (((((threadIdx.x / 32) / 2) * 32) + 16) * 128))], C_fr_1[3], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[(((((threadIdx.x / 32) % 2) * 64) + 32) + (((threadIdx.x / 32) / 2) * 4096))], C_fr_1[4], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[(((((threadIdx.x / 32) % 2) * 64) + 32) + (((((threadIdx.x / 32) / 2) * 32) + 16) * 128))], C_fr_1[5], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[(((((threadIdx.x / 32) % 2) * 64) + 48) + (((threadIdx.x / 32) / 2) * 4096))], C_fr_1[6], 128, wmma::mem_col_major);
  wmma::store_matrix_sync(&SRC_sh_85[(((((threadIdx.x / 32) % 2) * 64) + 48) + (((((threadIdx.x / 32) / 2) * 32) + 16) * 128))], C_fr_1[7], 128, wmma::mem_col_major);
  __syncthreads();
  for (int row91 = 0; row91 < 1; ++row91) {
    for (int col91 = 0; col91 < 4; ++col91) {
      C[((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + row91) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col91) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[(((((threadIdx.x / 32) % 8) * 16) + row91) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col91) * 128))]));
    }
  }
  for (int row93 = 0; row93 < 1; ++row93) {
    for (int col93 = 0; col93 < 4; ++col93) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 1) + row93) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col93) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 1) + row93) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col93) * 128))]));
    }
  }
  for (int row95 = 0; row95 < 1; ++row95) {
    for (int col95 = 0; col95 < 4; ++col95) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 2) + row95) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col95) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 2) + row95) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col95) * 128))]));
    }
  }
  for (int row97 = 0; row97 < 1; ++row97) {
    for (int col97 = 0; col97 < 4; ++col97) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 3) + row97) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col97) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 3) + row97) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col97) * 128))]));
    }
  }
  for (int row99 = 0; row99 < 1; ++row99) {
    for (int col99 = 0; col99 < 4; ++col99) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 4) + row99) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col99) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 4) + row99) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col99) * 128))]));
    }
  }
  for (int row101 = 0; row101 < 1; ++row101) {
    for (int col101 = 0; col101 < 4; ++col101) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 5) + row101) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col101) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 5) + row101) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col101) * 128))]));
    }
  }
  for (int row103 = 0; row103 < 1; ++row103) {
    for (int col103 = 0; col103 < 4; ++col103) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 6) + row103) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col103) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 6) + row103) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col103) * 128))]));
    }
  }
  for (int row105 = 0; row105 < 1; ++row105) {
    for (int col105 = 0; col105 < 4; ++col105) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 7) + row105) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col105) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 7) + row105) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col105) * 128))]));
    }
  }
  for (int row107 = 0; row107 < 1; ++row107) {
    for (int col107 = 0; col107 < 4; ++col107) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 8) + row107) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col107) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 8) + row107) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col107) * 128))]));
    }
  }
  for (int row109 = 0; row109 < 1; ++row109) {
    for (int col109 = 0; col109 < 4; ++col109) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 9) + row109) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col109) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 9) + row109) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col109) * 128))]));
    }
  }
  for (int row111 = 0; row111 < 1; ++row111) {
    for (int col111 = 0; col111 < 4; ++col111) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 10) + row111) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col111) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 10) + row111) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col111) * 128))]));
    }
  }
  for (int row113 = 0; row113 < 1; ++row113) {
    for (int col113 = 0; col113 < 4; ++col113) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 11) + row113) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col113) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 11) + row113) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col113) * 128))]));
    }
  }
  for (int row115 = 0; row115 < 1; ++row115) {
    for (int col115 = 0; col115 < 4; ++col115) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 12) + row115) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col115) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 12) + row115) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col115) * 128))]));
    }
  }
  for (int row117 = 0; row117 < 1; ++row117) {
    for (int col117 = 0; col117 < 4; ++col117) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 13) + row117) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col117) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 13) + row117) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col117) * 128))]));
    }
  }
  for (int row119 = 0; row119 < 1; ++row119) {
    for (int col119 = 0; col119 < 4; ++col119) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 14) + row119) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col119) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 14) + row119) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col119) * 128))]));
    }
  }
  for (int row121 = 0; row121 < 1; ++row121) {
    for (int col121 = 0; col121 < 4; ++col121) {
      C[(((((blockIdx.x * 128) + (((threadIdx.x / 32) % 8) * 16)) + 15) + row121) + (((((blockIdx.y * 128) + (((threadIdx.x / 32) / 8) * 128)) + ((threadIdx.x % 32) * 4)) + col121) * 256))] = fi_st<float>(fi_ld(SRC_sh_85[((((((threadIdx.x / 32) % 8) * 16) + 15) + row121) + ((((((threadIdx.x / 32) / 8) * 128) + ((threadIdx.x % 32) * 4)) + col121) * 128))]));
    }
  }
}
