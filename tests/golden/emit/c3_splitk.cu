// MatMul(1024,1024,32768)(GL,GL,GL)(Kernel)
// tcgen05 strategy: block tile 256x256 (cta_group::2), K block 64, split-K 4, stages max
// warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7 epilogue (TMEM->RF->GL)
#include "sm100/gemm_kernel.cuh"

namespace fi_generated {
using namespace fireiron::sm100;
constexpr int kCtaGroup = 2, kMmaN = 256, kSplitK = 4, kSlabs = 1, kNHalves = 1, kMcast = 1;
using Shape = GemmShape<kCtaGroup, kMmaN, kSplitK, kSlabs, kNHalves>;
// grid: one persistent CTA per SM (clusters of kCtaGroup*kSplitK), dynamic smem Shape::SMEM_BYTES
inline GemmArgs matmul_1024x1024x32768_args(void* C) {
  GemmArgs a;
  a.C = C;
  a.M = 1024; a.N = 1024; a.K = 32768;
  a.ldc = 1024;
  a.tiles_m = 4; a.tiles_n = 4;
  a.k_blocks = 128;
  a.ab_format = 0;  // f16
  a.a_mn_major = 1;
  a.b_mn_major = 0;
  a.c_row_major = 0;
  a.out_type = 0;
  return a;
}
__global__ void __launch_bounds__(256, 1) matmul_1024x1024x32768(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
    const __grid_constant__ CUtensorMap tmC2,
    const __grid_constant__ GemmArgs args) {
  fi_sm100_gemm_body<kCtaGroup, kMmaN, kSplitK, kSlabs, kNHalves, kMcast>(tmA, tmB, tmB2, tmC, tmC2, args);
}
}  // namespace fi_generated
