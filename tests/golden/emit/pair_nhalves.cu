// MatMul(8192,8192,8192)(GL,GL,GL)(Kernel)
// tcgen05 strategy: block tile 256x512 (cta_group::2), K block 64, split-K 1, stages max
// warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7 epilogue (TMEM->RF->GL)
#include "sm100/gemm_kernel.cuh"

namespace fi_generated {
using namespace fireiron::sm100;
constexpr int kCtaGroup = 2, kMmaN = 256, kSplitK = 1, kSlabs = 1, kNHalves = 2, kMcast = 1;
using Shape = GemmShape<kCtaGroup, kMmaN, kSplitK, kSlabs, kNHalves>;
// grid: one persistent CTA per SM (clusters of kCtaGroup*kSplitK), dynamic smem Shape::SMEM_BYTES
inline GemmArgs matmul_8192x8192x8192_args(void* C) {
  GemmArgs a;
  a.C = C;
  a.M = 8192; a.N = 8192; a.K = 8192;
  a.ldc = 8192;
  a.tiles_m = 32; a.tiles_n = 16;
  a.k_blocks = 128;
  a.ab_format = 0;  // f16
  a.a_mn_major = 1;
  a.b_mn_major = 0;
  a.c_row_major = 0;
  a.out_type = 0;
  return a;
}
__global__ void __launch_bounds__(256, 1) matmul_8192x8192x8192(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
    const __grid_constant__ CUtensorMap tmC2,
    const __grid_constant__ GemmArgs args) {
  fi_sm100_gemm_body<kCtaGroup, kMmaN, kSplitK, kSlabs, kNHalves, kMcast>(tmA, tmB, tmB2, tmC, tmC2, args);
}
}  // namespace fi_generated
