// Does a 2-CTA TMA load (cp.async.bulk.tensor.cta_group::2) issued by the CTAs
// of the second pair of a 4-CTA cluster land in their own smem and complete
// on their pair leader's barrier? Each pair loads its own K-major A (128 rows
// per CTA) and B (32 rows per CTA) tiles, the leaders issue one M=256,N=64,K=16
// MMA, every CTA reads back TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <vector>
#include "../../paper_2003_06324_b200/csrc/sm100/ptx.cuh"
using namespace fireiron::sm100;

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(128, 1)
k(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* out, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* A = smem;
    uint8_t* B = smem + 16384;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 32768);
    uint64_t* done = full + 1;
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
    const uint32_t crank = cluster_ctarank(), pr = crank & 1, pair = crank >> 1;
    if (threadIdx.x == 0) { mbar_init(full, 1); mbar_init(done, 1); fence_barrier_init(); }
    if (threadIdx.x / 32 == 1) tmem_alloc<2>(slot, 64);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (threadIdx.x == 0) {
        if (pr == 0) mbar_arrive_expect_tx(full, 2 * (16384 + 4096));
        // rows of A: pair * 256 + pr * 128; rows of B: pair * 64 + pr * 32
        tma_load_2d_pair(A, &tmA, full, 0, pair * 256 + pr * 128);
        tma_load_2d_pair(B, &tmB, full, 0, pair * 64 + pr * 32);
    }
    if (pr == 0 && threadIdx.x == 0) {
        mbar_wait(full, 0);
        tc_fence_after();
        const uint32_t idesc = (1u << 4) | ((64u >> 3) << 17) | ((256u >> 4) << 24);
        umma_f16<2>(tb, smem_desc_sw128(smem_u32(A), 16, 1024), smem_desc_sw128(smem_u32(B), 16, 1024), idesc, 0u);
        umma_commit_pair(done, static_cast<uint16_t>(3u << crank));
    }
    mbar_wait(done, 0);
    tc_fence_after();
    uint32_t r[32];
    tmem_ld_32x32b_x32(tb + ((threadIdx.x / 32 * 32) << 16), r);
    tmem_ld_wait();
    if (threadIdx.x % 32 == 0) { out[blockIdx.x * 8 + threadIdx.x / 32] = __uint_as_float(r[0]); out[blockIdx.x * 8 + 4 + threadIdx.x / 32] = __uint_as_float(r[31]); }
    tc_fence_before();
    cluster_sync();
    if (threadIdx.x / 32 == 1) tmem_dealloc<2>(tb, 64);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    // A: 512 rows x 64 K (K-major: row = 64 halves); B: 128 rows x 64 K. Row r of A = 1, row r of B = 1 + r / 32
    std::vector<__half> ha(512 * 64), hb(128 * 64);
    for (int r = 0; r < 512; ++r) for (int c = 0; c < 64; ++c) ha[r * 64 + c] = __float2half(1.0f + (r >= 256 ? 1.0f : 0.0f));
    for (int r = 0; r < 128; ++r) for (int c = 0; c < 64; ++c) hb[r * 64 + c] = __float2half(1.0f + r / 32);
    __half *da, *db; float* d;
    cudaMalloc(&da, ha.size() * 2); cudaMalloc(&db, hb.size() * 2); cudaMalloc(&d, 32 * 4);
    cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice); cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap ta, tbm;
    cuuint64_t dA[2] = {64, 512}, sA[1] = {128}, dB[2] = {64, 128}, sB[1] = {128};
    cuuint32_t boxA[2] = {64, 128}, boxB[2] = {64, 32}, es[2] = {1, 1};
    enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, da, dA, sA, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tbm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, db, dB, sB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    k<<<4, 128, 40 * 1024>>>(ta, tbm, d, 0);
    cudaError_t e = cudaDeviceSynchronize();
    float h[32]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // pair p: A rows value 1 + p, B rows: pair*64 + [0,64): value 1 + row/32 -> col 0 uses B row pair*64
    for (int b = 0; b < 4; ++b) printf("cta %d: col0 %g %g %g %g col31 %g  (expect col0 %g)\n", b, h[b*8], h[b*8+1], h[b*8+2], h[b*8+3], h[b*8+4],
                                       64.0 * (1 + b / 2) * (1 + 2 * (b / 2)));
    printf("%s\n", cudaGetErrorString(e));
}
