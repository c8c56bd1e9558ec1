// Does a tcgen05.mma.cta_group::2 issued by the leader of the second pair of a
// 4-CTA cluster (ranks 2,3) land in that pair's TMEM? Every CTA fills its A/B
// smem with ones (K-major, SW128), the pair leaders issue one M=256,N=64,K=16
// MMA (+ commit multicast to the pair), and every CTA reads back TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2003_06324_b200/csrc/sm100/ptx.cuh"
using namespace fireiron::sm100;

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(128, 1) k(float* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    __half* A = reinterpret_cast<__half*>(smem);            // 128 rows x 64 K (one SW128 atom row = 128 B)
    __half* B = reinterpret_cast<__half*>(smem + 16384);    // 32 rows x 64 K
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768);
    uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
    const uint32_t crank = cluster_ctarank(), pr = crank & 1;
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) A[i] = __float2half(1.0f);
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) B[i] = __float2half(1.0f + crank);  // pair-specific B
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
    fence_proxy_async();
    if (threadIdx.x / 32 == 1) tmem_alloc<2>(slot, 64);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tb = *slot;
    if (pr == 0 && threadIdx.x == 0) {
        // idesc: f32 acc (bit 4), f16 a/b, K-major both, N>>3 at 17, M>>4 at 24
        const uint32_t idesc = (1u << 4) | ((64u >> 3) << 17) | ((256u >> 4) << 24);
        const uint64_t ad = smem_desc_sw128(smem_u32(A), 16, 1024), bd = smem_desc_sw128(smem_u32(B), 16, 1024);
        umma_f16<2>(tb, ad, bd, idesc, 0u);
        umma_commit_pair(bar, static_cast<uint16_t>(3u << crank));
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    if (threadIdx.x < 128) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tb + ((threadIdx.x / 32 * 32) << 16), r);
        tmem_ld_wait();
        if (threadIdx.x % 32 == 0) out[blockIdx.x * 4 + threadIdx.x / 32] = __uint_as_float(r[0]);
    }
    tc_fence_before();
    cluster_sync();
    if (threadIdx.x / 32 == 1) tmem_dealloc<2>(tb, 64);
}

int main() {
    float* d; cudaMalloc(&d, 4 * 4 * sizeof(float)); cudaMemset(d, 0xff, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    k<<<4, 128, 40 * 1024>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[16]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int b = 0; b < 4; ++b) printf("cta %d: acc[warp0..3][col0] = %g %g %g %g  (expect %g)\n", b, h[b*4], h[b*4+1], h[b*4+2], h[b*4+3],
                                       16.0 * (b < 2 ? 1.5 : 3.5));
    printf("%s\n", cudaGetErrorString(e));
}
