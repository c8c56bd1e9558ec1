// Probe: where does tcgen05.mma put the rows of an M = 64 accumulator
// (cta_group::1) and of an M = 128 pair accumulator (cta_group::2, 64 rows per
// CTA) in tensor memory? One MMA (N = 64, K = 16) with A[m][0] = m, A[m][1] = 1,
// B[n][0] = 64, B[n][1] = n, so D[m][n] = 64 m + n; then every warp reads its
// 32-lane quarter with tcgen05.ld.32x32b and the host prints which TMEM lane
// holds which row.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "../../paper_2003_06324_b200/csrc/sm100/ptx.cuh"

using namespace fireiron::sm100;

// K-major SW128 operand: `rows` rows x 64 f16 (128 B per row), 8-row atoms 1 KB apart
__device__ void put(uint8_t* base, int row, int k, __half v) {
    const int chunk = (k * 2) / 16, within = (k * 2) % 16;
    const int off = (row / 8) * 1024 + (row % 8) * 128 + ((chunk ^ (row % 8)) * 16) + within;
    *reinterpret_cast<__half*>(base + off) = v;
}

template <int kCtaGroup>
__global__ void probe(float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;             // 64 rows (this CTA's A rows)
    uint8_t* sB = smem + 8192;      // 64 rows of B (N = 64) -- per CTA: 64 / kCtaGroup rows
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = kCtaGroup == 2 ? cluster_ctarank() : 0;
    for (int i = threadIdx.x; i < 16384 / 2; i += blockDim.x) reinterpret_cast<__half*>(smem)[i] = __float2half(0.f);
    __syncthreads();
    if (threadIdx.x < 64) {
        const int m = threadIdx.x;  // local row; global row = rank * 64 + m
        put(sA, m, 0, __float2half(static_cast<float>(rank * 64 + m)));
        put(sA, m, 1, __float2half(1.f));
    }
    constexpr int kBRows = 64 / kCtaGroup;
    if (threadIdx.x < kBRows) {
        const int n = rank * kBRows + threadIdx.x;
        put(sB, threadIdx.x, 0, __float2half(64.f));
        put(sB, threadIdx.x, 1, __float2half(static_cast<float>(n)));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<kCtaGroup>(&slot, 64);
    tc_fence_before();
    if constexpr (kCtaGroup == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t M = 64 * kCtaGroup, N = 64;
        const uint32_t idesc = (1u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24);  // f16 in, f32 acc, K-major
        const uint64_t ad = smem_desc_sw128(smem_u32(sA), 16, 1024);
        const uint64_t bd = smem_desc_sw128(smem_u32(sB), 16, 1024);
        umma_f16<kCtaGroup>(tmem, ad, bd, idesc, 0);
        if constexpr (kCtaGroup == 1) umma_commit(&bar);
        else umma_commit_pair(&bar, 3);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t v[32];
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
        tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[(rank * 128 + warp * 32 + lane) * 64 + c + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    if constexpr (kCtaGroup == 2) cluster_sync(); else __syncthreads();
    if (warp == 1) tmem_dealloc<kCtaGroup>(tmem, 64);
}

template <int kCtaGroup>
void run() {
    float* d;
    cudaMalloc(&d, 2 * 128 * 64 * 4);
    cudaMemset(d, 0xff, 2 * 128 * 64 * 4);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(kCtaGroup);
    lc.blockDim = dim3(128);
    lc.dynamicSmemBytes = 16384 + 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCtaGroup;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = kCtaGroup > 1 ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&lc, probe<kCtaGroup>, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    std::vector<float> h(2 * 128 * 64);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("== cta_group::%d, M = %d: launch %s / %s\n", kCtaGroup, 64 * kCtaGroup, cudaGetErrorString(e),
           cudaGetErrorString(e2));
    for (int r = 0; r < kCtaGroup; ++r)
        for (int lane = 0; lane < 128; ++lane) {
            const float* p = &h[(r * 128 + lane) * 64];
            // decode: a valid lane holds 64 m + n at column n for some row m
            int row = -1;
            bool ok = true;
            for (int c = 0; c < 64; ++c) {
                const float x = p[c];
                const int m = static_cast<int>(x) / 64, n = static_cast<int>(x) % 64;
                if (x != static_cast<float>(static_cast<int>(x)) || x < 0 || n != c) { ok = false; break; }
                if (row < 0) row = m; else if (row != m) { ok = false; break; }
            }
            if (ok) printf("cta %d lane %3d -> row %3d\n", r, lane, row);
            else if (lane % 16 == 0 || lane % 16 == 15)
                printf("cta %d lane %3d -> cols 0,1,31: %g %g %g | cols 32,33,63: %g %g %g\n", r, lane, p[0], p[1], p[31],
                       p[32], p[33], p[63]);
        }
    cudaFree(d);
}

int main() {
    run<1>();
    run<2>();
    return 0;
}
