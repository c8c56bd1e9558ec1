// Microbenchmark: issue cost of TMA tensor loads from one warp (the producer
// pattern of gemm_kernel.cuh). One CTA, one warp: N iterations of {elect;
// mbarrier.arrive.expect_tx; two cp.async.bulk.tensor 2D loads (16 KB A box of
// 64 x 128 rows, 8 KB B box of 64 x 64 rows, SW128)} into a ring of S stages,
// waiting only when a stage is reused; clock64 around the issue loop vs the
// time until the last load lands. Variants: 1 or 3 issuing warps.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tma_issue.cu -o tma_issue -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <vector>

#include "../../paper_2003_06324_b200/csrc/sm100/ptx.cuh"
using namespace fireiron::sm100;

constexpr int kStages = 8;
constexpr int kA = 16384, kB = 8192, kStage = kA + kB;

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tmA,
                                            const __grid_constant__ CUtensorMap tmB, int iters, int nwarps,
                                            long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    long long t0 = clock64(), t_issue = 0;
    if (warp < nwarps) {
        uint32_t ph = 0;
        int s = 0;
        for (int i = 0; i < iters; ++i) {
            if (i % nwarps == warp) {
                if (i >= kStages) mbar_wait(&full[s], ph ^ 1);  // the previous fill of this stage landed
                mbar_arrive_expect_tx_warp(&full[s], kStage);
                tma_load_2d_warp(ring + s * kStage, &tmA, &full[s], 0, (i * 128) % 8192);
                tma_load_2d_warp(ring + s * kStage + kA, &tmB, &full[s], 0, (i * 64) % 8192);
            }
            if (++s == kStages) { s = 0; ph ^= 1; }
        }
        t_issue = clock64() - t0;
    }
    __syncthreads();
    // wait for the last fill of every stage
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages && s < iters; ++s) {
            const int last = ((iters - 1 - s) / kStages) * kStages + s;  // last fill index of stage s
            mbar_wait(&full[s], static_cast<uint32_t>((last / kStages) & 1));
        }
        out[0] = clock64() - t0;
    }
    if (lane == 0 && warp < nwarps) out[1 + warp] = t_issue;
}

// one box of `bytes` per fill (box-size sweep)
__global__ void __launch_bounds__(128, 1) k1(const __grid_constant__ CUtensorMap tm, int bytes, int iters, int nwarps,
                                             long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    const int warp = threadIdx.x / 32;
    const int stage_bytes = bytes <= kStage ? kStage : bytes;
    const int nst = (kStages * kStage) / stage_bytes;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    long long t0 = clock64();
    if (warp < nwarps) {
        uint32_t ph = 0;
        int s = 0;
        for (int i = 0; i < iters; ++i) {
            if (i % nwarps == warp) {
                if (i >= nst) mbar_wait(&full[s], ph ^ 1);
                mbar_arrive_expect_tx_warp(&full[s], bytes);
                tma_load_2d_warp(ring + s * stage_bytes, &tm, &full[s], 0, (i * (bytes / 128)) % 8192);
            }
            if (++s == nst) { s = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst && s < iters; ++s) {
            const int last = ((iters - 1 - s) / nst) * nst + s;
            mbar_wait(&full[s], static_cast<uint32_t>((last / nst) & 1));
        }
        out[0] = clock64() - t0;
    }
}

// issue-loop cost with parts removed: mode 0 full (wait + expect_tx + load), 1 no
// wait, 2 no expect_tx (loads only; the barrier never completes -- issue time only),
// 3 wait + expect_tx, no load (the arrive alone completes the phase)
__global__ void __launch_bounds__(128, 1) k3(const __grid_constant__ CUtensorMap tm, int bytes, int iters, int nwarps,
                                             int mode, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    long long t0 = clock64();
    if (warp < nwarps) {
        uint32_t ph = 0;
        int s = 0;
        for (int i = 0; i < iters; ++i) {
            if (i % nwarps == warp) {
                if (i >= kStages && (mode == 0 || mode == 3)) mbar_wait(&full[s], ph ^ 1);
                if (mode != 2) mbar_arrive_expect_tx_warp(&full[s], mode == 3 ? 0 : bytes);
                if (mode != 3) tma_load_2d_warp(ring + s * kStage, &tm, &full[s], 0, (i * (bytes / 128)) % 8192);
            }
            if (++s == kStages) { s = 0; ph ^= 1; }
        }
        if ((threadIdx.x & 31) == 0) out[1 + warp] = clock64() - t0;
    }
    // loads issued without a barrier to wait on must land before the CTA exits
    const long long te = clock64();
    while (clock64() - te < 200000) {
    }
}

// issue loop with the tensor map read from global memory (pointer) instead of
// the kernel-parameter copy: loads only, 1 or 3 warps
__global__ void __launch_bounds__(128, 1) k4(const CUtensorMap* tmg, int bytes, int iters, int nwarps, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
        tma_prefetch_desc(tmg);
    }
    __syncthreads();
    long long t0 = clock64();
    if (warp < nwarps) {
        int s = 0;
        for (int i = 0; i < iters; ++i) {
            if (i % nwarps == warp) tma_load_2d_warp(ring + s * kStage, tmg, &full[s], 0, (i * (bytes / 128)) % 8192);
            if (++s == kStages) s = 0;
        }
        if ((threadIdx.x & 31) == 0) out[1 + warp] = clock64() - t0;
    }
    const long long te = clock64();  // let the unawaited loads land before exit
    while (clock64() - te < 200000) {
    }
}

// two CTAs per SM: each CTA runs its own 4-stage ring of 24 KB fills (A 16 KB +
// B 8 KB boxes) with 3 issuing warps; per-CTA cycles per fill, grid 148 vs 296
__global__ void __launch_bounds__(128, 2) k5(const __grid_constant__ CUtensorMap tmA,
                                             const __grid_constant__ CUtensorMap tmB, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    constexpr int kS = 3;  // warp w owns stage w (one owner per stage: no parity ambiguity)
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kS * kStage);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    long long t0 = clock64();
    if (warp < 3) {
        uint32_t ph = 0;
        int s = 0;
        for (int i = 0; i < iters; ++i) {
            if (s == warp) {
                if (i >= kS) mbar_wait(&full[s], ph ^ 1);
                mbar_arrive_expect_tx_warp(&full[s], kStage);
                const int row = (blockIdx.x * 37 + i) * 128 % 8192;
                tma_load_2d_warp(ring + s * kStage, &tmA, &full[s], 0, row);
                tma_load_2d_warp(ring + s * kStage + kA, &tmB, &full[s], 0, row / 2);
            }
            if (++s == kS) { s = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS && s < iters; ++s) {
            const int last = ((iters - 1 - s) / kS) * kS + s;
            mbar_wait(&full[s], static_cast<uint32_t>((last / kS) & 1));
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

// latency: one warp, one load in flight
__global__ void __launch_bounds__(128, 1) k2(const __grid_constant__ CUtensorMap tm, int bytes, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * kStage);
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            mbar_arrive_expect_tx_warp(&full[0], bytes);
            tma_load_2d_warp(ring, &tm, &full[0], 0, (i * (bytes / 128)) % 8192);
            mbar_wait(&full[0], static_cast<uint32_t>(i & 1));
        }
        if (threadIdx.x == 0) out[0] = clock64() - t0;
    }
}

int main(int argc, char** argv) {
    const bool only_k5 = argc > 1;
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<Encode>(fn);
    __half* A;
    cudaMalloc(&A, 8192ull * 64 * 2);
    cudaMemset(A, 0, 8192ull * 64 * 2);
    CUtensorMap ta, tb;
    cuuint64_t dims[2] = {64, 8192}, strides[1] = {128};
    cuuint32_t boxa[2] = {64, 128}, boxb[2] = {64, 64}, es[2] = {1, 1};
    encode(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, dims, strides, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    encode(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, dims, strides, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    long long* d;
    cudaMalloc(&d, 8 * sizeof(long long));
    const int smem = kStages * kStage + 1024 + 256;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // box-size sweep with 3 issuing warps: one load per fill of rows x 128 B (4..32 KB)
    for (int rows : {32, 64, 128, 256}) {
        if (only_k5) break;
        CUtensorMap tr;
        cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows)};
        encode(&tr, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(d, 0, 8 * sizeof(long long));
            k1<<<1, 128, smem>>>(tr, rows * 128, 512, 3, d);
            cudaDeviceSynchronize();
            long long h[8];
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            if (rep)
                std::printf("3 warps, one %2d KB box per fill: %5.0f cycles per fill, %.1f B/clk\n", rows * 128 / 1024,
                            double(h[0]) / 512, 512.0 * rows * 128 / h[0]);
        }
    }
    {
        CUtensorMap tr;
        cuuint32_t box[2] = {64, 128};
        encode(&tr, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const char* names[] = {"wait + expect_tx + load", "expect_tx + load (no wait)", "load only",
                               "wait + arrive (no load)"};
        for (int nw : {1, 3}) {
            if (only_k5) break;
            for (int mode = 0; mode < 4; ++mode) {
                cudaMemset(d, 0, 8 * sizeof(long long));
                k3<<<1, 128, smem>>>(tr, 16384, 512, nw, mode, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[8];
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                std::printf("%d warp(s), 16 KB fills, %-28s: issue loop %5.0f cycles per fill%s\n", nw, names[mode],
                            double(h[1]) / 512, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
    {
        CUtensorMap tr;
        cuuint32_t box[2] = {64, 128};
        encode(&tr, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUtensorMap* tg;
        cudaMalloc(&tg, sizeof(CUtensorMap));
        cudaMemcpy(tg, &tr, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
        for (int nw : {1, 3}) {
            if (only_k5) break;
            cudaMemset(d, 0, 8 * sizeof(long long));
            k4<<<1, 128, smem>>>(tg, 16384, 512, nw, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[8];
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            std::printf("%d warp(s), 16 KB fills, load only, tensor map in global memory: issue loop %5.0f cycles per fill%s\n",
                        nw, double(h[1]) / 512, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    {
        const int smem5 = 3 * kStage + 1024 + 256;
        cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, smem5);
        long long* d5;
        cudaMalloc(&d5, 296 * sizeof(long long));
        for (int grid : {148, 296}) {
            for (int rep = 0; rep < 2; ++rep) {
                k5<<<grid, 128, smem5>>>(ta, tb, 512, d5);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<long long> h(grid);
                cudaMemcpy(h.data(), d5, grid * sizeof(long long), cudaMemcpyDeviceToHost);
                std::sort(h.begin(), h.end());
                if (rep)
                    std::printf("grid %d (3-stage ring, 24 KB fills, 3 warps per CTA): median %5.0f cycles per fill per CTA"
                                " -> %.1f B/clk per SM%s\n", grid, double(h[grid / 2]) / 512,
                                (grid / 148) * 512.0 * kStage / h[grid / 2], e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
    // latency: one load in flight at a time (issue, wait for it to land, repeat)
    for (int rows : {32, 128, 256}) {
        CUtensorMap tr;
        cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows)};
        encode(&tr, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(d, 0, 8 * sizeof(long long));
            k2<<<1, 128, smem>>>(tr, rows * 128, 256, d);
            cudaDeviceSynchronize();
            long long h[8];
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            if (rep) std::printf("one %2d KB load at a time: %5.0f cycles issue -> landed\n", rows * 128 / 1024, double(h[0]) / 256);
        }
    }
    for (int nw : {1, 2, 3, 4}) {
        for (int iters : {64, 512}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(d, 0, 8 * sizeof(long long));
                k<<<1, 128, smem>>>(ta, tb, iters, nw, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[8];
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                if (rep)
                    std::printf("%d warps, %3d stage fills: all landed after %6lld cycles (%5.0f per fill, %.1f B/clk); "
                                "issue loop %lld cycles (warp 0)%s\n",
                                nw, iters, h[0], double(h[0]) / iters, double(iters) * kStage / h[0], h[1],
                                e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
