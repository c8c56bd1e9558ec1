// Microbenchmark: SM-driven reads of pinned host memory (zero-copy over PCIe)
// for a pitched region -- a row panel of a column-major fp32 matrix, lines of
// `seg` bytes -- converted to f16 into device memory, alone and with a
// concurrent 64 MiB D2H DMA copy. Varies the CTA count (SMs used).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

__global__ void gather_convert(const float4* __restrict__ src, __half2* __restrict__ dst, long width4, long height,
                               long pitch4) {
    const long n = width4 * height;
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long>(gridDim.x) * blockDim.x * 4) {
        float4 v[4];
        long o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // 4 independent 16B loads in flight per thread
            const long j = i + static_cast<long>(u) * gridDim.x * blockDim.x;
            const long y = j / width4, x = j - y * width4;
            o[u] = j < n ? y * pitch4 + x : -1;
            if (o[u] >= 0) v[u] = src[o[u]];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (o[u] >= 0) {
                dst[2 * o[u]] = __floats2half2_rn(v[u].x, v[u].y);
                dst[2 * o[u] + 1] = __floats2half2_rn(v[u].z, v[u].w);
            }
    }
}

int main() {
    const size_t n = 64ull << 20;
    float *h_a, *h_c, *d_c;
    __half* d_a;
    cudaHostAlloc(&h_a, n, cudaHostAllocMapped);
    cudaHostAlloc(&h_c, n, cudaHostAllocDefault);
    cudaMalloc(&d_a, n / 2);
    cudaMalloc(&d_c, n);
    for (size_t i = 0; i < n / 4; ++i) h_a[i] = 1.0f;
    float* dev_view = nullptr;
    cudaHostGetDevicePointer(&dev_view, h_a, 0);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const long pitch = 16384;  // floats: a 16384-row column-major matrix
    for (int seg : {2048, 8192, 65536}) {
        for (int ctas : {16, 32, 64, 148, 296}) {
            const long width = seg / 4, height = static_cast<long>(n / 4) / pitch;
            const long panels = pitch / width;
            float best_alone = 1e9f, best_both = 1e9f;
            for (int rep = 0; rep < 4; ++rep) {
                for (int both = 0; both < 2; ++both) {
                    cudaDeviceSynchronize();
                    cudaEventRecord(e0, s1);
                    if (both) cudaMemcpyAsync(h_c, d_c, n, cudaMemcpyDeviceToHost, s2);
                    for (long p = 0; p < panels; ++p)
                        gather_convert<<<ctas, 256, 0, s1>>>(reinterpret_cast<const float4*>(dev_view + p * width),
                                                             reinterpret_cast<__half2*>(d_a + p * width), width / 4,
                                                             height, pitch / 4);
                    cudaEventRecord(e1, s1);
                    cudaDeviceSynchronize();
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    (both ? best_both : best_alone) = std::min(both ? best_both : best_alone, ms);
                }
            }
            std::printf("lines %6d B, %3d CTAs: host->device read+convert alone %5.1f GB/s; with concurrent 64 MiB D2H "
                        "DMA: read %5.1f GB/s\n",
                        seg, ctas, n / best_alone / 1e6, n / best_both / 1e6);
        }
    }
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
