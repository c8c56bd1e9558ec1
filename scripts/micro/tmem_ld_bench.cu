// Microbenchmark: tcgen05.ld throughput (TMEM -> registers) on one SM, 4 warps
// covering the 128 TMEM lanes, 256 fp32 columns each (one 128x256 accumulator).
// Variants: 32x32b.x32 with / without wait per load, x64, x128, plus the same
// with the conflict-free STS of the epilogue. Prints cycles per 128x256 drain.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int N>
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* v);
#define LD_ASM(N, REGS) 
__device__ __forceinline__ void ld_x32(uint32_t t, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(t));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__global__ void __launch_bounds__(128, 1) bench(int mode, int reps, unsigned long long* out, float* sink, float* gws) {
    __shared__ uint32_t slot;
    extern __shared__ float stage[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (static_cast<uint32_t>(warp * 32) << 16);
    float acc = 0.f;
    uint32_t r0[32], r1[32];
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (mode == 0) {  // load + wait per chunk
            for (int c = 0; c < 8; ++c) { ld_x32(base + c * 32, r0); ld_wait(); acc += __uint_as_float(r0[c]); }
        } else if (mode == 1) {  // two loads in flight
            for (int c = 0; c < 8; c += 2) { ld_x32(base + c * 32, r0); ld_x32(base + c * 32 + 32, r1); ld_wait(); acc += __uint_as_float(r0[3]) + __uint_as_float(r1[5]); }
        } else if (mode == 2) {  // load + STS (the epilogue staging), wait per chunk
            for (int c = 0; c < 8; ++c) {
                ld_x32(base + c * 32, r0); ld_wait();
                float* d = stage + (c & 1) * 4096 + threadIdx.x;
#pragma unroll
                for (int j = 0; j < 32; ++j) d[j * 128] = __uint_as_float(r0[j]);
            }
        } else if (mode == 4 || mode == 5) {  // drain_pairs: 2 chunks, fence.proxy.async + named barrier, [bulk s2g]
            for (int c = 0; c < 8; c += 2) {
                ld_x32(base + c * 32, r0); ld_wait();
                ld_x32(base + c * 32 + 32, r1);
                float* d0 = stage + (c & 7) * 4096 + threadIdx.x;
#pragma unroll
                for (int j = 0; j < 32; ++j) d0[j * 128] = __uint_as_float(r0[j]);
                ld_wait();
                float* d1 = stage + ((c + 1) & 7) * 4096 + threadIdx.x;
#pragma unroll
                for (int j = 0; j < 32; ++j) d1[j * 128] = __uint_as_float(r1[j]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (mode == 5 && threadIdx.x == 0) {
                    for (int x = c; x < c + 2; ++x)
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gws + x * 4096),
                                     "r"(smem_u32(stage + x * 4096)), "r"(16384) : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
            if (mode == 5 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        } else if (mode == 6) {  // ld + coalesced STG.32 (column-major chunk: warp writes 128 B per j)
            for (int c = 0; c < 8; ++c) {
                ld_x32(base + c * 32, r0); ld_wait();
                float* d = gws + (c & 7) * 4096 + threadIdx.x;
#pragma unroll
                for (int j = 0; j < 32; ++j) d[j * 128] = __uint_as_float(r0[j]);
            }
            __threadfence();
        } else if (mode == 7) {  // ld + STG.128, each thread its row's 32 floats contiguous
            for (int c = 0; c < 8; ++c) {
                ld_x32(base + c * 32, r0); ld_wait();
                float4* d = reinterpret_cast<float4*>(gws + (c & 7) * 4096 + threadIdx.x * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j) d[j] = make_float4(__uint_as_float(r0[4*j]), __uint_as_float(r0[4*j+1]), __uint_as_float(r0[4*j+2]), __uint_as_float(r0[4*j+3]));
            }
            __threadfence();
        } else if (mode == 3) {  // STS only
            for (int c = 0; c < 8; ++c) {
                float* d = stage + (c & 1) * 4096 + threadIdx.x;
#pragma unroll
                for (int j = 0; j < 32; ++j) d[j * 128] = __uint_as_float(r0[j]) + it;
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[mode] = (t1 - t0) / reps;
    sink[threadIdx.x] = acc + stage[threadIdx.x];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    unsigned long long* out; float* sink;
    cudaMalloc(&out, 64); cudaMalloc(&sink, 4096);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    const char* names[] = {"ld+wait per 32-col chunk", "2 loads in flight", "ld+wait+STS (epilogue staging)", "STS only", "drain_pairs (fence+bar)", "drain_pairs + bulk s2g", "ld + STG.32 coalesced", "ld + STG.128 row-contiguous"};
    float* gws; cudaMalloc(&gws, 8 * 16384);
    for (int m = 0; m < 8; ++m) {
        bench<<<1, 128, 128 * 1024>>>(m, 100, out, sink, gws);
        bench<<<1, 128, 128 * 1024>>>(m, 1000, out, sink, gws);
        unsigned long long h[8];
        cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
        printf("%-34s %6llu cycles per 128x256 fp32 drain (%.1f B/clk)  err=%s\n", names[m], h[m], 131072.0 / h[m],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
