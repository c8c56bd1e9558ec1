// Microbenchmark: bulk copy throughput shared::cta -> shared::cluster (DSMEM push)
// between the two CTAs of a cluster, vs a bulk store to global memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) push(int mode, int reps, unsigned long long* out, float* gws) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const uint32_t bytes = 96 * 1024;  // src [0, 96K), dst [96K, 192K)
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    cluster.sync();
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (mode == 0) {  // rank 0 pushes 96 KB into rank 1's smem; rank 1 waits on its barrier
            if (rank == 1 && threadIdx.x == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes));
            }
            cluster.sync();
            if (rank == 0 && threadIdx.x == 0) {
                uint32_t dst, rbar;
                asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(dst) : "r"(smem_u32(smem + bytes)));
                asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(rbar) : "r"(smem_u32(&bar)));
                for (int c = 0; c < 6; ++c)
                    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(dst + c * 16384), "r"(smem_u32(smem + c * 16384)), "r"(16384), "r"(rbar) : "memory");
            }
            if (rank == 1 && threadIdx.x == 0) {
                asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)), "r"(phase));
            }
            phase ^= 1;
            cluster.sync();
        } else {  // each CTA bulk-stores 96 KB to global, waits for completion
            if (threadIdx.x == 0) {
                for (int c = 0; c < 6; ++c)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gws + rank * 24576 + c * 4096),
                                 "r"(smem_u32(smem + c * 16384)), "r"(16384) : "memory");
                asm volatile("cp.async.bulk.commit_group;");
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            }
            cluster.sync();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[mode] = (t1 - t0) / reps;
}

int main() {
    unsigned long long* out; float* gws;
    cudaMalloc(&out, 64); cudaMalloc(&gws, 2 << 20);
    cudaFuncSetAttribute(push, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"DSMEM bulk push 96 KB (rank0 -> rank1)", "bulk store 96 KB to global (each CTA)"};
    for (int m = 0; m < 2; ++m) {
        push<<<2, 128, 200 * 1024>>>(m, 20, out, gws);
        push<<<2, 128, 200 * 1024>>>(m, 200, out, gws);
        unsigned long long h[2];
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("%-42s %7llu cycles per iteration (%.1f B/clk)  %s\n", names[m], h[m], 98304.0 / h[m], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
