// Microbenchmark: GPU-side cost of launch configurations of an (almost) empty
// persistent-style kernel after an L2-flushing memset: plain, 227 KB dynamic
// smem, cluster of 2, cooperative, large __grid_constant__ parameter blocks
// (5 CUtensorMap-sized structs), a TMEM alloc/dealloc, and combinations.
// Single-launch event pairs are quantised (~2 us steps on the B200 box), so
// each configuration is timed as one event pair around R x (memset + kernel)
// minus one around R x memset, divided by R; "x2" appends a second launch of
// the same kernel to each iteration (its increment is the cost without a
// preceding kernel of another shared-memory configuration).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a launch_latency.cu -o launch_latency -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

struct alignas(64) Big {
    unsigned char b[128];
};
struct Params {
    Big m[5];
    unsigned char args[256];
};

__global__ void k_small(int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = 1;
}
__global__ void k_big(const __grid_constant__ Params p, int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = p.args[0] + p.m[4].b[3];
}
// variant bits: 1 relinquish the allocation permit, 2 dealloc at the end
template <int kVariant>
__global__ void k_tmem(int* out) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(&slot))));
        if (kVariant & 1) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if ((kVariant & 2) && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(slot));
    if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = 1;
}

int main() {
    int* d;
    cudaMalloc(&d, 4);
    void* flush;
    const size_t fb = 128u << 20;
    cudaMalloc(&flush, fb);
    for (auto f : {(const void*)k_small, (const void*)k_big, (const void*)k_tmem<3>, (const void*)k_tmem<2>,
                   (const void*)k_tmem<1>, (const void*)k_tmem<0>})
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    Params P{};
    struct Cfg {
        const char* name;
        int kind;  // 0 small, 1 big params, 2 tmem alloc+relinquish+dealloc, 3 alloc+dealloc, 4 alloc+relinquish, 5 alloc only
        int smem, cluster;
        bool coop;
        int grid, launches;
    };
    std::vector<Cfg> cfgs = {
        {"plain 148x256", 0, 0, 1, false, 148, 1},
        {"plain 148x256 x2", 0, 0, 1, false, 148, 2},
        {"smem 227K", 0, 227 * 1024, 1, false, 148, 1},
        {"smem 227K x2", 0, 227 * 1024, 1, false, 148, 2},
        {"cluster 2", 0, 0, 2, false, 148, 1},
        {"coop", 0, 0, 1, true, 148, 1},
        {"big params", 1, 0, 1, false, 148, 1},
        {"tmem alloc + relinquish + dealloc", 2, 0, 1, false, 148, 1},
        {"tmem alloc + dealloc", 3, 0, 1, false, 148, 1},
        {"tmem alloc + relinquish (no dealloc)", 4, 0, 1, false, 148, 1},
        {"tmem alloc only", 5, 0, 1, false, 148, 1},
        {"smem 227K + coop", 0, 227 * 1024, 1, true, 148, 1},
        {"big params + smem + coop", 1, 227 * 1024, 1, true, 148, 1},
        {"big params + cluster 2 + smem + coop", 1, 227 * 1024, 2, true, 148, 1},
        {"big params + cluster 2 + smem + coop x2", 1, 227 * 1024, 2, true, 148, 2},
        {"big params + smem, 16 CTAs", 1, 227 * 1024, 1, false, 16, 1},
        {"big params + smem + coop, 16 CTAs", 1, 227 * 1024, 1, true, 16, 1},
    };
    const int R = 50;
    auto seq = [&](const Cfg* c) {
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        for (int r = 0; r < R; ++r) {
            cudaMemsetAsync(flush, r, fb, s);
            if (!c) continue;
            for (int l = 0; l < c->launches; ++l) {
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(c->grid);
                lc.blockDim = dim3(256);
                lc.dynamicSmemBytes = c->smem;
                lc.stream = s;
                cudaLaunchAttribute at[2];
                int na = 0;
                if (c->cluster > 1) {
                    at[na].id = cudaLaunchAttributeClusterDimension;
                    at[na].val.clusterDim.x = c->cluster;
                    at[na].val.clusterDim.y = 1;
                    at[na].val.clusterDim.z = 1;
                    ++na;
                }
                if (c->coop) {
                    at[na].id = cudaLaunchAttributeCooperative;
                    at[na].val.cooperative = 1;
                    ++na;
                }
                lc.attrs = at;
                lc.numAttrs = na;
                cudaError_t err = c->kind == 1   ? cudaLaunchKernelEx(&lc, k_big, P, d)
                                  : c->kind == 2 ? cudaLaunchKernelEx(&lc, k_tmem<3>, d)
                                  : c->kind == 3 ? cudaLaunchKernelEx(&lc, k_tmem<2>, d)
                                  : c->kind == 4 ? cudaLaunchKernelEx(&lc, k_tmem<1>, d)
                                  : c->kind == 5 ? cudaLaunchKernelEx(&lc, k_tmem<0>, d)
                                                 : cudaLaunchKernelEx(&lc, k_small, d);
                if (err != cudaSuccess) {
                    std::printf("%s: %s\n", c->name, cudaGetErrorString(err));
                    return -1.0f;
                }
            }
        }
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms * 1000.f;
    };
    for (auto& c : cfgs) {
        std::vector<float> ts;
        seq(&c);
        for (int rep = 0; rep < 7; ++rep) {
            const float base = seq(nullptr);
            const float t = seq(&c);
            if (t < 0) break;
            ts.push_back((t - base) / R);
        }
        if (ts.empty()) continue;
        std::sort(ts.begin(), ts.end());
        std::printf("%-44s %.2f us per iteration (min %.2f)\n", c.name, ts[ts.size() / 2], ts[0]);
    }
    return 0;
}
