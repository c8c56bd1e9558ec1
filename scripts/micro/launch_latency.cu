// Microbenchmark: GPU-side cost of launch configurations of an (almost) empty
// persistent-style kernel, event-timed, after an L2-flushing memset: plain,
// 227 KB dynamic smem, cluster of 2, cooperative, large __grid_constant__
// parameter blocks (5 CUtensorMap-sized structs), and combinations; also the
// cost of TMEM alloc/dealloc is NOT included (kernel body is empty).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

struct alignas(64) Big { unsigned char b[128]; };
struct Params { Big m[5]; unsigned char args[256]; };

__global__ void k_small(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = 1; }
__global__ void k_big(const __grid_constant__ Params p, int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = p.args[0] + p.m[4].b[3];
}

int main() {
    int* d; cudaMalloc(&d, 4);
    void* flush; size_t fb = 512u << 20; cudaMalloc(&flush, fb);
    cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    Params P{};
    struct Cfg { const char* name; bool big; int smem; int cluster; bool coop; int grid; bool flush; };
    std::vector<Cfg> cfgs = {
        {"plain 148x256", false, 0, 1, false, 148, true},
        {"smem 227K", false, 227 * 1024, 1, false, 148, true},
        {"smem 227K, no flush before", false, 227 * 1024, 1, false, 148, false},
        {"cluster 2", false, 0, 2, false, 148, true},
        {"cluster 2 + smem 227K", false, 227 * 1024, 2, false, 148, true},
        {"cluster 2 + smem + coop", false, 227 * 1024, 2, true, 148, true},
        {"big params", true, 0, 1, false, 148, true},
        {"big params + cluster 2 + smem", true, 227 * 1024, 2, false, 148, true},
        {"big params + cluster 2 + smem + coop", true, 227 * 1024, 2, true, 148, true},
        {"big params + smem, 64 CTAs", true, 227 * 1024, 1, false, 64, true},
    };
    for (auto& c : cfgs) {
        std::vector<float> ts;
        for (int rep = 0; rep < 30; ++rep) {
            if (c.flush) cudaMemsetAsync(flush, rep, fb, s);
            else k_small<<<1, 32, 0, s>>>(nullptr);
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(c.grid); lc.blockDim = dim3(256); lc.dynamicSmemBytes = c.smem; lc.stream = s;
            cudaLaunchAttribute at[2]; int na = 0;
            if (c.cluster > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = c.cluster; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
            if (c.coop) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
            lc.attrs = at; lc.numAttrs = na;
            cudaEventRecord(e0, s);
            cudaError_t err = c.big ? cudaLaunchKernelEx(&lc, k_big, P, d) : cudaLaunchKernelEx(&lc, k_small, d);
            cudaEventRecord(e1, s);
            cudaStreamSynchronize(s);
            if (err != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(err)); break; }
            float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms * 1000.f);
        }
        if (ts.empty()) continue;
        std::sort(ts.begin(), ts.end());
        printf("%-42s median %.2f us  min %.2f\n", c.name, ts[ts.size() / 2], ts[0]);
    }
    return 0;
}
