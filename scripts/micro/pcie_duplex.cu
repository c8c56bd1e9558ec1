// Microbenchmark: PCIe duplex throughput of linear 8 MiB copies, H2D of a
// 128 MiB working set (two 64 MiB operands) against D2H of a 64 MiB result,
// with host buffers from cudaHostAlloc vs 2 MiB-aligned transparent-huge-page
// memory registered with cudaHostRegister; and a 64 MiB reused working set.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

static void* host_buf(size_t n, bool thp) {
    void* p = nullptr;
    if (!thp) {
        cudaHostAlloc(&p, n, cudaHostAllocDefault);
        return p;
    }
    p = std::aligned_alloc(2u << 20, n);
    madvise(p, n, MADV_HUGEPAGE);
    std::memset(p, 1, n);
    cudaHostRegister(p, n, cudaHostRegisterDefault);
    return p;
}

__global__ void spin(long ns) {
    long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > ns) break;
    }
}

int main() {
    const size_t mb = 1u << 20, n = 64 * mb, chunk = 8 * mb;
    char *d_a, *d_b, *d_c;
    cudaMalloc(&d_a, n);
    cudaMalloc(&d_b, n);
    cudaMalloc(&d_c, n);
    cudaStream_t up, dn;
    cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&dn, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    for (int thp = 0; thp < 2; ++thp) {
        char* h_a = static_cast<char*>(host_buf(n, thp));
        char* h_b = static_cast<char*>(host_buf(n, thp));
        char* h_c = static_cast<char*>(host_buf(n, thp));
        for (int reuse = 0; reuse < 2; ++reuse) {
            float best = 1e9f, up_ms = 0, dn_ms = 0;
            for (int rep = 0; rep < 5; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(e0, up);
                cudaStreamWaitEvent(dn, e0, 0);
                // up: A then B (128 MiB), down: C (64 MiB) -- all 8 MiB linear pieces
                for (size_t o = 0; o < 2 * n; o += chunk) {
                    const bool second = o >= n;
                    char* hs = reuse ? h_a : (second ? h_b : h_a);
                    char* dd = second ? d_b : d_a;
                    cudaMemcpyAsync(dd + o % n, hs + o % n, chunk, cudaMemcpyHostToDevice, up);
                    if (o % (2 * chunk) == 0)
                        cudaMemcpyAsync((reuse ? h_b : h_c) + (o / 2) % n, d_c + (o / 2) % n, chunk,
                                        cudaMemcpyDeviceToHost, dn);
                }
                cudaEventRecord(e1, up);
                cudaEventRecord(e2, dn);
                cudaDeviceSynchronize();
                float a = 0, b = 0;
                cudaEventElapsedTime(&a, e0, e1);
                cudaEventElapsedTime(&b, e0, e2);
                const float t = a > b ? a : b;
                if (t < best) best = t, up_ms = a, dn_ms = b;
            }
            std::printf("%s host memory, %s: 128 MiB up + 64 MiB down in %.3f ms = %.1f GB/s total (up done %.3f, down done %.3f)\n",
                        thp ? "THP+cudaHostRegister" : "cudaHostAlloc", reuse ? "64 MiB reused working set" : "192 MiB working set",
                        best, 3.0 * n / best / 1e6, up_ms, dn_ms);
        }
    }
    // the column-panel pipeline's pattern: A (64 MiB) up, then per panel j: B_j up,
    // [work on a third stream], C_j down gated on it
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t ev[16], evc[16];
    for (int j = 0; j < 16; ++j) cudaEventCreateWithFlags(&ev[j], cudaEventDisableTiming), cudaEventCreateWithFlags(&evc[j], cudaEventDisableTiming);
    char* h_a = static_cast<char*>(host_buf(n, false));
    char* h_b = static_cast<char*>(host_buf(n, false));
    char* h_c = static_cast<char*>(host_buf(n, false));
    for (int variant = 0; variant < 3; ++variant) {
        float best = 1e9f, up_ms = 0, dn_ms = 0;
        for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, up);
            cudaStreamWaitEvent(dn, e0, 0);
            cudaStreamWaitEvent(s, e0, 0);
            cudaMemcpyAsync(d_a, h_a, n, cudaMemcpyHostToDevice, up);
            for (int j = 0; j < 8; ++j) {
                cudaMemcpyAsync(d_b + j * chunk, h_b + j * chunk, chunk, cudaMemcpyHostToDevice, up);
                cudaEventRecord(ev[j], up);
                if (variant == 0) {  // no dependency
                    cudaMemcpyAsync(h_c + j * chunk, d_c + j * chunk, chunk, cudaMemcpyDeviceToHost, dn);
                } else {
                    cudaStreamWaitEvent(s, ev[j], 0);
                    if (variant == 2) spin<<<148, 32, 0, s>>>(50000);
                    cudaEventRecord(evc[j], s);
                    cudaStreamWaitEvent(dn, evc[j], 0);
                    cudaMemcpyAsync(h_c + j * chunk, d_c + j * chunk, chunk, cudaMemcpyDeviceToHost, dn);
                }
            }
            cudaEventRecord(e1, up);
            cudaEventRecord(e2, dn);
            cudaDeviceSynchronize();
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, e0, e1);
            cudaEventElapsedTime(&b, e0, e2);
            const float t = a > b ? a : b;
            if (t < best) best = t, up_ms = a, dn_ms = b;
        }
        std::printf("panel pattern (%s): %.3f ms (up done %.3f, down done %.3f)\n",
                    variant == 0 ? "C_j down ungated" : variant == 1 ? "C_j down gated on B_j up" : "gated + 50 us kernel per panel",
                    best, up_ms, dn_ms);
    }
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
