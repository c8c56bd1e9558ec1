// Microbenchmark: host-snapped uploads through (a) one large pinned staging
// buffer written with streaming stores (the runtime's scheme) vs (b) a small
// ring of pinned slots written with regular stores, so the copy engine may read
// them from the CPU's last-level cache instead of DRAM. 128 MiB fp32 -> 64 MiB
// f16 crosses PCIe while a 64 MiB D2H runs concurrently; T host threads convert.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
__attribute__((target("avx512f,f16c"))) static void cvt(const float* s, uint16_t* d, size_t n, bool stream) {
    for (size_t i = 0; i < n; i += 16) {
        __m256i h = _mm512_cvtps_ph(_mm512_loadu_ps(s + i), _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
        if (stream) _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), h);
        else _mm256_store_si256(reinterpret_cast<__m256i*>(d + i), h);
    }
}

int main() {
    const size_t MB = 1u << 20, total = 128 * MB, elems = total / 4;
    float* h_in;
    uint16_t* big;
    float* h_c;
    cudaHostAlloc(&h_in, total, 0);
    cudaHostAlloc(&big, total / 2, 0);
    cudaHostAlloc(&h_c, 64 * MB, 0);
    for (size_t i = 0; i < elems; ++i) h_in[i] = float(i % 2001) / 1000.f - 1.f;
    memset(big, 0, total / 2);
    memset(h_c, 0, 64 * MB);
    char *d_in, *d_c;
    cudaMalloc(&d_in, total / 2);
    cudaMalloc(&d_c, 64 * MB);
    cudaStream_t up, dn;
    cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&dn, cudaStreamNonBlocking);
    const unsigned T = std::min(16u, std::thread::hardware_concurrency());
    for (size_t slot_mb : {0u, 1u, 2u, 4u}) {       // 0 = one big buffer, streaming stores
        for (int nslots : {4, 8}) {
            if (slot_mb == 0 && nslots != 4) continue;
            const size_t slot_elems = slot_mb ? slot_mb * MB / 2 : 4 * MB / 2;  // f16 elements per piece
            const size_t npieces = elems / slot_elems;
            std::vector<double> ts;
            std::vector<cudaEvent_t> done(nslots);
            for (auto& e : done) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            for (int rep = 0; rep < 12; ++rep) {
                cudaDeviceSynchronize();
                std::atomic<size_t> next{0};
                std::vector<std::atomic<int>> ready(npieces);
                for (auto& r : ready) r = 0;
                std::atomic<size_t> released{0};  // pieces whose slot may be reused (ring mode)
                const double t0 = now_ms();
                for (size_t p = 0; p < 8; ++p)
                    cudaMemcpyAsync(reinterpret_cast<char*>(h_c) + p * 8 * MB, d_c + p * 8 * MB, 8 * MB, cudaMemcpyDeviceToHost, dn);
                std::vector<std::thread> th;
                for (unsigned t = 0; t < T; ++t)
                    th.emplace_back([&] {
                        for (size_t p; (p = next.fetch_add(1)) < npieces;) {
                            uint16_t* dst;
                            if (slot_mb == 0) dst = big + p * slot_elems;
                            else {
                                while (p >= released.load(std::memory_order_acquire) + nslots) _mm_pause();
                                dst = big + (p % nslots) * slot_elems;
                            }
                            cvt(h_in + p * slot_elems, dst, slot_elems, slot_mb == 0);
                            if (slot_mb == 0) _mm_sfence();
                            ready[p].store(1, std::memory_order_release);
                        }
                    });
                for (size_t p = 0; p < npieces; ++p) {
                    while (!ready[p].load(std::memory_order_acquire)) _mm_pause();
                    const uint16_t* src = slot_mb == 0 ? big + p * slot_elems : big + (p % nslots) * slot_elems;
                    cudaMemcpyAsync(d_in + p * slot_elems * 2, src, slot_elems * 2, cudaMemcpyHostToDevice, up);
                    if (slot_mb) {
                        cudaEventRecord(done[p % nslots], up);
                        // release the slot that piece p - nslots + 1 used once its copy is done
                        if (p + 1 >= static_cast<size_t>(nslots)) {
                            const size_t q = p + 1 - nslots;
                            cudaEventSynchronize(done[q % nslots]);
                            released.store(q + 1, std::memory_order_release);
                        }
                    }
                }
                released.store(npieces + nslots, std::memory_order_release);
                cudaDeviceSynchronize();
                for (auto& x : th) x.join();
                ts.push_back(now_ms() - t0);
            }
            std::sort(ts.begin(), ts.end());
            printf("%s slot %zu MiB x %d: median %.3f ms  min %.3f\n", slot_mb ? "ring (regular stores)" : "big buffer (streaming)",
                   slot_mb ? slot_mb : 0, slot_mb ? nslots : 0, ts[ts.size() / 2], ts[0]);
        }
    }
    return 0;
}
