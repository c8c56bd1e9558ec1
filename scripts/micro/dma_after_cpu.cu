// Microbenchmark: does host-side work on the pinned input change the copy
// engine's H2D rate afterwards? (a) 128 MiB H2D + 64 MiB D2H, repeated after
// various host actions.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
    const size_t MB = 1u << 20, total = 128 * MB, piece = 8 * MB, npieces = total / piece;
    float* h_in; uint16_t* h_f16; float* h_c;
    cudaHostAlloc(&h_in, total, 0); cudaHostAlloc(&h_f16, total / 2, 0); cudaHostAlloc(&h_c, 64 * MB, 0);
    for (size_t i = 0; i < total / 4; ++i) h_in[i] = float(i % 1000) / 1000.f;
    std::memset(h_f16, 0, total / 2); std::memset(h_c, 0, 64 * MB);
    char *d_in, *d_c; cudaMalloc(&d_in, total); cudaMalloc(&d_c, 64 * MB);
    cudaStream_t up, dn;
    cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&dn, cudaStreamNonBlocking);
    auto dma = [&](const char* tag, bool with_dn) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaDeviceSynchronize();
            double t0 = now_ms();
            for (size_t p = 0; p < npieces; ++p)
                cudaMemcpyAsync(d_in + p * piece, (char*)h_in + p * piece, piece, cudaMemcpyHostToDevice, up);
            if (with_dn) for (size_t p = 0; p < 8; ++p)
                cudaMemcpyAsync((char*)h_c + p * piece, d_c + p * piece, piece, cudaMemcpyDeviceToHost, dn);
            cudaDeviceSynchronize();
            std::printf("%-40s %s %.3f ms\n", tag, with_dn ? "up+down" : "up     ", now_ms() - t0);
        }
    };
    auto par = [&](unsigned T, auto fn) {
        std::atomic<size_t> next{0}; std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t) th.emplace_back([&] { for (size_t q; (q = next.fetch_add(1)) < 128;) fn(q); });
        for (auto& x : th) x.join();
    };
    for (int k = 0; k < 4; ++k) dma("start", true);
    par(16, [&](size_t) {});
    dma("after 16 empty threads", true);
    float* other; cudaHostAlloc(&other, total, 0); std::memset(other, 0, total);
    dma("after alloc+memset other pinned", true);
    volatile float sink = 0;
    par(16, [&](size_t q) { float s = 0; const float* p = other + q * (MB / 4); for (size_t i = 0; i < MB / 4; ++i) s += p[i]; sink = sink + s; });
    dma("after CPU read of other", true);
    par(1, [&](size_t q) { float s = 0; const float* p = h_in + q * (MB / 4); for (size_t i = 0; i < MB / 4; ++i) s += p[i]; sink = sink + s; });
    dma("after 1-thread read of h_in", true);
    par(16, [&](size_t q) { float s = 0; const float* p = h_in + q * (MB / 4); for (size_t i = 0; i < MB / 4; ++i) s += p[i]; sink = sink + s; });
    dma("after 16-thread read of h_in", true);
    for (size_t i = 0; i < total / 4; ++i) h_in[i] = float(i % 999) / 1000.f;
    dma("after main-thread rewrite of h_in", true);
    float* fresh; cudaHostAlloc(&fresh, total, 0);
    for (size_t i = 0; i < total / 4; ++i) fresh[i] = float(i % 1000) / 1000.f;
    h_in = fresh;
    dma("fresh buffer written by main thread", true);
    return 0;
}
