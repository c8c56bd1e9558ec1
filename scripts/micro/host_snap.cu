// Microbenchmark: can host cores snap part of the fp32 inputs to f16 while the
// copy engine uploads the rest, so fewer bytes cross PCIe?
//   (a) H2D of 128 MiB fp32 (8 MiB linear pieces), alone and against a 64 MiB D2H
//   (b) host fp32 -> f16 conversion of 128 MiB (F16C, plain vs streaming stores)
//       on T threads
//   (c) hybrid: T threads convert a fraction x of the 8 MiB pieces into a pinned
//       f16 staging buffer while the copy engine uploads the other pieces as
//       fp32; each converted piece is uploaded as f16 as soon as it is ready;
//       a 64 MiB D2H runs concurrently (the C download of the real call)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mf16c,-mavx2,-pthread
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void cvt_piece(const float* src, uint16_t* dst, size_t n, bool stream) {
    size_t i = 0;
    for (; i + 16 <= n; i += 16) {
        __m256 a = _mm256_loadu_ps(src + i), b = _mm256_loadu_ps(src + i + 8);
        __m128i ha = _mm256_cvtps_ph(a, _MM_FROUND_TO_NEAREST_INT), hb = _mm256_cvtps_ph(b, _MM_FROUND_TO_NEAREST_INT);
        __m256i h = _mm256_set_m128i(hb, ha);
        if (stream) _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), h);
        else _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), h);
    }
    for (; i < n; ++i) dst[i] = _cvtss_sh(src[i], 0);
}

int main() {
    const size_t MB = 1u << 20, total = 128 * MB, piece = 8 * MB, npieces = total / piece;
    const size_t elems = total / 4, pe = piece / 4;
    float* h_in;
    uint16_t* h_f16;
    float* h_c;
    cudaHostAlloc(&h_in, total, cudaHostAllocDefault);
    cudaHostAlloc(&h_f16, total / 2, cudaHostAllocDefault);
    cudaHostAlloc(&h_c, 64 * MB, cudaHostAllocDefault);
    for (size_t i = 0; i < elems; ++i) h_in[i] = static_cast<float>((i * 2654435761u) % 2001) / 1000.0f - 1.0f;
    std::memset(h_f16, 0, total / 2);
    std::memset(h_c, 0, 64 * MB);
    char *d_in, *d_c;
    cudaMalloc(&d_in, total);
    cudaMalloc(&d_c, 64 * MB);
    cudaStream_t up, dn;
    cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&dn, cudaStreamNonBlocking);
    const unsigned hw = std::thread::hardware_concurrency();
    std::printf("host threads available: %u\n", hw);

    // (a) DMA alone / with D2H
    for (int with_dn = 0; with_dn < 2; ++with_dn) {
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            double t0 = now_ms();
            for (size_t p = 0; p < npieces; ++p)
                cudaMemcpyAsync(d_in + p * piece, reinterpret_cast<char*>(h_in) + p * piece, piece, cudaMemcpyHostToDevice, up);
            if (with_dn)
                for (size_t p = 0; p < 8; ++p)
                    cudaMemcpyAsync(reinterpret_cast<char*>(h_c) + p * piece, d_c + p * piece, piece, cudaMemcpyDeviceToHost, dn);
            cudaDeviceSynchronize();
            best = std::min(best, now_ms() - t0);
        }
        std::printf("(a) H2D 128 MiB fp32%s: %.3f ms (%.1f GB/s up)\n", with_dn ? " + D2H 64 MiB" : "", best,
                    total / best / 1e6);
    }

    // (b) conversion throughput
    for (int stream = 0; stream < 2; ++stream)
        for (unsigned T : {1u, 2u, 4u, 8u, 12u, 16u, 24u, 32u}) {
            if (T > hw) continue;
            double best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                std::atomic<size_t> next{0};
                double t0 = now_ms();
                std::vector<std::thread> th;
                for (unsigned t = 0; t < T; ++t)
                    th.emplace_back([&] {
                        for (size_t p; (p = next.fetch_add(1)) < npieces * 8;)  // 1 MiB sub-pieces
                            cvt_piece(h_in + p * pe / 8, h_f16 + p * pe / 8, pe / 8, stream);
                    });
                for (auto& x : th) x.join();
                if (stream) _mm_sfence();
                best = std::min(best, now_ms() - t0);
            }
            std::printf("(b) convert 128 MiB fp32 -> f16, %u threads, %s stores: %.3f ms (%.1f GB/s of fp32 in)\n", T,
                        stream ? "streaming" : "plain", best, total / best / 1e6);
        }

    // (c) hybrid with a persistent pool (condition-variable wake, as a runtime
    // would keep it), configurations interleaved, 15 rounds: min and median
    struct Pool {
        std::mutex mu;
        std::condition_variable cv;
        unsigned epoch = 0, T = 0;
        size_t h = 0;
        std::atomic<size_t> next{0};
        std::atomic<int> left[64];
        std::vector<std::thread> th;
        bool stop = false;
    };
    const float* src = h_in;
    uint16_t* dstp = h_f16;
    Pool pool;
    for (unsigned t = 0; t < hw; ++t)
        pool.th.emplace_back([&, t] {
            unsigned seen = 0;
            for (;;) {
                {
                    std::unique_lock<std::mutex> lk(pool.mu);
                    pool.cv.wait(lk, [&] { return pool.stop || pool.epoch != seen; });
                    if (pool.stop) return;
                    seen = pool.epoch;
                    if (t >= pool.T) continue;
                }
                for (size_t q; (q = pool.next.fetch_add(1)) < pool.h * 8;) {
                    cvt_piece(src + q * pe / 8, dstp + q * pe / 8, pe / 8, true);
                    _mm_sfence();
                    pool.left[q / 8].fetch_sub(1, std::memory_order_release);
                }
            }
        });
    struct Cfg { unsigned T; size_t h; std::vector<double> ms; };
    std::vector<Cfg> cfgs;
    cfgs.push_back({0, 0, {}});  // no pool wake at all
    for (unsigned T : {4u, 8u, 16u})
        for (size_t h : {0u, 8u, 10u, 12u, 14u})
            if (T <= hw && !(h == 0 && T != 4)) cfgs.push_back({T, h, {}});
    for (int round = 0; round < 15; ++round)
        for (auto& c : cfgs) {
            cudaDeviceSynchronize();
            pool.next = 0;
            for (size_t p = 0; p < c.h; ++p) pool.left[p] = 8;
            const double t0 = now_ms();
            if (c.T) {
                {
                    std::lock_guard<std::mutex> lk(pool.mu);
                    pool.T = c.T;
                    pool.h = c.h;
                    ++pool.epoch;
                }
                pool.cv.notify_all();
            }
            for (size_t p = c.h; p < npieces; ++p)
                cudaMemcpyAsync(d_in + p * piece, reinterpret_cast<char*>(h_in) + p * piece, piece, cudaMemcpyHostToDevice, up);
            for (size_t p = 0; p < 8; ++p)
                cudaMemcpyAsync(reinterpret_cast<char*>(h_c) + p * piece, d_c + p * piece, piece, cudaMemcpyDeviceToHost, dn);
            for (size_t p = 0; p < c.h; ++p) {
                while (pool.left[p].load(std::memory_order_acquire) > 0) {}
                cudaMemcpyAsync(d_in + p * piece / 2, h_f16 + p * pe, piece / 2, cudaMemcpyHostToDevice, up);
            }
            cudaDeviceSynchronize();
            c.ms.push_back(now_ms() - t0);
        }
    for (auto& c : cfgs) {
        std::sort(c.ms.begin(), c.ms.end());
        std::printf("(c) hybrid T=%2u: %2zu of %zu pieces snapped on the host: up %.0f MiB + D2H 64 MiB: min %.3f median %.3f ms\n",
                    c.T, c.h, npieces, (c.h * piece / 2 + (npieces - c.h) * piece) / double(MB), c.ms.front(),
                    c.ms[c.ms.size() / 2]);
    }
    for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        double t0 = now_ms();
        for (size_t p = 0; p < npieces; ++p)
            cudaMemcpyAsync(d_in + p * piece, reinterpret_cast<char*>(h_in) + p * piece, piece, cudaMemcpyHostToDevice, up);
        for (size_t p = 0; p < 8; ++p)
            cudaMemcpyAsync(reinterpret_cast<char*>(h_c) + p * piece, d_c + p * piece, piece, cudaMemcpyDeviceToHost, dn);
        cudaDeviceSynchronize();
        std::printf("(a') again after (c): %.3f ms\n", now_ms() - t0);
    }
    {
        std::lock_guard<std::mutex> lk(pool.mu);
        pool.stop = true;
    }
    pool.cv.notify_all();
    for (auto& x : pool.th) x.join();
    return 0;
}
