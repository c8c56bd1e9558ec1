// Throughput of the product host snap (fi_host_snap_f32) on T threads, 128 MiB of fp32.
// g++ -O2 -o scripts/micro/snap_rate scripts/micro/snap_rate.cpp -L paper_2003_06324_b200/_lib -lfireiron_b200 -Wl,-rpath,$PWD/paper_2003_06324_b200/_lib -lpthread
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>
#include <cstdint>
extern "C" int fi_host_snap_f32(const float* src, void* dst, int64_t count, int elem);
int main() {
    const size_t n = 32u << 20, piece = 256 * 1024;
    float* src = (float*)aligned_alloc(4096, n * 4);
    uint16_t* dst = (uint16_t*)aligned_alloc(4096, n * 2);
    for (size_t i = 0; i < n; ++i) src[i] = (float)((i * 2654435761u) % 2001) / 1000.f - 1.f;
    memset(dst, 0, n * 2);
    for (int elem = 1; elem <= 2; ++elem)
        for (int T : {1, 2, 4, 8, 16}) {
            double best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                std::atomic<size_t> next{0};
                auto t0 = std::chrono::steady_clock::now();
                std::vector<std::thread> th;
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&] {
                        for (size_t p; (p = next.fetch_add(1)) < n / piece;)
                            fi_host_snap_f32(src + p * piece, dst + p * piece, piece, elem);
                    });
                for (auto& x : th) x.join();
                best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            }
            printf("%s T=%d: %.1f GB/s of fp32 in\n", elem == 1 ? "f16" : "bf16", T, n * 4 / best / 1e9);
        }
}
