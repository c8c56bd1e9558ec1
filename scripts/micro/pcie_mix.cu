// Microbenchmark: duplex PCIe throughput for copy mixes like the host
// pipelines' (runtime/plan.cpp HostIO): H2D pieces on one stream against D2H
// pieces on one or two streams, piece sizes given per direction, optionally
// while host threads stream through memory (the host snapping's load: read
// fp32, write half as many bytes) and with the upload source written by those
// threads just before (as the snapped staging is).
//   pcie_mix <up_MiB> <up_piece_MiB> <down_MiB> <down_piece_MiB> [down_streams] [host_load 0/1]
//            [down_line_bytes (0 = linear)]
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s up_MiB up_piece_MiB down_MiB down_piece_MiB [down_streams] [host_load] [down_line]\n",
                     argv[0]);
        return 2;
    }
    const size_t mb = 1u << 20;
    const size_t up = std::atof(argv[1]) * mb, upp = std::atof(argv[2]) * mb;
    const size_t dn = std::atof(argv[3]) * mb, dnp = std::atof(argv[4]) * mb;
    const int nds = argc > 5 ? std::atoi(argv[5]) : 1;
    const int load = argc > 6 ? std::atoi(argv[6]) : 0;
    const size_t line = argc > 7 ? std::atol(argv[7]) : 0;
    char *d_up, *d_dn, *h_up, *h_dn;
    float *h_src = nullptr, *h_dst = nullptr;
    cudaMalloc(&d_up, up);
    cudaMalloc(&d_dn, 4 * dn);
    cudaHostAlloc(reinterpret_cast<void**>(&h_up), up, cudaHostAllocPortable);
    cudaHostAlloc(reinterpret_cast<void**>(&h_dn), 4 * dn, cudaHostAllocPortable);
    std::memset(h_up, 1, up);
    std::memset(h_dn, 1, 4 * dn);
    const size_t load_bytes = 128 * mb;
    if (load) {
        cudaHostAlloc(reinterpret_cast<void**>(&h_src), load_bytes, cudaHostAllocPortable);
        cudaHostAlloc(reinterpret_cast<void**>(&h_dst), load_bytes / 2, cudaHostAllocPortable);
        std::memset(h_src, 0, load_bytes);
    }
    cudaStream_t su, sd[2];
    cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking);
    for (auto& s : sd) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, eu, ed[2];
    cudaEventCreate(&e0);
    cudaEventCreate(&eu);
    for (auto& e : ed) cudaEventCreate(&e);
    const int nthreads = 15;
    std::vector<float> t;
    for (int rep = 0; rep < 9; ++rep) {
        cudaDeviceSynchronize();
        std::atomic<bool> stop{false};
        std::vector<std::thread> th;
        if (load == 2) {  // the upload source written by the threads first (NT stores)
            for (int i = 0; i < nthreads; ++i)
                th.emplace_back([&, i] {
                    const size_t per = up / nthreads & ~size_t(63);
                    char* p = h_up + i * per;
                    const __m512i z = _mm512_set1_epi32(i);
                    for (size_t o = 0; o < per; o += 64) _mm512_stream_si512(reinterpret_cast<__m512i*>(p + o), z);
                    _mm_sfence();
                });
            for (auto& x : th) x.join();
            th.clear();
        }
        if (load)
            for (int i = 0; i < nthreads; ++i)
                th.emplace_back([&, i] {
                    const size_t n = load_bytes / 4 / nthreads & ~size_t(15);
                    const float* s = h_src + i * n;
                    unsigned short* d = reinterpret_cast<unsigned short*>(h_dst) + i * n;
                    while (!stop.load(std::memory_order_relaxed))
                        for (size_t o = 0; o < n && !stop.load(std::memory_order_relaxed); o += 16) {
                            __m256i h = _mm512_cvtps_ph(_mm512_loadu_ps(s + o), 0);
                            _mm256_stream_si256(reinterpret_cast<__m256i*>(d + o), h);
                        }
                });
        cudaEventRecord(e0, su);
        for (int k = 0; k < nds; ++k) cudaStreamWaitEvent(sd[k], e0, 0);
        size_t ou = 0, od = 0;
        int k = 0;
        // interleave enqueue order roughly by bytes (as the pipelines do)
        while (ou < up || od < dn) {
            if (ou < up && (od >= dn || ou * dn <= od * up)) {
                const size_t len = std::min(upp, up - ou);
                cudaMemcpyAsync(d_up + ou, h_up + ou, len, cudaMemcpyHostToDevice, su);
                ou += len;
            } else {
                const size_t len = std::min(dnp, dn - od);
                if (line == 0)
                    cudaMemcpyAsync(h_dn + od, d_dn + od, len, cudaMemcpyDeviceToHost, sd[k]);
                else  // lines of `line` bytes at a 4x pitch
                    cudaMemcpy2DAsync(h_dn + od * 4, 4 * line, d_dn + od * 4, 4 * line, line, len / line,
                                      cudaMemcpyDeviceToHost, sd[k]);
                k = (k + 1) % nds;
                od += len;
            }
        }
        cudaEventRecord(eu, su);
        for (int j = 0; j < nds; ++j) cudaEventRecord(ed[j], sd[j]);
        cudaDeviceSynchronize();
        stop = true;
        for (auto& x : th) x.join();
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, e0, eu);
        for (int j = 0; j < nds; ++j) {
            float c = 0;
            cudaEventElapsedTime(&c, e0, ed[j]);
            b = std::max(b, c);
        }
        if (rep >= 2) t.push_back(std::max(a, b));
    }
    std::sort(t.begin(), t.end());
    const double ms = t[t.size() / 2];
    std::printf("up %5.0f MiB in %5.1f MiB, down %5.0f MiB in %5.1f MiB (%d streams, lines %zu), host load %d: %.3f ms, %.1f GB/s\n",
                double(up) / mb, double(upp) / mb, double(dn) / mb, double(dnp) / mb, nds, line, load, ms,
                double(up + dn) / ms / 1e6);
    return 0;
}
