// Microbenchmark: the duplex floor for the host-snapped C2 byte counts --
// 64 MiB up (the f16 operands) against 64 MiB down (the fp32 result), linear
// copies on two streams, ungated, for several piece sizes; plus each direction
// alone. Host buffers from cudaHostAlloc (as the runtime's staging).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a pcie_balanced.cu -o pcie_balanced
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

int main() {
    const size_t mb = 1u << 20, n = 64 * mb;
    char *d_up, *d_down, *h_up, *h_down;
    cudaMalloc(&d_up, n);
    cudaMalloc(&d_down, n);
    cudaHostAlloc(reinterpret_cast<void**>(&h_up), n, cudaHostAllocPortable);
    cudaHostAlloc(reinterpret_cast<void**>(&h_down), n, cudaHostAllocPortable);
    for (size_t i = 0; i < n; i += 4096) h_up[i] = h_down[i] = 1;
    cudaMemset(d_down, 0, n);
    cudaStream_t su, sd;
    cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
    cudaEvent_t e0, eu, ed;
    cudaEventCreate(&e0);
    cudaEventCreate(&eu);
    cudaEventCreate(&ed);
    // down_line > 0: D2H as pitched copies of down_line-byte lines at 4x that pitch
    auto run = [&](size_t up_piece, size_t down_piece, bool up, bool down, size_t down_line = 0) {
        std::vector<float> t;
        for (int rep = 0; rep < 7; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, su);
            cudaStreamWaitEvent(sd, e0, 0);
            if (up)
                for (size_t o = 0; o < n; o += up_piece)
                    cudaMemcpyAsync(d_up + o, h_up + o, std::min(up_piece, n - o), cudaMemcpyHostToDevice, su);
            if (down)
                for (size_t o = 0; o < n; o += down_piece) {
                    const size_t len = std::min(down_piece, n - o);
                    if (down_line == 0)
                        cudaMemcpyAsync(h_down + o, d_down + o, len, cudaMemcpyDeviceToHost, sd);
                    else  // the same bytes as lines of down_line at pitch 4 * down_line (4 interleaved blocks)
                        cudaMemcpy2DAsync(h_down + (o / (4 * len)) * 4 * len + (o / len % 4) * down_line, 4 * down_line,
                                          d_down + o, 4 * down_line, down_line, len / down_line, cudaMemcpyDeviceToHost, sd);
                }
            cudaEventRecord(eu, su);
            cudaEventRecord(ed, sd);
            cudaDeviceSynchronize();
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, e0, eu);
            cudaEventElapsedTime(&b, e0, ed);
            t.push_back(std::max(a, b));
        }
        std::sort(t.begin(), t.end());
        const double ms = t[t.size() / 2];
        const double bytes = (up ? n : 0) + (down ? n : 0);
        std::printf("up %s piece %3zu MiB, down %s piece %3zu MiB lines %6zu: %.3f ms, %.1f GB/s total\n",
                    up ? "on " : "off", up_piece / mb, down ? "on " : "off", down_piece / mb, down_line, ms,
                    bytes / ms / 1e6);
    };
    for (size_t p : {2, 4, 8, 16, 64}) run(p * mb, p * mb, true, false);
    for (size_t p : {2, 4, 8, 16, 64}) run(p * mb, p * mb, false, true);
    for (size_t p : {2, 4, 8, 16, 64}) run(p * mb, p * mb, true, true);
    run(4 * mb, 16 * mb, true, true);
    run(16 * mb, 4 * mb, true, true);
    run(8 * mb, 16 * mb, true, true);
    run(4 * mb, 8 * mb, true, true);
    run(8 * mb, 4 * mb, true, true);
    for (size_t line : {4096, 8192, 16384}) {
        run(4 * mb, 4 * mb, false, true, line);
        run(4 * mb, 4 * mb, true, true, line);
        run(8 * mb, 8 * mb, true, true, line);
        run(8 * mb, 16 * mb, true, true, line);
    }
    return 0;
}
