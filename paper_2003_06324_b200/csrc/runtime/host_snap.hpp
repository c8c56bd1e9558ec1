// Host-side snapping of fp32 input panels to the f16 / bf16 grid, in parallel
// with the copy engine (run_host's blocked pipeline, plan.cpp).
//
// anvil::run ingests fp32 matrices and snaps F16 roots to the f16 grid
// (proj/include/anvil/sim.hpp:507-510, round_to_f16 matrix.hpp:67-80). Done on
// the device, every input element crosses PCIe as 4 bytes; snapped by host
// cores into a pinned staging buffer first, it crosses as 2. The host cores
// convert ~100 GB/s of fp32 on the B200 box's 16 vCPUs and the copy engine
// moves ~54 GB/s, so converting on the host is faster than uploading fp32
// (profiles/round2/host_snap_probe.txt). Results are bit-identical to the
// device conversion (runtime/convert.cu): f16 is IEEE RNE with the reference's
// saturation of finite |x| >= 2^16 to +-65504, bf16 is IEEE RNE, NaN becomes
// the canonical 0x7FFF of cvt.rn.
#pragma once

#include <atomic>
#include <cstdint>

namespace fireiron::rt {

// One 2D region: `height` lines of `width` elements, line i at src + i * spitch
// (floats) and dst + i * dpitch (elements of the target type). elem 0 copies
// fp32 (staging a pageable result into / out of pinned memory).
struct SnapJob {
    const float* src = nullptr;
    void* dst = nullptr;
    long width = 0, height = 0, spitch = 0, dpitch = 0;
    int elem = 1;  // 0 f32 copy, 1 f16, 2 bf16
    // filled by the pool
    long lines_per_piece = 0, npieces = 0;
    std::atomic<long> next{0}, done{0};
};

// Process-wide worker pool. Jobs are taken FIFO piece by piece (~1 MiB of
// fp32 each); wait() lets the calling thread convert pieces of that job too.
class HostSnapPool {
   public:
    // nullptr when host snapping is disabled (FI_HOST_SNAP=0) or the CPU lacks
    // F16C/AVX2. Workers: FI_HOST_SNAP_THREADS, else the CPUs this process may
    // run on, minus the calling thread.
    static HostSnapPool* get();
    int workers() const { return nworkers_; }
    // The job must stay alive until wait(job) returns.
    void submit(SnapJob* job);
    void wait(SnapJob* job);

   private:
    HostSnapPool(int n);
    void worker();
    bool run_one();  // convert one piece of the oldest unfinished job; false if none
    int nworkers_;
};

// Single-threaded conversion of n elements (tests and the pool's pieces).
void snap_f32(const float* src, uint16_t* dst, long n, int elem);
bool host_snap_supported();

}  // namespace fireiron::rt
