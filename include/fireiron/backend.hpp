// GPU execution backend: the drop-in for the reference's execution call
//   RunResult anvil::run(const Program&, const Matrix& a, const Matrix* b, RunOptions)
//   (proj/include/anvil/sim.hpp:495, tree overload :536)
// and its code generator seam (anvil::generate, codegen.hpp:275/291).
//
// A Program is executed on a B200 by one of two lowerings, chosen from the
// bound leaves:
//   * tensor-core strategies (TMA_LOAD / UMMA / TMEM_* leaves) map onto the
//     hand-written tcgen05 kernel family (sm100/gemm_kernel.cuh);
//   * every other simulatable tree (FMA / HFMA / COPY / WMMA leaves) is
//     emitted as sm_100a CUDA from the Program and compiled at runtime with
//     NVRTC (--fmad=false: the FMA leaf is bit-exact with the reference's
//     sequential-k, unfused fp32 semantics, sim.hpp:370-376).
// There is no CPU execution path.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "fireiron/matrix.hpp"
#include "fireiron/program.hpp"
#include "fireiron/script.hpp"

namespace fireiron {

// --- reference-compatible result types (sim.hpp:18-58) ---------------------
struct AccessRecord {
    long phase = 0, block = 0, thread = 0;
    char op = 'R';
    std::string buffer;
    long index = 0;
};
struct RaceRecord {
    std::string buffer;
    long index = 0;
    long writer = 0, other = 0;
    long phase = 0, block = 0;
};
struct RaceReport {
    std::vector<RaceRecord> records;
    long total = 0;
    bool empty() const { return total == 0; }
};
struct OwnershipRecord {
    std::string buffer;
    long index = 0;
    long owner = -1, accessor = 0, block = 0;
};

struct RunOptions {
    bool collect_ownership = false;  // accepted for compatibility; the GPU does not track owners
    bool log_accesses = false;       // accepted for compatibility; no access log on the GPU
    int device = 0;
    void* stream = nullptr;          // cudaStream_t; null = a plan-owned stream
};

struct RunResult {
    Matrix output;
    RaceReport races;
    std::vector<OwnershipRecord> ownership;
    std::vector<AccessRecord> log;
    double device_ms = 0.0;  // kernel time (CUDA events) of this run
};

// --- code generation ------------------------------------------------------
struct KernelSource {
    std::string source;
    LaunchConfig launch;
    BufferPlan plan;
    std::string entry_name;
};

// Emits the sm_100a translation unit for a validated tree. Deterministic.
// The shared-memory gate is the B200 per-CTA budget (227 KiB).
KernelSource generate(const Spec& root, const NodePtr& tree, const MicroKernelSet& mks = MicroKernelSet{});
KernelSource generate(const Program& prog);

// --- tensor-core strategy recognition --------------------------------------
struct TcStrategy {
    bool matched = false;
    std::string why_not;   // reason when not a tcgen05 strategy
    int cta_group = 1;     // .pair -> 2
    int tile_m = 128, tile_n = 128, tile_k = 64;
    int split_k = 1;       // .splitk ranks per output tile
    int mcast = 1;         // .multicast: 2 pair units along N share A stages
    int stages = 0;        // .stages (0 = deepest that fits)
    std::vector<int32_t> tile_order;  // Block .swizzle/.layout schedule, empty = default raster
};
TcStrategy match_tc_strategy(const Spec& root, const NodePtr& tree, const MicroKernelSet& mks = MicroKernelSet{});

// --- compiled plans --------------------------------------------------------
struct PlanInfo {
    int kind = 0;  // 0 generic (NVRTC), 1 tcgen05
    long grid_x = 1, grid_y = 1, block_threads = 1;
    long launch_ctas = 0;
    int cluster = 1, stages = 0, tmem_cols = 0, cta_group = 1, tile_m = 0, tile_n = 0, split_k = 1;
    int streamk = 0;  // tcgen05 plans: 0 data-parallel, 1 K-sliced tail/split, 2 N-split tail
    int remainder = 0;  // K-slice tail: 1 remainder slices on the idle clusters, 2 two-slice pull fixup
    int splitk_global = 0;  // .splitk lowered to cross-cluster K slices (else DSMEM cluster)
    long shared_bytes = 0;
    double flops = 0.0;
    std::string entry_name;
};

class Plan {
public:
    // parse/lower/emit/compile; throws fireiron::Error, or BackendError below
    static std::shared_ptr<Plan> create(const Spec& root, const NodePtr& tree,
                                        const MicroKernelSet& mks = MicroKernelSet{}, int device = 0);
    static std::shared_ptr<Plan> from_script(const std::string& script, long m = 0, long n = 0, long k = 0,
                                             int device = 0);
    ~Plan();

    // device buffers in the root element types and layouts; stream-ordered
    void launch(const void* dA, const void* dB, void* dC, void* stream) const;
    // tensor-core plans: B column chunks of chunk_cols gated by ready[j] >= epoch
    // (fi_plan_launch_gated), tile schedule starting at chunk first_chunk
    void launch_gated(const void* dA, const void* dB, void* dC, void* stream, const unsigned* ready,
                      unsigned epoch, long chunk_cols, int first_chunk) const;
    // anvil::run semantics on host fp32 matrices (grid snapping on ingestion)
    RunResult run_host(const Matrix& a, const Matrix* b, void* stream = nullptr) const;
    // Same on raw host fp32 arrays in the root physical layouts (extent
    // elements each; pinned memory makes the copies asynchronous DMA).
    // Returns the kernel time in ms.
    double run_host_raw(const float* A, const float* B, float* C, void* stream = nullptr) const;
    // bytes the last run_host moved host -> device and device -> host
    void last_host_bytes(long& up, long& down) const;

    const PlanInfo& info() const;
    const Program& program() const;
    const std::string& source() const;

    struct Impl;

private:
    explicit Plan(std::unique_ptr<Impl> impl);
    std::unique_ptr<Impl> impl_;
};

// Non-IR failures (CUDA / NVRTC / unsupported lowering). status mirrors the
// C ABI codes (include/fireiron_b200.h).
class BackendError : public std::runtime_error {
public:
    BackendError(int status, const std::string& msg) : std::runtime_error(msg), status_(status) {}
    int status() const { return status_; }

private:
    int status_;
};

// --- the execution seam ----------------------------------------------------
// anvil::run (proj/include/anvil/sim.hpp:495 / :536) with the same signatures
// and semantics (C = A*B from a zero C, F16 roots snapped on ingestion, output
// in C's root layout), executed on the B200 instead of the CPU model.
RunResult run(const Program& prog, const Matrix& a, const Matrix* b = nullptr, RunOptions opts = {});
RunResult run(const Spec& root, const NodePtr& tree, const Matrix& a, const Matrix* b = nullptr,
              RunOptions opts = {}, const MicroKernelSet& mks = MicroKernelSet{});

// The names SURVEY.md 8(b) gives the GPU entry points: run_gpu is run (which
// already executes on the GPU); GpuRunOptions carries the device, the stream
// and -- through RunResult::device_ms -- the kernel timing.
using GpuRunOptions = RunOptions;
inline RunResult run_gpu(const Program& prog, const Matrix& a, const Matrix* b = nullptr, GpuRunOptions opts = {}) {
    return run(prog, a, b, opts);
}
inline RunResult run_gpu(const Spec& root, const NodePtr& tree, const Matrix& a, const Matrix* b = nullptr,
                         GpuRunOptions opts = {}, const MicroKernelSet& mks = MicroKernelSet{}) {
    return run(root, tree, a, b, opts, mks);
}

}  // namespace fireiron
