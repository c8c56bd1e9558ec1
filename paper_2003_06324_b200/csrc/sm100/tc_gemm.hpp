// Host interface of the sm_100a tensor-core GEMM family (no CUDA headers needed
// beyond cudaStream_t).
#pragma once

#include <cuda_runtime.h>

namespace fireiron::sm100 {

constexpr int kTcOk = 0;
constexpr int kTcErrShape = 1;
constexpr int kTcErrUnsupported = 2;
constexpr int kTcErrTensorMap = 3;
constexpr int kTcErrCuda = 4;
constexpr int kTcErrCapture = 5;  // the workspace would be allocated inside a CUDA-graph capture

struct TcGemmConfig {
    int cta_group = 2;   // 1: tcgen05 cta_group::1, M tile 128; 2: CTA pair, M tile 256
    int bn = 256;        // N tile (UMMA N)
    int split_k = 1;     // CTAs of a cluster sharing one output tile (K slices)
    int ab_format = 0;   // 0 = f16, 1 = bf16
    int a_mn_major = 1;  // A col-major (Fireiron default)
    int b_mn_major = 0;  // B col-major => K-major (Fireiron default)
    int c_row_major = 0;
    int out_type = 0;    // 0 f32, 1 f16, 2 bf16
    int group_m = 8;     // raster band for the default tile order
    int stages = 0;      // pipeline depth (0 = deepest that fits in shared memory)
    int slabs = 1;       // 2: A slabs per CTA (pair tile 512 x 256, cta_group 2, BN 256)
    int n_halves = 1;    // 2: N halves sharing A (pair tile 256 x 512, cta_group 2, BN 256)
    int mcast = 1;       // 2: two CTA pairs (neighbours along N) share A stages by TMA multicast
};

struct TcWorkspace;

struct TcGemmProblem {
    const void* A = nullptr;
    const void* B = nullptr;
    void* C = nullptr;
    int M = 0, N = 0, K = 0;
    long lda = 0, ldb = 0, ldc = 0;  // elements, physical leading dimension
    const int* tile_order = nullptr; // device array, tiles_m*tiles_n entries, or null
    int num_sms = 148;
    int max_ctas = 0;                // 0 = persistent over all SMs
    int streamk = -1;                // -1 auto, 0 data-parallel, 1 K-slice tail, 2 N-split tail
    int force_slices = 0;            // >1: K-slice every tile into this many slices (.splitk on pairs)
    int remainder = 1;               // K-slice tails may add a remainder slice on idle clusters
    // stream-K partial workspace; null = the library pool, which keeps one
    // workspace per (device, stream) so only launches on the same stream share
    // one. A caller-owned workspace: launches that share it must be ordered on
    // one stream.
    TcWorkspace* workspace = nullptr;
    // gated B (fused all-gather): B's column chunks of b_chunk_n columns become
    // readable when b_ready[j] >= b_epoch; the schedule starts at chunk b_first_chunk
    const unsigned* b_ready = nullptr;
    unsigned b_epoch = 0;
    long b_chunk_n = 0;
    int b_first_chunk = 0;
};

// Device workspace of the stream-K fixup: one fp32 partial tile per CTA
// (clusters x cta_group x BN x 128) + one epoch flag per CTA.
struct TcWorkspace {
    float* partials = nullptr;
    unsigned* flags = nullptr;
    size_t partial_floats = 0, flag_count = 0;
    unsigned epoch = 0;  // incremented by every launch that uses it
    unsigned* ctr = nullptr;  // device {epoch, CTAs done}: the graph-safe epoch (GemmArgs::epoch_ctr)
    ~TcWorkspace();
};

struct TcLaunchInfo {
    int ctas = 0, clusters = 0, streamk = 0;
    int remainder = 0;  // K-slice tail: 1 remainder slices, 2 two-slice pull fixup
};
TcLaunchInfo tc_gemm_last_launch();

int tc_gemm_check(const TcGemmConfig& c, int M, int N, int K);
int tc_gemm_stages(const TcGemmConfig& c);
int tc_gemm_smem_bytes(const TcGemmConfig& c);
int tc_gemm_tmem_cols(const TcGemmConfig& c);
int tc_gemm_launch(const TcGemmConfig& cfg, const TcGemmProblem& p, cudaStream_t stream, bool dry_run = false);
// Grid / scheduling decision of a launch without launching (needs the device).
TcLaunchInfo tc_gemm_plan(const TcGemmConfig& cfg, const TcGemmProblem& p);

}  // namespace fireiron::sm100
