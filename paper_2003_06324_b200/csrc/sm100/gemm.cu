// Host side of the tcgen05 GEMM family: TMA descriptor encoding, kernel
// selection by (cta_group, BN, split-K) and cluster launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <map>
#include <memory>
#include <mutex>
#include <utility>

#include "gemm_kernel.cuh"
#include "tc_gemm.hpp"

namespace fireiron::sm100 {

namespace {

// The driver entry point is resolved through the runtime so the library loads
// (and its IR services work) on hosts without libcuda.so.1.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

CUresult encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t d0,
                   uint64_t d1, uint64_t stride1_bytes, uint32_t box0, uint32_t box1,
                   CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFn encode = encode_tiled_fn();
    if (!encode) return CUDA_ERROR_NOT_INITIALIZED;
    cuuint64_t dims[2] = {d0, d1};
    cuuint64_t strides[1] = {stride1_bytes};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t estr[2] = {1, 1};
    return encode(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

thread_local TcLaunchInfo g_last;

// Library pool for callers without their own workspace: one workspace per
// (device, stream), so launches that share one are stream-ordered. The caller
// of tc_gemm_launch holds pool_mutex() while the launch is enqueued.
std::mutex& pool_mutex() {
    static std::mutex mu;
    return mu;
}

TcWorkspace* pool_workspace(int device, cudaStream_t stream) {
    static std::map<std::pair<int, cudaStream_t>, std::unique_ptr<TcWorkspace>> pool;
    auto& ws = pool[{device, stream}];
    if (!ws) ws = std::make_unique<TcWorkspace>();
    return ws.get();
}

// Per-device state of one kernel instance: function attributes apply per
// device context, and the occupancy cap stream-K relies on is a property of
// the device the launch goes to.
struct DeviceState {
    bool attr_done = false;
    cudaError_t attr_err = cudaSuccess;
    int max_active = -1;
};
constexpr int kMaxDevices = 64;

CUresult encode_nd(CUtensorMap* map, CUtensorMapDataType dt, const void* base, int rank, const cuuint64_t* dims,
                   const cuuint64_t* strides, const cuuint32_t* box) {
    EncodeTiledFn encode = encode_tiled_fn();
    if (!encode) return CUDA_ERROR_NOT_INITIALIZED;
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(map, dt, rank, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <int kCtaGroup, int BN, int kSplitK, int kSlabs = 1, int kNHalves = 1, int kMcast = 1, int kKB = 1>
int launch_impl(const TcGemmConfig& cfg, const TcGemmProblem& p, cudaStream_t stream, bool dry_run = false) {
    using S = GemmShape<kCtaGroup, BN, kSplitK, kSlabs, kNHalves, kKB>;
    auto kernel = fi_sm100_gemm<kCtaGroup, BN, kSplitK, kSlabs, kNHalves, kMcast, kKB>;
    constexpr int kCluster = kCtaGroup * kSplitK * kMcast;

    const CUtensorMapDataType dt =
        cfg.ab_format == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUtensorMap tmA, tmB, tmB2, tmC, tmC2;
    CUresult r;
    const cuuint64_t kblocks = static_cast<cuuint64_t>(p.K / 64);
    if (kKB == 2 && cfg.a_mn_major) {
        // (64 rows, 64 k, M/64 panels, K/64 blocks): box {64, 64, 2, 2} = both panels of two K blocks
        cuuint64_t dims[4] = {64, 64, static_cast<cuuint64_t>(p.M / 64), kblocks};
        cuuint64_t strides[3] = {static_cast<cuuint64_t>(p.lda) * 2, 128, static_cast<cuuint64_t>(p.lda) * 128};
        cuuint32_t box[4] = {64, 64, 2, 2};
        r = encode_nd(&tmA, dt, p.A, 4, dims, strides, box);
    } else if (kKB == 2) {
        // K-major: (64 k, M rows, K/64 blocks): box {64, 128, 2}
        cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(p.M), kblocks};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.lda) * 2, 128};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(S::BM), 2};
        r = encode_nd(&tmA, dt, p.A, 3, dims, strides, box);
    } else if (cfg.a_mn_major && kMcast == 1) {
        // (64 rows, K, M/64 panels): box {64, 64, 2} = one slab's two SW128 panels
        EncodeTiledFn encode = encode_tiled_fn();
        cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(p.K), static_cast<cuuint64_t>(p.M / 64)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.lda) * 2, 128};
        cuuint32_t box[3] = {64, 64, 2};
        cuuint32_t estr[3] = {1, 1, 1};
        r = encode ? encode(&tmA, dt, 3, const_cast<void*>(p.A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                   : CUDA_ERROR_NOT_INITIALIZED;
    } else if (cfg.a_mn_major)
        r = encode_2d(&tmA, dt, p.A, p.M, p.K, static_cast<uint64_t>(p.lda) * 2, 64, 64);
    else
        r = encode_2d(&tmA, dt, p.A, p.K, p.M, static_cast<uint64_t>(p.lda) * 2, 64, kMcast > 1 ? 64 : S::BM);
    if (r != CUDA_SUCCESS) return kTcErrTensorMap;
    if (cfg.b_mn_major) {
        r = encode_2d(&tmB, dt, p.B, p.N, p.K, static_cast<uint64_t>(p.ldb) * 2, 64, 64);
    } else if (kKB == 2) {
        // K-major: (64 k, N rows, K/64 blocks): box {64, BN_LOCAL, 2}
        cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(p.N), kblocks};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.ldb) * 2, 128};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(S::BN_LOCAL), 2};
        r = encode_nd(&tmB, dt, p.B, 3, dims, strides, box);
    } else {
        r = encode_2d(&tmB, dt, p.B, p.K, p.N, static_cast<uint64_t>(p.ldb) * 2, 64, S::BN_LOCAL);
    }
    if (r == CUDA_SUCCESS && !cfg.b_mn_major && S::BN_LOCAL >= 16) {  // half-width tail units
        if (kKB == 2) {
            cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(p.N), kblocks};
            cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.ldb) * 2, 128};
            cuuint32_t box[3] = {64, static_cast<cuuint32_t>(S::BN_LOCAL / 2), 2};
            r = encode_nd(&tmB2, dt, p.B, 3, dims, strides, box);
        } else {
            r = encode_2d(&tmB2, dt, p.B, p.K, p.N, static_cast<uint64_t>(p.ldb) * 2, 64, S::BN_LOCAL / 2);
        }
    } else {
        tmB2 = tmB;
    }
    if (r != CUDA_SUCCESS) return kTcErrTensorMap;
    // f32 column-major C: the epilogue stages 128x32 chunks in smem and stores
    // them with one TMA bulk tensor store each (FI_TC_CSTORE=0 disables)
    static const bool cstore_env = [] {
        const char* v = std::getenv("FI_TC_CSTORE");
        return !(v && v[0] == '0');
    }();
    const bool c_tma = cstore_env && kSplitK == 1 && cfg.out_type == 0 && !cfg.c_row_major &&
                       (static_cast<uint64_t>(p.ldc) * 4) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(p.C) & 15) == 0;
    if (c_tma) {
        r = encode_2d(&tmC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p.C, p.M, p.N, static_cast<uint64_t>(p.ldc) * 4,
                      S::BM, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (r != CUDA_SUCCESS) return kTcErrTensorMap;
        // 64-column box: two adjacent staged chunks in one store
        r = encode_2d(&tmC2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, p.C, p.M, p.N, static_cast<uint64_t>(p.ldc) * 4,
                      S::BM, 64, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (r != CUDA_SUCCESS) return kTcErrTensorMap;
    } else {
        tmC = tmA;  // unused
        tmC2 = tmA;
    }

    GemmArgs args;
    args.C = p.C;
    args.ldc = p.ldc;
    args.M = p.M;
    args.N = p.N;
    args.K = p.K;
    args.tiles_m = p.M / S::BM_TILE;
    args.tiles_n = p.N / (S::BN_TILE * kMcast);  // scheduled units span both pairs of a multicast cluster
    args.k_blocks = p.K / S::BK / kSplitK;
    args.ab_format = cfg.ab_format;
    args.a_mn_major = cfg.a_mn_major;
    args.b_mn_major = cfg.b_mn_major;
    args.c_row_major = cfg.c_row_major;
    args.out_type = cfg.out_type;
    args.group_m = cfg.group_m > 0 ? cfg.group_m : 8;
    args.tile_order = p.tile_order;
    if (p.b_ready) {
        const long unit_n = static_cast<long>(S::BN_TILE) * kMcast;
        if (p.tile_order || p.b_chunk_n <= 0 || p.b_chunk_n % unit_n != 0 || p.N % p.b_chunk_n != 0)
            return kTcErrShape;
        args.b_ready = p.b_ready;
        args.b_epoch = p.b_epoch;
        args.b_chunk_tiles = static_cast<int>(p.b_chunk_n / unit_n);
        args.n_rot = (p.b_first_chunk * args.b_chunk_tiles) % args.tiles_n;
    }
    args.stages = cfg.stages;
    args.c_tma = c_tma ? 1 : 0;
    static const bool ring_drain_env = [] {
        const char* v = std::getenv("FI_TC_RING_DRAIN");
        return !(v && v[0] == '0');
    }();
    args.ring_drain = ring_drain_env ? 1 : 0;
    static const int l2_hint_env = [] {
        const char* v = std::getenv("FI_TC_L2HINT");
        return v ? std::atoi(v) : 0;
    }();
    args.l2_hint = l2_hint_env;

    static std::mutex dev_mu;
    static DeviceState dev_state[kMaxDevices];
    int device = 0;
    if (cudaGetDevice(&device) != cudaSuccess || device < 0 || device >= kMaxDevices) return kTcErrCuda;
    std::unique_lock<std::mutex> dev_lock(dev_mu);
    DeviceState& ds = dev_state[device];
    if (!ds.attr_done) {
        ds.attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
        if (ds.attr_err == cudaSuccess && kCluster > 8)
            ds.attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        ds.attr_done = true;
    }
    if (ds.attr_err != cudaSuccess) return kTcErrCuda;

    const int tiles = args.tiles_m * args.tiles_n;
    int sms = p.num_sms > 0 ? p.num_sms : 148;
    int clusters = sms / kCluster;
    if (p.max_ctas > 0 && p.max_ctas / kCluster < clusters) clusters = p.max_ctas / kCluster;

    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(clusters * kCluster, 1, 1);
    lc.blockDim = dim3(S::kThreads, 1, 1);
    lc.dynamicSmemBytes = S::SMEM_BYTES;
    lc.stream = stream;
    cudaLaunchAttribute attrs[2];
    int nattr = 0;
    if (kCluster > 1) {
        attrs[0].id = cudaLaunchAttributeClusterDimension;
        attrs[0].val.clusterDim.x = kCluster;
        attrs[0].val.clusterDim.y = 1;
        attrs[0].val.clusterDim.z = 1;
        nattr = 1;
    }
    lc.attrs = attrs;
    lc.numAttrs = nattr;

    // Stream-K needs every cluster co-resident (owners spin on later
    // segments' flags): cap the grid at the occupancy limit.
    if (ds.max_active < 0) {
        lc.gridDim = dim3(clusters * kCluster, 1, 1);
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kernel, &lc) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = clusters;
        }
        ds.max_active = n;
    }
    if (clusters > ds.max_active) clusters = ds.max_active;
    dev_lock.unlock();
    const int kb = args.k_blocks;
    // FI_TC_PULL_D: publish time of the 2-slice pull fixup in K-blocks (-1 disables)
    static const int pull_d_env = [] {
        const char* v = std::getenv("FI_TC_PULL_D");
        return v ? std::atoi(v) : BN / 32;
    }();
    static const int head_env = [] {
        const char* v = std::getenv("FI_TC_HEAD");
        return v ? std::atoi(v) : 1;
    }();
    // slab / N-half tiles (512 x 256, 256 x 512 pair tiles) run whole tiles only: no tail split
    const SchedulePlan plan = kSlabs * kNHalves * kMcast > 1 ? plan_schedule<kCtaGroup, BN, kSplitK>(tiles, kb, clusters, cfg.b_mn_major != 0,
                                                                                0, 0, 0, -1, 0)
                                         : plan_schedule<kCtaGroup, BN, kSplitK>(
                                               tiles, kb, clusters, cfg.b_mn_major != 0, p.streamk, p.force_slices,
                                               p.remainder, pull_d_env, head_env);
    if (plan.status != 0) return kTcErrShape;
    const int mode = plan.mode;
    const bool sk = mode != 0;
    if (dry_run) {
        g_last = TcLaunchInfo{plan.clusters * kCluster, plan.clusters, mode, plan.sk_pull ? 2 : plan.sk_w > 0 ? 1 : 0};
        return kTcOk;
    }
    if (sk) {
        args.sk_tile_begin = plan.sk_begin;
        args.sk_slices = plan.slices;
        args.sk_w = plan.sk_w;
        args.sk_extra = plan.sk_extra;
        args.sk_q = plan.sk_q;
        args.sk_pull = plan.sk_pull;
        args.sk_head = plan.sk_head;
        TcWorkspace* ws = p.workspace ? p.workspace : pool_workspace(device, stream);
        const size_t slots = static_cast<size_t>(plan.slots);
        const size_t need_p = slots * kCtaGroup * S::WS_FLOATS;
        const size_t need_f = slots * kCtaGroup;
        // memory allocated while a stream is being captured would belong to the
        // graph: the plan must have run once (outside the capture) first
        if (ws->partial_floats < need_p || ws->flag_count < need_f || !ws->ctr) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (cudaStreamIsCapturing(stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
                return kTcErrCapture;
        }
        // growth is stream-ordered (cudaFreeAsync / cudaMallocAsync): a launch that
        // needs a larger workspace must not synchronise the device, e.g. inside
        // the host pipeline while uploads are still in flight
        if (ws->partial_floats < need_p) {
            const size_t grow = need_p + need_p / 4;
            if (ws->partials) cudaFreeAsync(ws->partials, stream);
            ws->partials = nullptr;
            if (cudaMallocAsync(&ws->partials, grow * sizeof(float), stream) != cudaSuccess) return kTcErrCuda;
            ws->partial_floats = grow;
        }
        if (ws->flag_count < need_f) {
            if (ws->flags) cudaFreeAsync(ws->flags, stream);
            ws->flags = nullptr;
            if (cudaMallocAsync(&ws->flags, need_f * sizeof(unsigned), stream) != cudaSuccess) return kTcErrCuda;
            if (cudaMemsetAsync(ws->flags, 0, need_f * sizeof(unsigned), stream) != cudaSuccess) return kTcErrCuda;
            ws->flag_count = need_f;
            ws->epoch = 0;
        }
        if (!ws->ctr) {
            if (cudaMallocAsync(&ws->ctr, 2 * sizeof(unsigned), stream) != cudaSuccess) return kTcErrCuda;
            if (cudaMemsetAsync(ws->ctr, 0, 2 * sizeof(unsigned), stream) != cudaSuccess) return kTcErrCuda;
        }
        args.streamk = mode;
        args.workspace = ws->partials;
        args.flags = ws->flags;
        args.epoch = ++ws->epoch;
        args.epoch_ctr = ws->ctr;
    }
    clusters = plan.clusters;
    lc.gridDim = dim3(clusters * kCluster, 1, 1);
    g_last = TcLaunchInfo{clusters * kCluster, clusters, mode, plan.sk_pull ? 2 : plan.sk_w > 0 ? 1 : 0};
    // debugging aid: FI_TC_TRACE=<file> records a per-unit timeline of this launch
    const char* trace_path = std::getenv("FI_TC_TRACE");
    static unsigned long long* trace_buf = nullptr;
    const size_t trace_n = static_cast<size_t>(clusters) * kCluster * 16 * 16;
    if (trace_path) {
        if (!trace_buf) cudaMalloc(&trace_buf, 148 * 16 * 16 * sizeof(unsigned long long));
        cudaMemsetAsync(trace_buf, 0, trace_n * sizeof(unsigned long long), stream);
        args.trace = trace_buf;
    }
    // stream-K owners spin on flags other clusters publish, so every CTA must be
    // resident at once: a cooperative launch guarantees it even when kernels on
    // other streams hold SMs (two concurrent stream-K launches could otherwise
    // each wait on CTAs of their own that cannot be scheduled)
    static const bool coop_env = [] {
        const char* v = std::getenv("FI_TC_COOP");
        if (v) return v[0] != '0';
        // Nsight Compute replays each launch in passes and rejects cooperative
        // cluster launches (LaunchFailed): under a Nsight tool launch normally
        // (the kernel is profiled alone, so co-residency is not at risk)
        return !(std::getenv("NV_TPS_LAUNCH_TOKEN") || std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") ||
                 std::getenv("CUDA_INJECTION64_PATH"));
    }();
    if (sk && coop_env) {
        attrs[lc.numAttrs].id = cudaLaunchAttributeCooperative;
        attrs[lc.numAttrs].val.cooperative = 1;
        ++lc.numAttrs;
    }
    cudaError_t e = cudaLaunchKernelEx(&lc, kernel, tmA, tmB, tmB2, tmC, tmC2, args);
    if (trace_path && e == cudaSuccess) {
        std::vector<unsigned long long> h(trace_n);
        cudaMemcpyAsync(h.data(), trace_buf, trace_n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        if (FILE* f = std::fopen(trace_path, "a")) {
            std::fprintf(f, "launch ctas %d cluster %d mode %d tiles %d kb %d\n", clusters * kCluster, kCluster,
                         args.streamk, tiles, kb);
            // cta unit t0 t1 t2 t3 clk0 clk1 t4 t5 t6 clk2 clk6 t7 (globaltimer ns, clock64)
            for (size_t i = 0; i < trace_n; i += 16)
                if (h[i] || h[i + 2] || h[i + 7])
                    std::fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", i / 256,
                                 (i / 16) % 16, h[i], h[i + 1], h[i + 2], h[i + 3], h[i + 8], h[i + 9], h[i + 4], h[i + 5],
                                 h[i + 6], h[i + 10], h[i + 14], h[i + 7]);
            // diagnostic builds (FI_TC_WAITPROF): MMA full-wait / loop cycles, producer
            // empty-wait / loop cycles, K blocks
            for (size_t i = 15 * 16; i < trace_n; i += 256)
                if (h[i + 9] || h[i + 11])
                    std::fprintf(f, "wait %zu %llu %llu %llu %llu %llu\n", i / 256, h[i + 8], h[i + 9], h[i + 10],
                                 h[i + 11], h[i + 12]);
            std::fclose(f);
        }
    }
    return e == cudaSuccess ? kTcOk : kTcErrCuda;
}

}  // namespace

TcWorkspace::~TcWorkspace() {
    if (partials) cudaFree(partials);
    if (flags) cudaFree(flags);
    if (ctr) cudaFree(ctr);
}

TcLaunchInfo tc_gemm_last_launch() { return g_last; }

int tc_gemm_stages(const TcGemmConfig& c) {
#define FI_STAGES(CG, BN, SK)                                          \
    if (c.cta_group == CG && c.bn == BN && c.split_k == SK && c.slabs == 1 && c.n_halves == 1) { \
        const int mx = GemmShape<CG, BN, SK>::kStages;                 \
        return (c.stages > 0 && c.stages < mx) ? c.stages : mx;        \
    }
    FI_STAGES(1, 64, 1) FI_STAGES(1, 128, 1) FI_STAGES(1, 256, 1)
    FI_STAGES(2, 64, 1) FI_STAGES(2, 128, 1) FI_STAGES(2, 256, 1)
    if (c.cta_group == 2 && c.bn == 256 && c.split_k == 1 && (c.slabs == 2 || c.n_halves == 2)) {
        const int mx = c.slabs == 2 ? GemmShape<2, 256, 1, 2>::kStages : GemmShape<2, 256, 1, 1, 2>::kStages;
        return (c.stages > 0 && c.stages < mx) ? c.stages : mx;
    }
    FI_STAGES(1, 64, 2) FI_STAGES(1, 128, 2) FI_STAGES(1, 128, 4) FI_STAGES(1, 256, 2) FI_STAGES(1, 256, 4) FI_STAGES(2, 256, 2) FI_STAGES(2, 256, 4) FI_STAGES(2, 128, 2) FI_STAGES(2, 128, 4)
#undef FI_STAGES
    return 0;
}

int tc_gemm_smem_bytes(const TcGemmConfig& c) {
#define FI_SMEM(CG, BN, SK) \
    if (c.cta_group == CG && c.bn == BN && c.split_k == SK && c.slabs == 1 && c.n_halves == 1) return GemmShape<CG, BN, SK>::SMEM_BYTES;
    if (c.cta_group == 2 && c.bn == 256 && c.split_k == 1 && c.slabs == 2) return GemmShape<2, 256, 1, 2>::SMEM_BYTES;
    if (c.cta_group == 2 && c.bn == 256 && c.split_k == 1 && c.n_halves == 2) return GemmShape<2, 256, 1, 1, 2>::SMEM_BYTES;
    FI_SMEM(1, 64, 1) FI_SMEM(1, 128, 1) FI_SMEM(1, 256, 1)
    FI_SMEM(2, 64, 1) FI_SMEM(2, 128, 1) FI_SMEM(2, 256, 1)
    FI_SMEM(1, 64, 2) FI_SMEM(1, 128, 2) FI_SMEM(1, 128, 4) FI_SMEM(1, 256, 2) FI_SMEM(1, 256, 4) FI_SMEM(2, 256, 2) FI_SMEM(2, 256, 4) FI_SMEM(2, 128, 2) FI_SMEM(2, 128, 4)
#undef FI_SMEM
    return 0;
}

int tc_gemm_tmem_cols(const TcGemmConfig& c) {
#define FI_TMEM(CG, BN, SK) \
    if (c.cta_group == CG && c.bn == BN && c.split_k == SK && c.slabs == 1 && c.n_halves == 1) return GemmShape<CG, BN, SK>::TMEM_COLS;
    if (c.cta_group == 2 && c.bn == 256 && c.split_k == 1 && c.slabs == 2) return GemmShape<2, 256, 1, 2>::TMEM_COLS;
    if (c.cta_group == 2 && c.bn == 256 && c.split_k == 1 && c.n_halves == 2) return GemmShape<2, 256, 1, 1, 2>::TMEM_COLS;
    FI_TMEM(1, 64, 1) FI_TMEM(1, 128, 1) FI_TMEM(1, 256, 1)
    FI_TMEM(2, 64, 1) FI_TMEM(2, 128, 1) FI_TMEM(2, 256, 1)
    FI_TMEM(1, 64, 2) FI_TMEM(1, 128, 2) FI_TMEM(1, 128, 4) FI_TMEM(1, 256, 2) FI_TMEM(1, 256, 4) FI_TMEM(2, 256, 2) FI_TMEM(2, 256, 4) FI_TMEM(2, 128, 2) FI_TMEM(2, 128, 4)
#undef FI_TMEM
    return 0;
}

int tc_gemm_check(const TcGemmConfig& c, int M, int N, int K) {
    if (!tc_gemm_stages(c)) return kTcErrUnsupported;
    const bool wide_ok = c.cta_group == 2 && c.bn == 256 && c.split_k == 1 && c.slabs * c.n_halves == 2;
    if (c.slabs * c.n_halves != 1 && !wide_ok) return kTcErrUnsupported;
    if (c.mcast != 1 && !(c.mcast == 2 && c.cta_group == 2 && c.split_k == 1 && c.slabs * c.n_halves == 1))
        return kTcErrUnsupported;
    const int bm = 128 * c.cta_group * c.slabs;
    if (M <= 0 || N <= 0 || K <= 0) return kTcErrShape;
    if (M % bm || N % (c.bn * c.n_halves * c.mcast) || K % (64 * c.split_k)) return kTcErrShape;
    if (c.b_mn_major && (c.bn / c.cta_group) % 64) return kTcErrShape;
    if (c.split_k > 1 && (c.bn / c.split_k) % 32) return kTcErrShape;
    return kTcOk;
}

TcLaunchInfo tc_gemm_plan(const TcGemmConfig& cfg, const TcGemmProblem& p) {
    g_last = TcLaunchInfo{};
    tc_gemm_launch(cfg, p, nullptr, true);
    return g_last;
}

int tc_gemm_launch(const TcGemmConfig& cfg, const TcGemmProblem& p, cudaStream_t stream, bool dry_run) {
    int chk = tc_gemm_check(cfg, p.M, p.N, p.K);
    if (chk != kTcOk) return chk;
    // without a caller-owned workspace, the pool's per-(device, stream) entry is
    // grown and its epoch advanced under the pool lock
    std::unique_lock<std::mutex> pool_lock(pool_mutex(), std::defer_lock);
    if (!p.workspace && !dry_run) pool_lock.lock();
    // FI_TC_KB=2: two-K-block stages (half the TMA operations) for the pair 256 x 256 tile
    static const int kb_env = [] {
        const char* v = std::getenv("FI_TC_KB");
        return v ? std::atoi(v) : 1;
    }();
    if (kb_env == 2 && cfg.cta_group == 2 && cfg.bn == 256 && cfg.split_k == 1 && cfg.slabs == 1 &&
        cfg.n_halves == 1 && cfg.mcast == 1)
        return launch_impl<2, 256, 1, 1, 1, 1, 2>(cfg, p, stream, dry_run);
    if (cfg.slabs == 2) return launch_impl<2, 256, 1, 2>(cfg, p, stream, dry_run);
    if (cfg.n_halves == 2) return launch_impl<2, 256, 1, 1, 2>(cfg, p, stream, dry_run);
    if (cfg.mcast == 2) {
        if (cfg.bn == 64) return launch_impl<2, 64, 1, 1, 1, 2>(cfg, p, stream, dry_run);
        if (cfg.bn == 128) return launch_impl<2, 128, 1, 1, 1, 2>(cfg, p, stream, dry_run);
        if (cfg.bn == 256) return launch_impl<2, 256, 1, 1, 1, 2>(cfg, p, stream, dry_run);
        return kTcErrUnsupported;
    }
#define FI_LAUNCH(CG, BN, SK) \
    if (cfg.cta_group == CG && cfg.bn == BN && cfg.split_k == SK) return launch_impl<CG, BN, SK>(cfg, p, stream, dry_run);
    FI_LAUNCH(1, 64, 1) FI_LAUNCH(1, 128, 1) FI_LAUNCH(1, 256, 1)
    FI_LAUNCH(2, 64, 1) FI_LAUNCH(2, 128, 1) FI_LAUNCH(2, 256, 1)
    FI_LAUNCH(1, 64, 2) FI_LAUNCH(1, 128, 2) FI_LAUNCH(1, 128, 4) FI_LAUNCH(1, 256, 2) FI_LAUNCH(1, 256, 4) FI_LAUNCH(2, 256, 2) FI_LAUNCH(2, 256, 4) FI_LAUNCH(2, 128, 2) FI_LAUNCH(2, 128, 4)
#undef FI_LAUNCH
    return kTcErrUnsupported;
}

}  // namespace fireiron::sm100
