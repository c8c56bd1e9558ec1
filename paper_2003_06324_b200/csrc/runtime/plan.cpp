// Runtime: compiles, caches and launches lowered strategies on the B200.
//   generic plans  -> emitted CUDA -> NVRTC (sm_100a, --fmad=false) -> cubin
//                     (memory + on-disk cache keyed by source/options) -> cuModule
//   tcgen05 plans  -> the AOT tensor-core kernel family (sm100/gemm.cu)
// NVRTC and the driver API are resolved at run time (dlopen / driver entry
// points) so the library loads on hosts without a GPU.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>

#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <fstream>
#include <functional>
#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>

#include "../sm100/tc_gemm.hpp"
#include "host_snap.hpp"
#include "fireiron/backend.hpp"

namespace fireiron {

long generic_shared_bytes(const Program& prog);
namespace rt {
cudaError_t convert_f32(const float* src, void* dst, int64_t n, int elem, cudaStream_t s);
cudaError_t widen_to_f32(const void* src, float* dst, int64_t n, int elem, cudaStream_t s);
cudaError_t convert_f32_2d(const float* src, void* dst, int64_t width, int64_t height, int64_t pitch, int elem,
                           cudaStream_t s);
cudaError_t widen_to_f32_2d(const void* src, float* dst, int64_t width, int64_t height, int64_t pitch, int elem,
                            cudaStream_t s);
int device_sm_count();
}  // namespace rt

namespace {

[[noreturn]] void cuda_fail(const std::string& what, cudaError_t e) {
    throw BackendError(100, what + ": " + cudaGetErrorString(e));
}
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) cuda_fail(what, e);
}

// status of sm100::tc_gemm_launch -> BackendError (every tcgen05 launch site)
void check_tc_launch(int r) {
    if (r == sm100::kTcOk) return;
    if (r == sm100::kTcErrCapture)
        throw BackendError(104, "the plan's stream-K workspace is not allocated yet: launch it once outside "
                                "the CUDA-graph capture");
    if (r == sm100::kTcErrCuda)
        throw BackendError(100, std::string("tcgen05 GEMM launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    throw BackendError(100, "tcgen05 GEMM launch failed (code " + std::to_string(r) + ")");
}

// ---------------------------------------------------------------- NVRTC
struct Nvrtc {
    using Prog = void*;
    int (*create)(Prog*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    int (*compile)(Prog, int, const char* const*) = nullptr;
    int (*log_size)(Prog, size_t*) = nullptr;
    int (*log)(Prog, char*) = nullptr;
    int (*cubin_size)(Prog, size_t*) = nullptr;
    int (*cubin)(Prog, char*) = nullptr;
    int (*destroy)(Prog*) = nullptr;
    int (*version)(int*, int*) = nullptr;
    bool ok = false;
    std::string error;

    static const Nvrtc& get() {
        static Nvrtc n = [] {
            Nvrtc x;
            void* h = nullptr;
            for (const char* p : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"})
                if ((h = dlopen(p, RTLD_NOW | RTLD_GLOBAL))) break;
            if (!h) {
                x.error = "libnvrtc.so.12 not found";
                return x;
            }
            auto sym = [&](const char* s) { return dlsym(h, s); };
            x.create = reinterpret_cast<decltype(x.create)>(sym("nvrtcCreateProgram"));
            x.compile = reinterpret_cast<decltype(x.compile)>(sym("nvrtcCompileProgram"));
            x.log_size = reinterpret_cast<decltype(x.log_size)>(sym("nvrtcGetProgramLogSize"));
            x.log = reinterpret_cast<decltype(x.log)>(sym("nvrtcGetProgramLog"));
            x.cubin_size = reinterpret_cast<decltype(x.cubin_size)>(sym("nvrtcGetCUBINSize"));
            x.cubin = reinterpret_cast<decltype(x.cubin)>(sym("nvrtcGetCUBIN"));
            x.destroy = reinterpret_cast<decltype(x.destroy)>(sym("nvrtcDestroyProgram"));
            x.version = reinterpret_cast<decltype(x.version)>(sym("nvrtcVersion"));
            x.ok = x.create && x.compile && x.log_size && x.log && x.cubin_size && x.cubin && x.destroy;
            if (!x.ok) x.error = "libnvrtc is missing required symbols";
            return x;
        }();
        return n;
    }
};

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

std::string cache_dir() {
    if (const char* e = std::getenv("FI_KERNEL_CACHE")) return e;
    const char* home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/fireiron_b200";
}

void mkdirs(const std::string& path) {
    std::string cur;
    for (size_t i = 0; i < path.size(); ++i) {
        cur += path[i];
        if (path[i] == '/' && cur.size() > 1) mkdir(cur.c_str(), 0755);
    }
    mkdir(path.c_str(), 0755);
}

// source -> cubin (sm_100a), memoised in process and on disk
std::string compile_cubin(const std::string& source, const std::string& name) {
    static std::mutex mu;
    static std::map<uint64_t, std::string> memo;
    const std::vector<std::string> opts = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17",
                                           "-default-device", "-lineinfo",
                                           "--include-path=/usr/local/cuda/include"};
    std::string key_text = source;
    for (const auto& o : opts) key_text += "\n" + o;
    const uint64_t key = fnv1a(key_text);
    {
        std::lock_guard<std::mutex> g(mu);
        if (auto it = memo.find(key); it != memo.end()) return it->second;
    }
    char hex[32];
    std::snprintf(hex, sizeof(hex), "%016llx", static_cast<unsigned long long>(key));
    const std::string path = cache_dir() + "/" + hex + ".cubin";
    {
        std::ifstream in(path, std::ios::binary);
        if (in) {
            std::ostringstream ss;
            ss << in.rdbuf();
            std::string bin = ss.str();
            if (!bin.empty()) {
                std::lock_guard<std::mutex> g(mu);
                memo[key] = bin;
                return bin;
            }
        }
    }
    const Nvrtc& nv = Nvrtc::get();
    if (!nv.ok) throw BackendError(101, "NVRTC unavailable: " + nv.error);
    Nvrtc::Prog p = nullptr;
    if (nv.create(&p, source.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) != 0)
        throw BackendError(101, "nvrtcCreateProgram failed");
    std::vector<const char*> argv;
    for (const auto& o : opts) argv.push_back(o.c_str());
    const int rc = nv.compile(p, static_cast<int>(argv.size()), argv.data());
    if (rc != 0) {
        size_t n = 0;
        nv.log_size(p, &n);
        std::string log(n, '\0');
        nv.log(p, log.data());
        nv.destroy(&p);
        throw BackendError(101, "NVRTC compilation of " + name + " failed:\n" + log);
    }
    size_t n = 0;
    nv.cubin_size(p, &n);
    std::string bin(n, '\0');
    nv.cubin(p, bin.data());
    nv.destroy(&p);
    mkdirs(cache_dir());
    {
        const std::string tmp = path + ".tmp" + std::to_string(getpid());
        std::ofstream out(tmp, std::ios::binary);
        out.write(bin.data(), static_cast<std::streamsize>(bin.size()));
        out.close();
        std::rename(tmp.c_str(), path.c_str());
    }
    std::lock_guard<std::mutex> g(mu);
    memo[key] = bin;
    return bin;
}

// ---------------------------------------------------------------- driver API
struct Driver {
    CUresult (*module_load_data)(CUmodule*, const void*) = nullptr;
    CUresult (*module_get_function)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*module_unload)(CUmodule) = nullptr;
    CUresult (*func_set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*launch_kernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                              CUstream, void**, void**) = nullptr;
    CUresult (*get_error_string)(CUresult, const char**) = nullptr;

    static const Driver& get() {
        static Driver d = [] {
            Driver x;
            auto sym = [](const char* s) -> void* {
                void* p = nullptr;
                cudaDriverEntryPointQueryResult q;
                if (cudaGetDriverEntryPoint(s, &p, cudaEnableDefault, &q) != cudaSuccess ||
                    q != cudaDriverEntryPointSuccess)
                    return nullptr;
                return p;
            };
            x.module_load_data = reinterpret_cast<decltype(x.module_load_data)>(sym("cuModuleLoadData"));
            x.module_get_function = reinterpret_cast<decltype(x.module_get_function)>(sym("cuModuleGetFunction"));
            x.module_unload = reinterpret_cast<decltype(x.module_unload)>(sym("cuModuleUnload"));
            x.func_set_attribute = reinterpret_cast<decltype(x.func_set_attribute)>(sym("cuFuncSetAttribute"));
            x.launch_kernel = reinterpret_cast<decltype(x.launch_kernel)>(sym("cuLaunchKernel"));
            x.get_error_string = reinterpret_cast<decltype(x.get_error_string)>(sym("cuGetErrorString"));
            return x;
        }();
        if (!d.module_load_data || !d.launch_kernel) throw BackendError(100, "CUDA driver entry points unavailable");
        return d;
    }
    void check(CUresult r, const char* what) const {
        if (r == CUDA_SUCCESS) return;
        const char* s = "unknown";
        if (get_error_string) get_error_string(r, &s);
        throw BackendError(100, std::string(what) + ": " + s);
    }
};

int elem_code(ElemType e) { return e == ElemType::F32 ? 0 : e == ElemType::F16 ? 1 : 2; }

bool reads_buffer(const StmtList& body, int id) {
    for (const auto& s : body) {
        if (const auto* l = std::get_if<LoopStmt>(&s.v)) {
            if (reads_buffer(l->body, id)) return true;
        } else if (const auto* f = std::get_if<FmaStmt>(&s.v)) {
            if (f->c.buf == id || f->a.buf == id || f->b.buf == id) return true;
        } else if (const auto* c = std::get_if<CopyStmt>(&s.v)) {
            if (c->src.buf == id) return true;
        } else if (const auto* w = std::get_if<WmmaLoadStmt>(&s.v)) {
            if (w->src.buf == id) return true;
        } else if (const auto* m = std::get_if<MicroKernelStmt>(&s.v)) {
            for (const auto& o : m->operands)
                if (o.second.buf == id) return true;
        }
    }
    return false;
}

}  // namespace

// ---------------------------------------------------------------- Plan
struct Plan::Impl {
    Program prog;
    MicroKernelSet mks;  // owned copy (the Program's micro-kernel pointers index it)
    PlanInfo info;
    std::string source;
    int device = 0;
    // generic
    CUmodule module = nullptr;
    CUfunction func = nullptr;
    long smem = 0;
    bool zero_c = false;
    // tcgen05
    sm100::TcGemmConfig tc;
    sm100::TcGemmProblem tp;
    int32_t* d_tile_order = nullptr;
    mutable sm100::TcWorkspace ws;  // stream-K partials + epoch flags of this plan
    // run_host scratch
    mutable std::mutex mu;
    mutable void* scratch = nullptr;
    mutable size_t scratch_bytes = 0;
    mutable cudaStream_t own_stream = nullptr;
    mutable cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // pipelined run_host: copy-engine streams (H2D, D2H) and per-chunk events
    mutable cudaStream_t up_stream = nullptr, down_stream = nullptr;
    mutable std::vector<cudaEvent_t> pev;
    // pinned host staging of host-snapped inputs (typed layout of each root)
    mutable void* host_stage = nullptr;
    mutable size_t host_stage_bytes = 0;
    mutable void* host_cstage = nullptr;  // pinned staging of a pageable C
    mutable size_t host_cstage_bytes = 0;
    mutable std::vector<cudaEvent_t> hev;  // host pipeline: C region landed (staged C)
    // bytes the last run_host moved across PCIe (host -> device, device -> host)
    mutable long last_up = 0, last_down = 0;

    ~Impl() {
        if (module) {
            try {
                Driver::get().module_unload(module);
            } catch (...) {
            }
        }
        if (d_tile_order) cudaFree(d_tile_order);
        if (scratch) cudaFree(scratch);
        if (own_stream) cudaStreamDestroy(own_stream);
        if (up_stream) cudaStreamDestroy(up_stream);
        if (down_stream) cudaStreamDestroy(down_stream);
        for (cudaEvent_t e : pev) cudaEventDestroy(e);
        if (host_stage) cudaFreeHost(host_stage);
        if (host_cstage) cudaFreeHost(host_cstage);
        for (cudaEvent_t e : hev) cudaEventDestroy(e);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }

    const BufferDecl& root(int i) const { return prog.plan.at(i); }
    int out_root() const { return prog.root.is_matmul() ? 2 : 1; }
};

namespace {

// ---------------------------------------------------------------- pipelined run_host
// The host boundary moves fp32 matrices over PCIe (anvil::Matrix is fp32):
// 4(MK + KN) bytes up and 4MN down, ~25x the GEMM's own time at 4096^3. For
// tcgen05 plans with column-major B and C (Fireiron's default layouts) the
// output is computed in column panels so the three engines overlap:
//   up stream   : H2D A in pieces, then H2D B panel by panel
//   main stream : snap A pieces to f16/bf16 as they land; per panel j: snap
//                 B_j, GEMM on the (M x N/P x K) panel (pointer offsets into
//                 the same TMA-described buffers), [widen C_j]
//   down stream : D2H C_j while B_{j+1} is still coming up (PCIe is duplex)
// Returns the number of panels P, or 0 when the plain path applies.
int pipeline_chunks(const Plan::Impl& I) {
    if (I.info.kind != 1 || !I.prog.root.is_matmul() || I.tp.tile_order) return 0;
    if (I.tc.b_mn_major || I.tc.c_row_major) return 0;  // panels must be contiguous column ranges
    if (const char* e = std::getenv("FI_HOST_PIPELINE"); e && (e[0] == '0' || e[0] == 'b')) return 0;
    const long tiles_n = I.tp.N / (I.tc.bn * I.tc.n_halves * I.tc.mcast);  // whole scheduled tiles per panel
    const double b_bytes = 4.0 * I.tp.K * I.tp.N;
    int best = 0, cap = 8;
    if (const char* v = std::getenv("FI_HOST_PANELS")) cap = std::atoi(v);
    for (int p = 2; p <= cap; ++p)  // panels of >= 4 MiB each, whole block tiles
        if (tiles_n % p == 0 && b_bytes / p >= 4.0 * (1 << 20)) best = p;
    return best;
}

// ---------------------------------------------------------------- blocked run_host
// The column-panel pipeline above still uploads all of A before the first GEMM.
// The blocked pipeline cuts A into P row panels and B into Q column panels and
// uploads them alternately (balanced by bytes); as each panel lands, ONE GEMM
// computes the C blocks it completes -- row panel i against the B panels already
// up, or the A panels already up against column panel j -- and that C region
// goes down while later panels come up. The first GEMM waits for one panel of
// each operand, so PCIe runs both directions for most of the call. Panels and
// C regions are pitched 2D copies, so any root layout qualifies.
struct Region {
    long off, width, height, pitch;  // elements: `height` lines of `width`, `pitch` apart
};

bool blocked_split(const Plan::Impl& I, int& P, int& Q) {
    if (I.info.kind != 1 || !I.prog.root.is_matmul() || I.tp.tile_order) return false;
    const char* e = std::getenv("FI_HOST_PIPELINE");
    if (e && (e[0] == '0' || e[0] == 'p')) return false;  // off, or the column-panel pipeline
    const long tm = 128L * I.tc.cta_group * I.tc.slabs;
    const long tn = static_cast<long>(I.tc.bn) * I.tc.n_halves * I.tc.mcast;
    double piece = 16.0 * (1 << 20);  // target panel size: 16 MiB of fp32 (measured: profiles/round1/e2e_host_pipeline.txt)
    if (const char* v = std::getenv("FI_HOST_PANEL_MB")) piece = std::atof(v) * (1 << 20);
    // a panel cut across the contiguous dimension is a pitched copy whose lines
    // must stay >= 4 KiB: shorter lines cost PCIe duplex bandwidth (2 KiB lines:
    // 62 GB/s both ways vs 99 linear, profiles/round1/e2e_host_pipeline.txt)
    const bool a_strided = I.tc.a_mn_major || I.tc.c_row_major == 0;  // A or C lines of M/P elements
    const bool b_strided = I.tc.b_mn_major || I.tc.c_row_major != 0;  // B or C lines of N/Q elements
    long min_line = 1024;
    if (const char* v = std::getenv("FI_HOST_MIN_LINE")) min_line = std::atol(v);
    auto pick = [&](long dim, long tile, double bytes, bool strided) {
        int best = 1;
        for (int p = 2; p <= 64; ++p)
            if (dim % (p * tile) == 0 && bytes / p >= piece && (!strided || dim / p >= min_line)) best = p;
        return best;
    };
    // measured crossover: 4096^3 (128 MiB up) blocked 3.08 ms vs column panels
    // 3.5-3.7; 1024^2 x 32768 (256 MiB) equal; 16384^3 (2 GiB) blocked 47.4 ms vs
    // 45.7 (there the pitched A copies cost more than the early C download gains)
    double up_limit = 512.0 * (1 << 20);
    if (const char* v = std::getenv("FI_HOST_BLOCKED_MAX_MB")) up_limit = std::atof(v) * (1 << 20);
    if (4.0 * I.tp.K * (static_cast<double>(I.tp.M) + I.tp.N) > up_limit) return false;
    P = pick(I.tp.M, tm, 4.0 * I.tp.M * I.tp.K, a_strided);
    Q = pick(I.tp.N, tn, 4.0 * I.tp.K * I.tp.N, b_strided);
    return P * Q >= 4;
}

// ---------------------------------------------------------------- host side of both pipelines
// Uploads: each input region is cut into pieces of whole lines (~FI_HOST_PIECE_MB
// of fp32, default 8). Host snapping (runtime/host_snap.hpp): a fraction
// FI_HOST_SNAP_RATIO (default 1: all but the first) of the pieces of f16/bf16 roots, spread
// evenly over the upload order, is converted by host cores into pinned staging
// while the copy engine moves the others as fp32 (snapped on the device), and
// then crosses PCIe in 2-byte elements. The ratio balances the two engines
// measured on the B200 box: the copy engine moves ~54 GB/s; with the AVX-512
// conversion (112 GB/s alone on 16 threads) the host keeps ahead of the copy
// engine even while it also reads host memory, so every piece but the first is
// host-snapped (0.8 was best with the slower AVX2 conversion;
// profiles/round2/host_snap_probe.txt, host_snap_e2e_ab.log, host_snap_avx512.log). The first
// FI_HOST_SNAP_SKIP pieces (default 1) are snapped on the device so the copy
// engine starts at once. Pageable inputs (anvil::Matrix is a std::vector) are
// snapped on the host entirely: the driver's staged pageable copies are slower
// than the host conversion. A piece is either converted on the host or uploaded
// as fp32, never both: once many host threads have read a pinned buffer the copy
// engine reads it at ~60 % speed (profiles/round2/dma_after_cpu_read.txt).
// Downloads: C regions go down on the down stream; a pageable C is staged in
// pinned memory and copied out by the host pool as each region lands.
struct HostIO {
    struct Piece {
        int which;  // 0 A, 1 B
        int tag;    // caller's label (panel index) for the trace
        Region r;
        std::unique_ptr<rt::SnapJob> job;
    };
    struct Down {
        Region r;
        cudaEvent_t ev;
        std::unique_ptr<rt::SnapJob> job;
    };

    const Plan::Impl& I;
    cudaStream_t s;
    char* base;
    const size_t* f32_in;
    const size_t* typed_in;
    const float* in[2];
    float* C;
    int elem[2];
    size_t w[2];
    rt::HostSnapPool* pool = nullptr;
    bool pinned[2] = {true, true};
    float* c_stage = nullptr;  // pinned staging of a pageable C
    std::vector<Piece> pieces;
    std::vector<Down> downs;
    size_t nev = 0;
    const bool tracing = std::getenv("FI_HOST_PIPELINE_TRACE") != nullptr;
    std::vector<std::pair<long, cudaEvent_t>> down_done;  // traced: bytes and completion of each C region

    static bool is_pinned(const void* p) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (a.type == cudaMemoryTypeDevice)  // the host pipelines read and write host memory
            throw BackendError(104, "run_host expects host buffers (got a device pointer; use fi_plan_launch)");
        return a.type == cudaMemoryTypeHost;
    }

    HostIO(const Plan::Impl& I_, cudaStream_t s_, char* base_, const size_t* f32_in_, const size_t* typed_in_,
           const float* A, const float* B, float* C_)
        : I(I_), s(s_), base(base_), f32_in(f32_in_), typed_in(typed_in_), in{A, B}, C(C_) {
        for (int i = 0; i < 2; ++i) {
            elem[i] = elem_code(I.root(i).elem);
            w[i] = byte_width(I.root(i).elem);
        }
        if (elem[0] != 0 || elem[1] != 0 || !is_pinned(C)) pool = rt::HostSnapPool::get();
        if (pool) {
            pinned[0] = is_pinned(A);
            pinned[1] = is_pinned(B);
            if (!is_pinned(C)) {
                const size_t cbytes = static_cast<size_t>(I.root(I.out_root()).extent()) * 4;
                if (I.host_cstage_bytes < cbytes) {
                    if (I.host_cstage) cudaFreeHost(I.host_cstage);
                    I.host_cstage = nullptr;
                    I.host_cstage_bytes = 0;
                    ck(cudaHostAlloc(&I.host_cstage, cbytes, cudaHostAllocPortable), "cudaHostAlloc");
                    I.host_cstage_bytes = cbytes;
                }
                c_stage = static_cast<float*>(I.host_cstage);
            }
        }
    }
    // every submitted job is waited for, also when an enqueue throws: the pool's
    // workers must not touch a job (or the caller's buffers) after we return
    ~HostIO() {
        // an enqueue failed mid-call: copies already queued may still read the
        // pinned staging (or write C) -- drain them before the staging is reused
        if (std::uncaught_exceptions() > 0) {
            if (I.up_stream) cudaStreamSynchronize(I.up_stream);
            if (I.down_stream) cudaStreamSynchronize(I.down_stream);
            cudaGetLastError();
        }
        for (auto& d : down_done) cudaEventDestroy(d.second);
        if (!pool) return;
        for (auto& p : pieces)
            if (p.job) pool->wait(p.job.get());
        for (auto& d : downs)
            if (d.job) pool->wait(d.job.get());
    }

    cudaEvent_t event() {
        if (nev == I.hev.size()) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            I.hev.push_back(e);
        }
        return I.hev[nev++];
    }

    // cut region r of input `which` into pieces of whole lines; returns one past the last
    int add(int which, const Region& r, int tag) {
        double piece_bytes = 8.0 * (1 << 20);
        if (const char* v = std::getenv("FI_HOST_PIECE_MB")) piece_bytes = std::atof(v) * (1 << 20);
        long nsub = std::max(1L, std::lround(4.0 * r.width * r.height / piece_bytes));
        if (r.width == r.pitch && r.height < nsub) {
            // contiguous storage with few lines (a whole operand): cut element
            // ranges on 1024-element boundaries
            const long n = r.width * r.height;
            for (long q = 0; q < nsub; ++q) {
                const long e0 = (n * q / nsub) & ~1023L, e1 = q + 1 == nsub ? n : (n * (q + 1) / nsub) & ~1023L;
                if (e1 > e0) pieces.push_back(Piece{which, tag, Region{r.off + e0, e1 - e0, 1, e1 - e0}, nullptr});
            }
            return static_cast<int>(pieces.size());
        }
        nsub = std::min(nsub, r.height);
        for (long q = 0; q < nsub; ++q) {
            const long l0 = r.height * q / nsub, l1 = r.height * (q + 1) / nsub;
            pieces.push_back(Piece{which, tag, Region{r.off + l0 * r.pitch, r.width, l1 - l0, r.pitch}, nullptr});
        }
        return static_cast<int>(pieces.size());
    }

    // decide host / device snapping per piece and start the host conversions.
    // Host-snapped pieces are staged densely packed, so their upload reads host
    // memory sequentially even when the piece is a pitched panel of the root
    // (short lines cost PCIe bandwidth, profiles/round1/e2e_host_pipeline.txt).
    void start() {
        if (!pool || (elem[0] == 0 && elem[1] == 0)) return;
        // leading pieces snapped on the device: 1 for pinned inputs (the copy engine
        // starts at once), none for pageable ones (their staged copies are slow)
        int skip = -1;
        if (const char* v = std::getenv("FI_HOST_SNAP_SKIP")) skip = std::atoi(v);
        double ratio = 1.0;
        if (const char* v = std::getenv("FI_HOST_SNAP_RATIO")) ratio = std::atof(v);
        ratio = std::min(ratio, ratio * (pool->workers() + 1) / 16.0);  // fewer host threads convert less
        const int npc = static_cast<int>(pieces.size());
        std::vector<size_t> off(static_cast<size_t>(npc), 0);
        size_t hbytes = 0;
        std::vector<char> host(static_cast<size_t>(npc), 0);
        for (int j = 0, h = 0; j < npc; ++j) {
            const Piece& pc = pieces[static_cast<size_t>(j)];
            if (elem[pc.which] == 0) continue;
            const int sk = skip >= 0 ? skip : pinned[pc.which] ? 1 : 0;
            if (j < sk) continue;
            bool on_host = !pinned[pc.which];  // pageable input: every piece
            if (!on_host) {
                // piece j - sk goes to the host when the running share crosses an integer
                const int want = static_cast<int>(std::floor((j - sk + 1) * ratio + 1e-9));
                on_host = want > h;
                h = std::max(h, want);
            }
            if (!on_host) continue;
            host[static_cast<size_t>(j)] = 1;
            off[static_cast<size_t>(j)] = hbytes;
            hbytes += (static_cast<size_t>(pc.r.width * pc.r.height) * 2 + 255) & ~size_t(255);
        }
        if (hbytes == 0) return;
        if (I.host_stage_bytes < hbytes) {
            if (I.host_stage) cudaFreeHost(I.host_stage);
            I.host_stage = nullptr;
            I.host_stage_bytes = 0;
            ck(cudaHostAlloc(&I.host_stage, hbytes, cudaHostAllocPortable), "cudaHostAlloc");
            I.host_stage_bytes = hbytes;
        }
        for (int j = 0; j < npc; ++j) {
            if (!host[static_cast<size_t>(j)]) continue;
            Piece& pc = pieces[static_cast<size_t>(j)];
            auto job = std::make_unique<rt::SnapJob>();
            job->src = in[pc.which] + pc.r.off;
            job->dst = static_cast<char*>(I.host_stage) + off[static_cast<size_t>(j)];
            job->width = pc.r.width;
            job->height = pc.r.height;
            job->spitch = pc.r.pitch;
            job->dpitch = pc.r.width;  // packed
            job->elem = elem[pc.which];
            if (pc.r.width == pc.r.pitch) {  // contiguous: one long line
                job->width = pc.r.width * pc.r.height;
                job->height = 1;
            }
            pc.job = std::move(job);
        }
        for (auto& pc : pieces)  // FIFO: converted in upload order
            if (pc.job) pool->submit(pc.job.get());
    }

    static void copy2d(void* dst, const void* src, const Region& r, cudaMemcpyKind kind, cudaStream_t st, size_t w) {
        if (r.width == r.pitch)  // contiguous lines: one linear copy
            ck(cudaMemcpyAsync(dst, src, static_cast<size_t>(r.width * r.height) * w, kind, st), "cudaMemcpyAsync");
        else
            ck(cudaMemcpy2DAsync(dst, r.pitch * w, src, r.pitch * w, r.width * w, r.height, kind, st),
               "cudaMemcpy2DAsync");
    }

    // one piece: H2D into the fp32 staging (or straight into an fp32 root), then
    // snapped to the root's element grid on s (sim.hpp:507-510); or, when host
    // snapped, H2D of the snapped piece straight into the typed root. `done` is
    // recorded on the up stream and s waits for it.
    void upload(int j, cudaEvent_t done) {
        const Piece& pc = pieces[static_cast<size_t>(j)];
        const int which = pc.which, e = elem[which];
        const Region& r = pc.r;
        char* typed = base + typed_in[which];
        if (pc.job) {
            pool->wait(pc.job.get());
            if (r.width == r.pitch)
                ck(cudaMemcpyAsync(typed + static_cast<size_t>(r.off) * w[which], pc.job->dst,
                                   static_cast<size_t>(r.width * r.height) * w[which], cudaMemcpyHostToDevice, I.up_stream),
                   "cudaMemcpyAsync");
            else  // packed staging -> pitched root
                ck(cudaMemcpy2DAsync(typed + static_cast<size_t>(r.off) * w[which], r.pitch * w[which], pc.job->dst,
                                     r.width * w[which], r.width * w[which], r.height, cudaMemcpyHostToDevice, I.up_stream),
                   "cudaMemcpy2DAsync");
            I.last_up += r.width * r.height * static_cast<long>(w[which]);
        } else {
            float* stage = e == 0 ? reinterpret_cast<float*>(typed) : reinterpret_cast<float*>(base + f32_in[which]);
            copy2d(stage + r.off, in[which] + r.off, r, cudaMemcpyHostToDevice, I.up_stream, 4);
            I.last_up += r.width * r.height * 4;
        }
        ck(cudaEventRecord(done, I.up_stream), "cudaEventRecord");
        ck(cudaStreamWaitEvent(s, done, 0), "cudaStreamWaitEvent");
        if (!pc.job && e != 0) {
            float* stage = reinterpret_cast<float*>(base + f32_in[which]);
            ck(rt::convert_f32_2d(stage + r.off, typed + static_cast<size_t>(r.off) * w[which], r.width, r.height,
                                  r.pitch, e, s),
               "input conversion");
        }
    }

    // D2H of C region cr from the fp32 device result (after `ready` on s)
    void download(const float* result, const Region& cr, cudaEvent_t ready) {
        ck(cudaStreamWaitEvent(I.down_stream, ready, 0), "cudaStreamWaitEvent");
        copy2d((c_stage ? c_stage : C) + cr.off, result + cr.off, cr, cudaMemcpyDeviceToHost, I.down_stream, 4);
        I.last_down += cr.width * cr.height * 4;
        if (tracing) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            ck(cudaEventRecord(e, I.down_stream), "cudaEventRecord");
            down_done.emplace_back(cr.width * cr.height * 4, e);
        }
        if (c_stage) {
            downs.push_back(Down{cr, event(), nullptr});
            ck(cudaEventRecord(downs.back().ev, I.down_stream), "cudaEventRecord");
        }
    }

    // staged C: copy each region out as it lands (host pool; the caller helps)
    void finish() {
        if (!c_stage) return;
        for (auto& d : downs) {
            ck(cudaEventSynchronize(d.ev), "cudaEventSynchronize");
            auto job = std::make_unique<rt::SnapJob>();
            job->src = c_stage + d.r.off;
            job->dst = C + d.r.off;
            job->width = d.r.width;
            job->height = d.r.height;
            job->spitch = job->dpitch = d.r.pitch;
            job->elem = 0;
            if (d.r.width == d.r.pitch) {
                job->width = d.r.width * d.r.height;
                job->height = 1;
            }
            d.job = std::move(job);
            pool->submit(d.job.get());
        }
        for (auto& d : downs) pool->wait(d.job.get());
    }

    void trace_pieces(const std::function<float(cudaEvent_t)>& at, const cudaEvent_t* ev_up) const {
        std::fprintf(stderr, "%d pieces (%d host workers%s%s): up", static_cast<int>(pieces.size()),
                     pool ? pool->workers() : -1, pinned[0] && pinned[1] ? "" : ", pageable input",
                     c_stage ? ", pageable C" : "");
        for (size_t j = 0; j < pieces.size(); ++j) {
            const Piece& pc = pieces[j];
            std::fprintf(stderr, " %c%d%s%.3f", pc.which ? 'B' : 'A', pc.tag, pc.job ? "h" : "", at(ev_up[j]));
        }
        std::fprintf(stderr, " | down");
        for (const auto& d : down_done) std::fprintf(stderr, " %.1fM@%.3f", d.first / 1048576.0, at(d.second));
    }
};

double run_host_blocked(const Plan::Impl& I, const float* A, const float* B, float* C, cudaStream_t s, int P,
                        int Q, char* base, const size_t* f32_in, const size_t* typed_in, size_t typed_c,
                        size_t f32_c) {
    const auto h_setup = std::chrono::steady_clock::now();
    if (!I.up_stream) {
        ck(cudaStreamCreateWithFlags(&I.up_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&I.down_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    const BufferDecl& rc = I.root(2);
    const int ec = elem_code(rc.elem);
    const size_t wa = byte_width(I.root(0).elem), wb = byte_width(I.root(1).elem), wc = byte_width(rc.elem);
    const long M = I.tp.M, N = I.tp.N, K = I.tp.K, lda = I.tp.lda, ldb = I.tp.ldb, ldc = I.tp.ldc;
    const bool a_row = !I.tc.a_mn_major, b_row = I.tc.b_mn_major != 0, c_row = I.tc.c_row_major != 0;
    const long mc = M / P, nc = N / Q;
    auto a_region = [&](long r0, long r1) { return a_row ? Region{r0 * lda, K, r1 - r0, lda} : Region{r0, r1 - r0, K, lda}; };
    auto b_region = [&](long c0, long c1) { return b_row ? Region{c0, c1 - c0, K, ldb} : Region{c0 * ldb, K, c1 - c0, ldb}; };
    auto c_region = [&](long r0, long r1, long c0, long c1) {
        return c_row ? Region{r0 * ldc + c0, c1 - c0, r1 - r0, ldc} : Region{r0 + c0 * ldc, r1 - r0, c1 - c0, ldc};
    };
    // the panel order: A row panels and B column panels alternately, balanced by bytes
    const double a_piece = 4.0 * mc * K, b_piece = 4.0 * K * nc;
    std::vector<char> order;
    for (int ia = 0, ib = 0; ia < P || ib < Q;) {
        const bool take_a = ib == Q || (ia < P && ia * a_piece <= ib * b_piece);
        order.push_back(take_a ? 'A' : 'B');
        (take_a ? ia : ib)++;
    }
    const int np = P + Q;
    HostIO io(I, s, base, f32_in, typed_in, A, B, C);
    std::vector<int> panel_end(static_cast<size_t>(np));  // one past each panel's last piece
    for (int i = 0, ia = 0, ib = 0; i < np; ++i) {
        const bool is_a = order[static_cast<size_t>(i)] == 'A';
        panel_end[static_cast<size_t>(i)] =
            io.add(is_a ? 0 : 1, is_a ? a_region(ia * mc, (ia + 1) * mc) : b_region(ib * nc, (ib + 1) * nc), i);
        (is_a ? ia : ib)++;
    }
    const int npc = static_cast<int>(io.pieces.size());
    // events: [start][upload per piece][gemm begin, end per panel][C ready per panel][down done]
    const size_t need = 1 + npc + 2 * np + np + 1;
    while (I.pev.size() < need) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        I.pev.push_back(e);
    }
    cudaEvent_t* ev = I.pev.data();
    cudaEvent_t ev_start = ev[0], *ev_up = ev + 1, *ev_g = ev_up + npc, *ev_c = ev_g + 2 * np, ev_down = ev_c[np];
    io.start();
    ck(cudaEventRecord(ev_start, s), "cudaEventRecord");  // scratch reuse: after earlier work on s
    ck(cudaStreamWaitEvent(I.up_stream, ev_start, 0), "cudaStreamWaitEvent");
    ck(cudaStreamWaitEvent(I.down_stream, ev_start, 0), "cudaStreamWaitEvent");
    const auto h_start = std::chrono::steady_clock::now();
    int ng = 0;
    auto gemm = [&](long r0, long r1, long c0, long c1) {
        sm100::TcGemmProblem p = I.tp;
        p.workspace = &I.ws;
        p.A = base + typed_in[0] + static_cast<size_t>(a_region(r0, r1).off) * wa;
        p.B = base + typed_in[1] + static_cast<size_t>(b_region(c0, c1).off) * wb;
        const Region cr = c_region(r0, r1, c0, c1);
        p.C = base + typed_c + static_cast<size_t>(cr.off) * wc;
        p.M = static_cast<int>(r1 - r0);
        p.N = static_cast<int>(c1 - c0);
        ck(cudaEventRecord(ev_g[2 * ng], s), "cudaEventRecord");
        const int r = sm100::tc_gemm_launch(I.tc, p, s);
        check_tc_launch(r);
        ck(cudaEventRecord(ev_g[2 * ng + 1], s), "cudaEventRecord");
        const float* result = reinterpret_cast<const float*>(base + typed_c);
        if (ec != 0) {
            ck(rt::widen_to_f32_2d(base + typed_c + static_cast<size_t>(cr.off) * wc,
                                   reinterpret_cast<float*>(base + f32_c) + cr.off, cr.width, cr.height, cr.pitch, ec, s),
               "output conversion");
            result = reinterpret_cast<const float*>(base + f32_c);
        }
        ck(cudaEventRecord(ev_c[ng], s), "cudaEventRecord");
        io.download(result, cr, ev_c[ng]);
        ++ng;
    };
    for (int i = 0, ia = 0, ib = 0, j = 0; i < np; ++i) {
        for (; j < panel_end[static_cast<size_t>(i)]; ++j) io.upload(j, ev_up[j]);
        if (order[static_cast<size_t>(i)] == 'A') {
            ++ia;
            if (ib > 0) gemm((ia - 1) * mc, ia * mc, 0, ib * nc);
        } else {
            ++ib;
            if (ia > 0) gemm(0, ia * mc, (ib - 1) * nc, ib * nc);
        }
    }
    const auto h_enqueued = std::chrono::steady_clock::now();
    ck(cudaEventRecord(ev_down, I.down_stream), "cudaEventRecord");
    ck(cudaStreamWaitEvent(s, ev_down, 0), "cudaStreamWaitEvent");
    io.finish();
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    const auto h_done = std::chrono::steady_clock::now();
    float ms_total = 0.f;
    for (int g = 0; g < ng; ++g) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_g[2 * g], ev_g[2 * g + 1]);
        ms_total += ms;
    }
    if (std::getenv("FI_HOST_PIPELINE_TRACE")) {  // event timeline relative to the start (ms)
        auto at = [&](cudaEvent_t e) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev_start, e);
            return ms;
        };
        auto us = [&](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
            return std::chrono::duration<double, std::micro>(b - a).count();
        };
        std::fprintf(stderr, "host: setup %.0f us, start->enqueued %.0f us, start->synced %.0f us | ",
                     us(h_setup, h_start), us(h_start, h_enqueued), us(h_start, h_done));
        std::fprintf(stderr, "blocked %dx%d panels, ", P, Q);
        io.trace_pieces(at, ev_up);
        std::fprintf(stderr, " | gemm");
        for (int g = 0; g < ng; ++g) std::fprintf(stderr, " %.3f-%.3f", at(ev_g[2 * g]), at(ev_g[2 * g + 1]));
        std::fprintf(stderr, " | C down done %.3f\n", at(ev_down));
    }
    return ms_total;
}

double run_host_pipelined(const Plan::Impl& I, const float* A, const float* B, float* C, cudaStream_t s,
                          int chunks, char* base, const size_t* f32_in, const size_t* typed_in, size_t typed_c,
                          size_t f32_c) {
    if (!I.up_stream) {
        ck(cudaStreamCreateWithFlags(&I.up_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&I.down_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    const BufferDecl& ra = I.root(0);
    const BufferDecl& rb = I.root(1);
    const BufferDecl& rc = I.root(2);
    const int ec = elem_code(rc.elem);
    const size_t wb = byte_width(rb.elem), wc = byte_width(rc.elem);
    HostIO io(I, s, base, f32_in, typed_in, A, B, C);
    // A as one contiguous region (its storage), then B panel by panel
    const long a_ext = ra.extent();
    const int a_end = io.add(0, Region{0, a_ext, 1, a_ext}, 0);
    const long nc = I.tp.N / chunks;  // columns per panel
    const long b_ext = rb.extent(), c_ext = rc.extent();
    std::vector<int> panel_end(static_cast<size_t>(chunks));
    for (int j = 0; j < chunks; ++j) {
        const long b0 = j * nc * I.tp.ldb, b1 = j + 1 == chunks ? b_ext : (j + 1) * nc * I.tp.ldb;
        panel_end[static_cast<size_t>(j)] = io.add(1, Region{b0, b1 - b0, 1, b1 - b0}, j + 1);
    }
    const int npc = static_cast<int>(io.pieces.size());
    // events: [start][upload per piece][C panels][gemm begin/end per panel][down done]
    const size_t need = 1 + npc + chunks + 2 * chunks + 1;
    while (I.pev.size() < need) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        I.pev.push_back(e);
    }
    cudaEvent_t* ev = I.pev.data();
    cudaEvent_t ev_start = ev[0], *ev_up = ev + 1, *ev_c = ev_up + npc;
    cudaEvent_t *ev_g = ev_c + chunks, ev_down = ev_g[2 * chunks];
    io.start();
    // scratch reuse across calls: the upload must not overtake earlier work on s
    ck(cudaEventRecord(ev_start, s), "cudaEventRecord");
    ck(cudaStreamWaitEvent(I.up_stream, ev_start, 0), "cudaStreamWaitEvent");
    ck(cudaStreamWaitEvent(I.down_stream, ev_start, 0), "cudaStreamWaitEvent");
    int j_up = 0;
    for (; j_up < a_end; ++j_up) io.upload(j_up, ev_up[j_up]);
    float ms_total = 0.f;
    for (int j = 0; j < chunks; ++j) {
        for (; j_up < panel_end[static_cast<size_t>(j)]; ++j_up) io.upload(j_up, ev_up[j_up]);
        const long b0 = j * nc * I.tp.ldb;
        sm100::TcGemmProblem p = I.tp;
        p.workspace = &I.ws;
        p.A = base + typed_in[0];
        p.B = base + typed_in[1] + static_cast<size_t>(b0) * wb;
        const long c0 = j * nc * I.tp.ldc, c1 = j + 1 == chunks ? c_ext : (j + 1) * nc * I.tp.ldc;
        p.C = base + typed_c + static_cast<size_t>(c0) * wc;
        p.N = static_cast<int>(nc);
        ck(cudaEventRecord(ev_g[2 * j], s), "cudaEventRecord");
        const int r = sm100::tc_gemm_launch(I.tc, p, s);
        check_tc_launch(r);
        ck(cudaEventRecord(ev_g[2 * j + 1], s), "cudaEventRecord");
        const float* result = reinterpret_cast<const float*>(base + typed_c);
        if (ec != 0) {
            float* wide = reinterpret_cast<float*>(base + f32_c);
            ck(rt::widen_to_f32(base + typed_c + static_cast<size_t>(c0) * wc, wide + c0, c1 - c0, ec, s),
               "output conversion");
            result = wide;
        }
        ck(cudaEventRecord(ev_c[j], s), "cudaEventRecord");
        io.download(result, Region{c0, c1 - c0, 1, c1 - c0}, ev_c[j]);
    }
    ck(cudaEventRecord(ev_down, I.down_stream), "cudaEventRecord");
    ck(cudaStreamWaitEvent(s, ev_down, 0), "cudaStreamWaitEvent");
    io.finish();
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    for (int j = 0; j < chunks; ++j) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_g[2 * j], ev_g[2 * j + 1]);
        ms_total += ms;
    }
    if (std::getenv("FI_HOST_PIPELINE_TRACE")) {  // event timeline relative to the start (ms)
        auto at = [&](cudaEvent_t e) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev_start, e);
            return ms;
        };
        std::fprintf(stderr, "pipeline %d panels, ", chunks);
        io.trace_pieces(at, ev_up);
        std::fprintf(stderr, " | gemm");
        for (int j = 0; j < chunks; ++j) std::fprintf(stderr, " %.3f-%.3f", at(ev_g[2 * j]), at(ev_g[2 * j + 1]));
        std::fprintf(stderr, " | C down done %.3f\n", at(ev_down));
    }
    return ms_total;
}

}  // namespace

Plan::Plan(std::unique_ptr<Impl> impl) : impl_(std::move(impl)) {}
Plan::~Plan() = default;
const PlanInfo& Plan::info() const { return impl_->info; }
void Plan::last_host_bytes(long& up, long& down) const {
    std::lock_guard<std::mutex> g(impl_->mu);
    up = impl_->last_up;
    down = impl_->last_down;
}
const Program& Plan::program() const { return impl_->prog; }
const std::string& Plan::source() const { return impl_->source; }

std::shared_ptr<Plan> Plan::from_script(const std::string& script, long m, long n, long k, int device) {
    ParsedScript ps = parse_script(script);
    apply_size_overrides(ps, m, n, k);
    return create(ps.root, ps.tree, ps.micro_kernels, device);
}

std::shared_ptr<Plan> Plan::create(const Spec& root, const NodePtr& tree, const MicroKernelSet& mks, int device) {
    auto impl = std::make_unique<Impl>();
    impl->mks = mks;
    impl->device = device;
    impl->prog = lower(root, tree, impl->mks);  // throws on invalid trees
    Program& prog = impl->prog;
    PlanInfo& info = impl->info;
    info.grid_x = prog.launch.grid_x;
    info.grid_y = prog.launch.grid_y;
    info.block_threads = prog.launch.block_threads;
    info.entry_name = prog.entry_name;
    info.flops = root.is_matmul() ? 2.0 * static_cast<double>(root.m()) * root.n() * root.k() : 0.0;

    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaFree(nullptr), "CUDA context initialisation");

    if (prog.uses_hmma)
        throw BackendError(103, "HMMA.884.F16.TN is a Volta quad-pair leaf with no defined thread "
                                "semantics in the reference (sim.hpp:436-437); bind UMMA on sm_100a");
    if (prog.uses_tcgen05) {
        TcStrategy tc = match_tc_strategy(root, tree, impl->mks);
        if (!tc.matched) throw BackendError(103, "tensor-core tree has no sm_100a lowering: " + tc.why_not);
        const auto& mm = root.mm();
        sm100::TcGemmConfig& c = impl->tc;
        c.cta_group = tc.cta_group;
        c.bn = tc.tile_n;
        c.split_k = tc.split_k;
        c.ab_format = mm.a.elem == ElemType::BF16 ? 1 : 0;
        c.a_mn_major = mm.a.layout.major == Major::ColMajor ? 1 : 0;
        c.b_mn_major = mm.b.layout.major == Major::RowMajor ? 1 : 0;
        c.c_row_major = mm.c.layout.major == Major::RowMajor ? 1 : 0;
        c.out_type = elem_code(mm.c.elem);
        c.stages = tc.stages;
        c.slabs = tc.tile_m / (128 * tc.cta_group);
        c.n_halves = tc.tile_n == 512 ? 2 : 1;  // two N = 256 MMAs sharing A
        c.mcast = tc.mcast;
        c.bn = tc.tile_n / c.n_halves;
        // raster band: 8 tile rows; 256 x 256 pair tiles whose whole A fits in a
        // third of L2 (<= 48 MiB) sweep it column by column instead (one band of
        // every tile row): C2 4096^3 +0.9 %, 4096 x 8192 x 4096 +2-5 %; narrow
        // 1-CTA tiles on tall shapes lose 5-8 % that way, so they keep 8
        // (profiles/round2/ab_group_m.log)
        c.group_m = 8;
        if (c.cta_group == 2 && c.bn == 256 && c.slabs == 1 && c.n_halves == 1 && c.mcast == 1 &&
            static_cast<double>(root.m()) * root.k() * 2.0 <= 48.0 * (1 << 20))
            c.group_m = static_cast<int>(root.m() / 256);
        if (const char* e = std::getenv("FI_TC_GROUP_M")) c.group_m = std::atoi(e);  // raster band (experiments)
        if (sm100::tc_gemm_check(c, static_cast<int>(root.m()), static_cast<int>(root.n()),
                                 static_cast<int>(root.k())) != sm100::kTcOk)
            throw BackendError(103, "no tcgen05 kernel instance for this tile configuration");
        sm100::TcGemmProblem& p = impl->tp;
        p.M = static_cast<int>(root.m());
        p.N = static_cast<int>(root.n());
        p.K = static_cast<int>(root.k());
        p.lda = mm.a.layout.leading_dim(mm.a.rows, mm.a.cols);
        p.ldb = mm.b.layout.leading_dim(mm.b.rows, mm.b.cols);
        p.ldc = mm.c.layout.leading_dim(mm.c.rows, mm.c.cols);
        if ((p.lda * 2) % 16 || (p.ldb * 2) % 16)
            throw BackendError(103, "TMA needs 16-byte aligned operand strides (leading dim % 8)");
        p.num_sms = rt::device_sm_count();
        if (!tc.tile_order.empty()) {
            ck(cudaMalloc(&impl->d_tile_order, tc.tile_order.size() * sizeof(int32_t)), "cudaMalloc");
            ck(cudaMemcpy(impl->d_tile_order, tc.tile_order.data(), tc.tile_order.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice),
               "cudaMemcpy");
            p.tile_order = impl->d_tile_order;
        }
        // `.splitk` lowering: on CTA pairs the K slices run on separate clusters
        // (partials exchanged through L2, summed in shared memory in slice
        // order) when every (tile, slice) fits one wave -- measured 1082 vs
        // 799 TF for the in-cluster DSMEM reduction at 1024x1024x32768
        // (profiles/round1/); otherwise the cluster/DSMEM reduction.
        const long tiles = (root.m() / tc.tile_m) * (root.n() / tc.tile_n);
        if (tc.split_k > 1 && tc.cta_group == 2 && tiles * tc.split_k <= p.num_sms / 2) {
            c.split_k = 1;
            p.force_slices = tc.split_k;
            info.splitk_global = 1;
        }
        info.kind = 1;
        info.cta_group = tc.cta_group;
        info.tile_m = tc.tile_m;
        info.tile_n = tc.tile_n;
        info.split_k = tc.split_k;
        info.cluster = tc.cta_group * c.split_k * c.mcast;
        info.stages = sm100::tc_gemm_stages(c);
        info.tmem_cols = sm100::tc_gemm_tmem_cols(c);
        info.shared_bytes = sm100::tc_gemm_smem_bytes(c);
        if (const char* e = std::getenv("FI_STREAMK")) p.streamk = std::atoi(e);
        if (const char* e = std::getenv("FI_REMAINDER")) p.remainder = std::atoi(e);
        if (const char* e = std::getenv("FI_TC_MAX_CTAS")) p.max_ctas = std::atoi(e);  // experiments: smaller grid
        const sm100::TcLaunchInfo li = sm100::tc_gemm_plan(c, p);
        info.launch_ctas = li.ctas;
        info.streamk = li.streamk;
        info.remainder = li.remainder;
        impl->source = generate(prog).source;
        return std::shared_ptr<Plan>(new Plan(std::move(impl)));
    }

    // generic: emit -> NVRTC -> module
    impl->source = generate(prog).source;
    impl->smem = generic_shared_bytes(prog);
    const std::string cubin = compile_cubin(impl->source, prog.entry_name);
    const Driver& drv = Driver::get();
    drv.check(drv.module_load_data(&impl->module, cubin.data()), "cuModuleLoadData");
    drv.check(drv.module_get_function(&impl->func, impl->module, prog.entry_name.c_str()), "cuModuleGetFunction");
    if (impl->smem > 48 * 1024)
        drv.check(drv.func_set_attribute(impl->func, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                         static_cast<int>(impl->smem)),
                  "cuFuncSetAttribute");
    impl->zero_c = reads_buffer(prog.body, impl->out_root());
    info.kind = 0;
    info.shared_bytes = impl->smem;
    info.launch_ctas = prog.launch.grid_x * prog.launch.grid_y;
    return std::shared_ptr<Plan>(new Plan(std::move(impl)));
}

void Plan::launch_gated(const void* dA, const void* dB, void* dC, void* stream, const unsigned* ready,
                        unsigned epoch, long chunk_cols, int first_chunk) const {
    const Impl& I = *impl_;
    if (I.info.kind != 1) throw BackendError(103, "gated launches need a tensor-core (tcgen05) plan");
    if (!ready || chunk_cols <= 0 || I.tp.N % chunk_cols != 0 || first_chunk < 0 ||
        first_chunk >= I.tp.N / chunk_cols)
        throw BackendError(104, "gated launch: chunk_cols must divide N, first_chunk in range, flags non-null");
    sm100::TcGemmProblem p = I.tp;
    p.workspace = &I.ws;
    p.A = dA;
    p.B = dB;
    p.C = dC;
    if ((reinterpret_cast<uintptr_t>(dA) | reinterpret_cast<uintptr_t>(dB)) & 15)
        throw BackendError(104, "TMA operands must be 16-byte aligned");
    p.b_ready = ready;
    p.b_epoch = epoch;
    p.b_chunk_n = chunk_cols;
    p.b_first_chunk = first_chunk;
    const int r = sm100::tc_gemm_launch(I.tc, p, static_cast<cudaStream_t>(stream));
    if (r == sm100::kTcErrShape)
        throw BackendError(104, "gated launch: chunk_cols must be a multiple of the scheduled tile width");
    check_tc_launch(r);
}

void Plan::launch(const void* dA, const void* dB, void* dC, void* stream) const {
    const Impl& I = *impl_;
    auto s = static_cast<cudaStream_t>(stream);
    if (I.info.kind == 1) {
        sm100::TcGemmProblem p = I.tp;
        p.workspace = &I.ws;
        p.A = dA;
        p.B = dB;
        p.C = dC;
        if ((reinterpret_cast<uintptr_t>(dA) | reinterpret_cast<uintptr_t>(dB)) & 15)
            throw BackendError(104, "TMA operands must be 16-byte aligned");
        const int r = sm100::tc_gemm_launch(I.tc, p, s);
        check_tc_launch(r);
        return;
    }
    const BufferDecl& out = I.root(I.out_root());
    if (I.zero_c) ck(cudaMemsetAsync(dC, 0, static_cast<size_t>(out.extent()) * byte_width(out.elem), s), "cudaMemsetAsync");
    void* args[3];
    const void* a = dA;
    const void* b = dB;
    void* c = dC;
    int nargs = 0;
    if (I.prog.root.is_matmul()) {
        args[0] = &a;
        args[1] = &b;
        args[2] = &c;
        nargs = 3;
    } else {
        args[0] = &a;
        args[1] = &c;
        nargs = 2;
    }
    (void)nargs;
    const Driver& drv = Driver::get();
    drv.check(drv.launch_kernel(I.func, static_cast<unsigned>(I.prog.launch.grid_x),
                                static_cast<unsigned>(I.prog.launch.grid_y), 1,
                                static_cast<unsigned>(std::max<long>(1, I.prog.launch.block_threads)), 1, 1,
                                static_cast<unsigned>(I.smem), reinterpret_cast<CUstream>(s), args, nullptr),
              "cuLaunchKernel");
}

double Plan::run_host_raw(const float* A, const float* B, float* C, void* stream) const {
    const Impl& I = *impl_;
    const Spec& root = I.prog.root;
    std::lock_guard<std::mutex> g(I.mu);
    ck(cudaSetDevice(I.device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!s) {
        if (!I.own_stream) ck(cudaStreamCreateWithFlags(&I.own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        s = I.own_stream;
    }
    const int nin = root.is_matmul() ? 2 : 1;
    const float* ins[2] = {A, B};
    if (root.is_matmul() && !B) fail(ErrorKind::ShapeMismatch, "matmul execution needs both A and B inputs");
    const BufferDecl& out = I.root(I.out_root());
    // scratch: [f32 staging of each input][typed inputs][typed C][f32 C]
    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0, f32_in[2] = {0, 0}, typed_in[2] = {0, 0};
    for (int i = 0; i < nin; ++i) {
        f32_in[i] = off;
        off = align(off + static_cast<size_t>(I.root(i).extent()) * 4);
    }
    for (int i = 0; i < nin; ++i) {
        typed_in[i] = off;
        off = align(off + static_cast<size_t>(I.root(i).extent()) * byte_width(I.root(i).elem));
    }
    const size_t typed_c = off;
    off = align(off + static_cast<size_t>(out.extent()) * byte_width(out.elem));
    const size_t f32_c = off;
    off = align(off + static_cast<size_t>(out.extent()) * 4);
    if (I.scratch_bytes < off) {
        if (I.scratch) cudaFree(I.scratch);
        I.scratch = nullptr;
        ck(cudaMalloc(&I.scratch, off), "cudaMalloc");
        I.scratch_bytes = off;
    }
    auto* base = static_cast<char*>(I.scratch);
    I.last_up = I.last_down = 0;
    if (!I.ev0) {
        ck(cudaEventCreate(&I.ev0), "cudaEventCreate");
        ck(cudaEventCreate(&I.ev1), "cudaEventCreate");
    }
    if (int P = 0, Q = 0; blocked_split(I, P, Q))
        return run_host_blocked(I, A, B, C, s, P, Q, base, f32_in, typed_in, typed_c, f32_c);
    if (const int chunks = pipeline_chunks(I); chunks > 0)
        return run_host_pipelined(I, A, B, C, s, chunks, base, f32_in, typed_in, typed_c, f32_c);
    for (int i = 0; i < nin; ++i) {
        const BufferDecl& r = I.root(i);
        I.last_up += r.extent() * 4;
        if (r.elem == ElemType::F32) {  // copy straight into the typed buffer
            ck(cudaMemcpyAsync(base + typed_in[i], ins[i], static_cast<size_t>(r.extent()) * 4,
                               cudaMemcpyHostToDevice, s),
               "cudaMemcpyAsync");
            continue;
        }
        ck(cudaMemcpyAsync(base + f32_in[i], ins[i], static_cast<size_t>(r.extent()) * 4, cudaMemcpyHostToDevice, s),
           "cudaMemcpyAsync");
        // snapping to the root's element grid on ingestion (sim.hpp:507-510)
        ck(rt::convert_f32(reinterpret_cast<float*>(base + f32_in[i]), base + typed_in[i], r.extent(),
                           elem_code(r.elem), s),
           "input conversion");
    }
    ck(cudaEventRecord(I.ev0, s), "cudaEventRecord");
    launch(base + typed_in[0], nin > 1 ? base + typed_in[1] : nullptr, base + typed_c, s);
    ck(cudaEventRecord(I.ev1, s), "cudaEventRecord");
    const void* result = base + typed_c;
    if (out.elem != ElemType::F32) {
        ck(rt::widen_to_f32(base + typed_c, reinterpret_cast<float*>(base + f32_c), out.extent(),
                            elem_code(out.elem), s),
           "output conversion");
        result = base + f32_c;
    }
    ck(cudaMemcpyAsync(C, result, static_cast<size_t>(out.extent()) * 4, cudaMemcpyDeviceToHost, s),
       "cudaMemcpyAsync");
    I.last_down = out.extent() * 4;
    ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, I.ev0, I.ev1);
    return ms;
}

RunResult Plan::run_host(const Matrix& a, const Matrix* b, void* stream) const {
    const Impl& I = *impl_;
    const Spec& root = I.prog.root;
    const int nin = root.is_matmul() ? 2 : 1;
    const Matrix* ins[2] = {&a, b};
    if (root.is_matmul() && !b) fail(ErrorKind::ShapeMismatch, "matmul execution needs both A and B inputs");
    std::vector<float> staged[2];
    const float* ptr[2] = {nullptr, nullptr};
    for (int i = 0; i < nin; ++i) {
        const BufferDecl& r = I.root(i);
        if (ins[i]->rows != r.rows || ins[i]->cols != r.cols)
            fail(ErrorKind::ShapeMismatch, "input for " + r.name + " must be " + std::to_string(r.rows) + "x" +
                                               std::to_string(r.cols));
        if (static_cast<long>(ins[i]->data.size()) == r.extent() && ins[i]->layout == r.layout) {
            ptr[i] = ins[i]->data.data();
            continue;
        }
        // re-lay the logical matrix into the root's physical layout (pads = 0)
        Matrix tmp = Matrix::zeros(r.rows, r.cols, r.layout);
        for (long rr = 0; rr < r.rows; ++rr)
            for (long cc = 0; cc < r.cols; ++cc) tmp.at(rr, cc) = ins[i]->at(rr, cc);
        staged[i] = std::move(tmp.data);
        ptr[i] = staged[i].data();
    }
    const BufferDecl& out = I.root(I.out_root());
    RunResult res;
    res.output = Matrix::zeros(out.rows, out.cols, out.layout);
    res.device_ms = run_host_raw(ptr[0], ptr[1], res.output.data.data(), stream);
    return res;
}

// ---------------------------------------------------------------- run (drop-in)
namespace {
void collect_micro_kernels(const StmtList& body, MicroKernelSet& mks) {
    for (const auto& s : body) {
        if (const auto* l = std::get_if<LoopStmt>(&s.v)) collect_micro_kernels(l->body, mks);
        if (const auto* m = std::get_if<MicroKernelStmt>(&s.v))
            if (m->mk && !mks.find(m->mk->name)) mks.register_kernel(*m->mk);
    }
}
}  // namespace

RunResult run(const Program& prog, const Matrix& a, const Matrix* b, RunOptions opts) {
    if (!prog.tree) fail(ErrorKind::InvalidTree, "program carries no strategy tree (build it with lower())");
    MicroKernelSet mks;
    collect_micro_kernels(prog.body, mks);
    auto plan = Plan::create(prog.root, prog.tree, mks, opts.device);
    return plan->run_host(a, b, opts.stream);
}

RunResult run(const Spec& root, const NodePtr& tree, const Matrix& a, const Matrix* b, RunOptions opts,
              const MicroKernelSet& mks) {
    auto plan = Plan::create(root, tree, mks, opts.device);
    return plan->run_host(a, b, opts.stream);
}

}  // namespace fireiron
