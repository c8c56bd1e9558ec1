// ref_driver.cpp -- drives the UNMODIFIED reference implementation ("anvil",
// header-only C++20, compiled in place from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/). TEST INFRASTRUCTURE ONLY: this is the
// parity oracle and the CPU baseline arm of bench.py, never the product.
//
// Exposes a small C API (for ctypes) plus a CLI:
//   ref_run            -- anvil::run (sim.hpp:495) on caller-provided inputs
//   ref_time_blocks    -- per-block timing through anvil::detail::Machine
//                         (sim.hpp:189-485, 517-526): the CPU baseline sample
//   ref_elaborate / ref_plan / ref_codegen -- text fixtures for IR parity tests
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "anvil/anvil.hpp"
#include "support/tree_gen.hpp"

using namespace anvil;

namespace {

thread_local std::string g_err;

int fail_code(const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.kind()) + 1;
}

ParsedScript load(const char* script, int64_t m, int64_t n, int64_t k) {
    ParsedScript s = parse_script(script);
    // --m/--n/--k overrides, as tools/anvil.cpp:29-60 re-derives the root
    if (m > 0 || n > 0 || k > 0) {
        if (s.root.is_matmul()) {
            auto& mm = s.root.mm();
            long M = m > 0 ? m : s.root.m(), N = n > 0 ? n : s.root.n(), K = k > 0 ? k : s.root.k();
            mm.a.rows = M; mm.a.cols = K; mm.b.rows = K; mm.b.cols = N; mm.c.rows = M; mm.c.cols = N;
        } else {
            auto& mv = s.root.mv();
            long R = m > 0 ? m : mv.src.rows, Cc = n > 0 ? n : mv.src.cols;
            mv.src.rows = mv.dst.rows = R;
            mv.src.cols = mv.dst.cols = Cc;
        }
        MicroKernelSet rebuilt;
        for (const auto& sec : s.micro_kernel_sections) {
            MicroKernel mk;
            mk.name = sec.name;
            mk.pattern = parse_spec_short_form(sec.pattern_line, &s.root, sec.line);
            mk.body = sec.body;
            mk.declared_vars = sec.vars;
            rebuilt.register_kernel(std::move(mk));
        }
        s.micro_kernels = std::move(rebuilt);
    }
    return s;
}

// logical row-major float buffer -> Matrix in the given layout
Matrix from_logical(const float* src, long rows, long cols, Layout l) {
    Matrix m = Matrix::zeros(rows, cols, l);
    for (long r = 0; r < rows; ++r)
        for (long c = 0; c < cols; ++c) m.at(r, c) = src[r * cols + c];
    return m;
}

int copy_text(const std::string& s, char* buf, int64_t cap) {
    if (buf && cap > 0) {
        size_t nn = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::memcpy(buf, s.data(), nn);
        buf[nn] = 0;
    }
    return static_cast<int>(s.size());
}

const char* mem_tok(const MemLevel& m) {
    switch (m.kind) {
        case MemKind::GL: return "GL";
        case MemKind::SH: return "SH";
        case MemKind::RF: return "RF";
        case MemKind::FR: return "FR";
    }
    return "?";
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Runs the reference simulator. A/B/out are logical row-major fp32 (out is
// M x N for MatMul, R x C for Move). Returns 0 or ErrorKind+1; *races gets the
// race total.
int ref_run(const char* script, int64_t m, int64_t n, int64_t k, const float* A, const float* B,
            float* out, int64_t* races, int64_t* ownership) {
    try {
        ParsedScript s = load(script, m, n, k);
        Program prog = lower(s.root, s.tree, s.micro_kernels);
        RunOptions opts;
        opts.collect_ownership = ownership != nullptr;
        RunResult r;
        if (s.root.is_matmul()) {
            Matrix a = from_logical(A, s.root.m(), s.root.k(), s.root.mm().a.layout);
            Matrix b = from_logical(B, s.root.k(), s.root.n(), s.root.mm().b.layout);
            r = run(prog, a, &b, opts);
        } else {
            const auto& src = s.root.mv().src;
            Matrix a = from_logical(A, src.rows, src.cols, src.layout);
            r = run(prog, a, nullptr, opts);
        }
        for (long i = 0; i < r.output.rows; ++i)
            for (long j = 0; j < r.output.cols; ++j) out[i * r.output.cols + j] = r.output.at(i, j);
        if (races) *races = r.races.total;
        if (ownership) *ownership = static_cast<int64_t>(r.ownership.size());
        return 0;
    } catch (const Error& e) {
        return fail_code(e);
    }
}

// Generates the reference inputs (fill_integers / fill_uniform, A seed s, B
// seed s+1 as tools/anvil.cpp:79-101) into logical row-major buffers.
int ref_make_inputs(const char* script, int64_t m, int64_t n, int64_t k, uint64_t seed,
                    int float_mode, float* A, float* B) {
    try {
        ParsedScript s = load(script, m, n, k);
        auto gen = [&](long rows, long cols, uint64_t sd, float* dst) {
            Matrix mm = Matrix::zeros(rows, cols, Layout::row_major());
            if (float_mode) fill_uniform(mm, sd);
            else fill_integers(mm, sd);
            for (long r = 0; r < rows; ++r)
                for (long c = 0; c < cols; ++c) dst[r * cols + c] = mm.at(r, c);
        };
        if (s.root.is_matmul()) {
            gen(s.root.m(), s.root.k(), seed, A);
            if (B) gen(s.root.k(), s.root.n(), seed + 1, B);
        } else {
            gen(s.root.mv().src.rows, s.root.mv().src.cols, seed, A);
        }
        return 0;
    } catch (const Error& e) {
        return fail_code(e);
    }
}

// Digest of the reference run on its own seeded inputs (as `anvil simulate`).
int ref_simulate_digest(const char* script, int64_t m, int64_t n, int64_t k, uint64_t seed,
                        int float_mode, uint64_t* digest_out, int64_t* races) {
    try {
        ParsedScript s = load(script, m, n, k);
        Program prog = lower(s.root, s.tree, s.micro_kernels);
        RunResult r;
        if (s.root.is_matmul()) {
            Matrix a = Matrix::zeros(s.root.m(), s.root.k(), s.root.mm().a.layout);
            Matrix b = Matrix::zeros(s.root.k(), s.root.n(), s.root.mm().b.layout);
            if (float_mode) { fill_uniform(a, seed); fill_uniform(b, seed + 1); }
            else { fill_integers(a, seed); fill_integers(b, seed + 1); }
            r = run(prog, a, &b, {});
        } else {
            const auto& src = s.root.mv().src;
            Matrix a = Matrix::zeros(src.rows, src.cols, src.layout);
            if (float_mode) fill_uniform(a, seed); else fill_integers(a, seed);
            r = run(prog, a, nullptr, {});
        }
        *digest_out = digest(r.output);
        if (races) *races = r.races.total;
        return 0;
    } catch (const Error& e) {
        return fail_code(e);
    }
}

// CPU baseline: execute `blocks` CTA blocks (round-robin over the grid,
// starting at block 0) of the lowered program through the reference Machine
// on `threads` host threads (one Machine each, disjoint blocks), as
// BASELINE.md section 4 prescribes. Returns seconds in *secs and the grid
// size in *grid_blocks; the caller extrapolates.
int ref_time_blocks(const char* script, int64_t m, int64_t n, int64_t k, int64_t blocks,
                    int threads, double* secs, int64_t* grid_blocks) {
    try {
        ParsedScript s = load(script, m, n, k);
        Program prog = lower(s.root, s.tree, s.micro_kernels);
        if (!prog.simulatable) fail(ErrorKind::UnsimulatableResidual, "codegen-only tree");
        const long gx = prog.launch.grid_x, gy = prog.launch.grid_y;
        const long total = gx * gy;
        *grid_blocks = total;
        if (blocks > total) blocks = total;
        if (threads < 1) threads = 1;
        Matrix a, b;
        if (s.root.is_matmul()) {
            a = Matrix::zeros(s.root.m(), s.root.k(), s.root.mm().a.layout);
            b = Matrix::zeros(s.root.k(), s.root.n(), s.root.mm().b.layout);
            fill_uniform(a, 1);
            fill_uniform(b, 2);
        } else {
            a = Matrix::zeros(s.root.mv().src.rows, s.root.mv().src.cols, s.root.mv().src.layout);
            fill_uniform(a, 1);
        }
        std::atomic<long> next{0};
        std::vector<std::thread> pool;
        std::vector<std::string> errs(static_cast<size_t>(threads));
        auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    detail::Machine mach(prog, RunOptions{});
                    mach.env.resize(16, 0);
                    if (s.root.is_matmul()) {
                        mach.ingest(0, a, s.root.mm().a.elem == ElemType::F16);
                        mach.ingest(1, b, s.root.mm().b.elem == ElemType::F16);
                    } else {
                        mach.ingest(0, a, s.root.mv().src.elem == ElemType::F16);
                    }
                    for (long i = next++; i < blocks; i = next++) {
                        long lin = (i * 7919) % total;  // spread the sample over the grid
                        long bx = lin % gx, by = lin / gx;
                        mach.block_x = bx;
                        mach.block_y = by;
                        mach.block_linear = lin;
                        mach.env[static_cast<size_t>(mach.slot_bx)] = bx;
                        mach.env[static_cast<size_t>(mach.slot_by)] = by;
                        mach.reset_block();
                        mach.exec_list(prog.body);
                    }
                } catch (const std::exception& e) {
                    errs[static_cast<size_t>(t)] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto& e : errs)
            if (!e.empty()) { g_err = e; return 100; }
        return 0;
    } catch (const Error& e) {
        return fail_code(e);
    }
}

int ref_elaborate(const char* script, int with_subs, char* buf, int64_t cap) {
    try {
        ParsedScript s = parse_script(script);
        auto trace = elaborate(s.root, s.tree, s.micro_kernels);
        return copy_text(render_trace(trace, with_subs != 0), buf, cap);
    } catch (const Error& e) {
        return -fail_code(e);
    }
}

int ref_validate(const char* script, int64_t m, int64_t n, int64_t k, char* buf, int64_t cap) {
    try {
        ParsedScript s = load(script, m, n, k);
        ValidationReport r = validate_with_plan(s.root, s.tree, s.micro_kernels);
        return copy_text(r.to_string(), buf, cap);
    } catch (const Error& e) {
        return -fail_code(e);
    }
}

// Buffer plan + program summary, one line per buffer.
int ref_plan(const char* script, int64_t m, int64_t n, int64_t k, char* buf, int64_t cap) {
    try {
        ParsedScript s = load(script, m, n, k);
        Program p = lower(s.root, s.tree, s.micro_kernels);
        std::ostringstream o;
        o << "entry " << p.entry_name << "\n";
        o << "grid " << p.launch.grid_x << " " << p.launch.grid_y << " warps "
          << p.launch.warps_per_block << " threads " << p.launch.block_threads << "\n";
        o << "shared_bytes " << p.plan.shared_bytes << "\n";
        o << "barriers " << count_barriers(p.body) << "\n";
        o << "simulatable " << (p.simulatable ? 1 : 0) << " wmma " << (p.uses_wmma ? 1 : 0) << "\n";
        for (const auto& b : p.plan.buffers)
            o << "buf " << b.id << " " << b.name << " " << mem_tok(b.mem) << " "
              << elem_name(b.elem) << " " << b.rows << "x" << b.cols << " local " << b.local_rows
              << "x" << b.local_cols << " " << (b.layout.major == Major::RowMajor ? "row" : "col")
              << " pad " << b.layout.pad_cols << " extent " << b.extent() << " align "
              << b.align_bytes << " home " << level_name(b.home) << " root " << (b.is_root ? 1 : 0)
              << " alias " << b.alias_of << "\n";
        return copy_text(o.str(), buf, cap);
    } catch (const Error& e) {
        return -fail_code(e);
    }
}

int ref_codegen(const char* script, int64_t m, int64_t n, int64_t k, char* buf, int64_t cap) {
    try {
        ParsedScript s = load(script, m, n, k);
        return copy_text(generate(s.root, s.tree, s.micro_kernels).source, buf, cap);
    } catch (const Error& e) {
        return -fail_code(e);
    }
}

// The reference's random register-blocked tree generator
// (proj/tests/support/tree_gen.hpp:60-162), printed as a canonical script.
int ref_corpus_script(uint64_t seed, char* buf, int64_t cap) {
    try {
        auto gen = anvil::testing::random_tree(seed);
        ParsedScript ps;
        ps.root = gen.root;
        ps.tree = gen.tree;
        return copy_text(print_script(ps), buf, cap);
    } catch (const Error& e) {
        return -fail_code(e);
    }
}

int ref_print(const char* script, char* buf, int64_t cap) {
    try {
        return copy_text(print_script(parse_script(script)), buf, cap);
    } catch (const Error& e) {
        return -fail_code(e);
    }
}

}  // extern "C"

#ifdef REF_MAIN
// CLI: ref_anvil digest <script.fi> [m n k seed float]
//      ref_anvil time <script.fi> m n k blocks threads
int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s digest|time|plan|elaborate <script> [...]\n", argv[0]);
        return 2;
    }
    std::ifstream in(argv[2]);
    std::stringstream ss;
    ss << in.rdbuf();
    std::string text = ss.str();
    std::string cmd = argv[1];
    auto arg = [&](int i, long d) { return argc > i ? std::atol(argv[i]) : d; };
    if (cmd == "digest") {
        uint64_t d = 0;
        int64_t races = 0;
        int rc = ref_simulate_digest(text.c_str(), arg(3, 0), arg(4, 0), arg(5, 0),
                                     static_cast<uint64_t>(arg(6, 1)), static_cast<int>(arg(7, 0)), &d,
                                     &races);
        if (rc) { std::fprintf(stderr, "error: %s\n", ref_last_error()); return 1; }
        std::printf("digest=0x%016llx races=%lld\n", static_cast<unsigned long long>(d),
                    static_cast<long long>(races));
        return 0;
    }
    if (cmd == "time") {
        double secs = 0;
        int64_t grid = 0;
        int rc = ref_time_blocks(text.c_str(), arg(3, 0), arg(4, 0), arg(5, 0), arg(6, 1),
                                 static_cast<int>(arg(7, 1)), &secs, &grid);
        if (rc) { std::fprintf(stderr, "error: %s\n", ref_last_error()); return 1; }
        std::printf("blocks=%ld grid=%lld secs=%.6f\n", arg(6, 1), static_cast<long long>(grid), secs);
        return 0;
    }
    std::vector<char> buf(1 << 22);
    int rc = 0;
    if (cmd == "plan") rc = ref_plan(text.c_str(), arg(3, 0), arg(4, 0), arg(5, 0), buf.data(), buf.size());
    else if (cmd == "elaborate") rc = ref_elaborate(text.c_str(), static_cast<int>(arg(3, 0)), buf.data(), buf.size());
    else if (cmd == "codegen") rc = ref_codegen(text.c_str(), arg(3, 0), arg(4, 0), arg(5, 0), buf.data(), buf.size());
    else { std::fprintf(stderr, "unknown command\n"); return 2; }
    if (rc < 0) { std::fprintf(stderr, "error: %s\n", ref_last_error()); return 1; }
    std::fputs(buf.data(), stdout);
    return 0;
}
#endif
