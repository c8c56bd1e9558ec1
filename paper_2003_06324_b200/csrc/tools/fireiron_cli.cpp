// fireiron: the anvil CLI (proj/tools/anvil.cpp:145-269) re-targeted to the
// B200 backend. Same subcommands, flags, output lines and exit contract:
//   fireiron elaborate <script.fi> [--m M --n N --k K] [--dump-trace]
//   fireiron codegen   <script.fi> [--m ...] [--out file]
//   fireiron simulate  <script.fi> [--m ...] [--seed S] [--float] [--load-a f] [--load-b f] [--dump-c f]
//   fireiron verify    <script.fi> [--m ...] [--seed S] [--float] [--tolerance T]
// simulate/verify execute on the GPU (anvil::run equivalent); races and
// ownership are reported as 0 (the GPU runs race-free programs only).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "fireiron/async_check.hpp"
#include "fireiron/anvil.hpp"

using namespace fireiron;

namespace {

struct Args {
    std::string cmd, script;
    long m = 0, n = 0, k = 0;
    uint64_t seed = 1;
    bool float_mode = false, dump_trace = false;
    double tolerance = -1.0;
    std::string out, load_a, load_b, dump_c;
    int gated_chunks = 0, gated_first = 0;  // check-async: model a gated launch
};

[[noreturn]] void usage() {
    std::fprintf(stderr,
                 "usage: fireiron {elaborate|codegen|simulate|verify|check-async} <script.fi> [--m M] [--n N] [--k K]\n"
                 "       [--seed S] [--float] [--load-a F] [--load-b F] [--dump-c F] [--tolerance T]\n"
                 "       [--dump-trace] [--out F] [--gated-chunks C [--gated-first F]]\n");
    std::exit(2);
}

Args parse_args(int argc, char** argv) {
    if (argc < 3) usage();
    Args a;
    a.cmd = argv[1];
    a.script = argv[2];
    for (int i = 3; i < argc; ++i) {
        const std::string f = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage();
            return argv[++i];
        };
        if (f == "--m") a.m = std::stol(val());
        else if (f == "--n") a.n = std::stol(val());
        else if (f == "--k") a.k = std::stol(val());
        else if (f == "--seed") a.seed = std::stoull(val());
        else if (f == "--float") a.float_mode = true;
        else if (f == "--dump-trace") a.dump_trace = true;
        else if (f == "--tolerance") a.tolerance = std::stod(val());
        else if (f == "--out") a.out = val();
        else if (f == "--load-a") a.load_a = val();
        else if (f == "--load-b") a.load_b = val();
        else if (f == "--dump-c") a.dump_c = val();
        else if (f == "--gated-chunks") a.gated_chunks = std::stoi(val());
        else if (f == "--gated-first") a.gated_first = std::stoi(val());
        else usage();
    }
    return a;
}

std::string slurp(const std::string& path) {
    std::ifstream in(path);
    if (!in) fail(ErrorKind::IoError, "cannot open '" + path + "'");
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

ParsedScript load(const Args& a) {  // tools/anvil.cpp:62-72
    ParsedScript s = parse_script(slurp(a.script));
    apply_size_overrides(s, a.m, a.n, a.k);
    ValidationReport r = validate(s.root, s.tree, s.micro_kernels);
    if (!r.ok()) {
        std::cerr << "validation failed for " << a.script << ":\n" << r.to_string();
        std::exit(1);
    }
    return s;
}

struct Inputs {
    Matrix a, b;
    bool has_b = false;
};

Inputs make_inputs(const ParsedScript& s, const Args& a) {  // tools/anvil.cpp:79-101
    Inputs in;
    const Spec& root = s.root;
    auto gen = [&](Matrix& m, const std::string& load_path, Layout l, uint64_t seed) {
        if (!load_path.empty()) m = read_matrix(load_path, l);
        else if (a.float_mode) fill_uniform(m, seed);
        else fill_integers(m, seed);
    };
    if (root.is_matmul()) {
        in.has_b = true;
        in.a = Matrix::zeros(root.m(), root.k(), root.mm().a.layout);
        in.b = Matrix::zeros(root.k(), root.n(), root.mm().b.layout);
        gen(in.a, a.load_a, root.mm().a.layout, a.seed);
        gen(in.b, a.load_b, root.mm().b.layout, a.seed + 1);
    } else {
        in.a = Matrix::zeros(root.mv().src.rows, root.mv().src.cols, root.mv().src.layout);
        gen(in.a, a.load_a, root.mv().src.layout, a.seed);
    }
    return in;
}

Matrix oracle(const ParsedScript& s, const Inputs& in) {  // tools/anvil.cpp:105-125 semantics
    const Spec& root = s.root;
    if (root.is_move()) {
        Matrix out = in.a;
        round_matrix(out, root.mv().src.elem);
        return out;
    }
    Matrix a = in.a, b = in.b;
    round_matrix(a, root.mm().a.elem);
    round_matrix(b, root.mm().b.elem);
    Matrix c = Matrix::zeros(root.m(), root.n(), root.mm().c.layout);
    for (long i = 0; i < root.m(); ++i)
        for (long j = 0; j < root.n(); ++j) {
            double acc = 0.0;
            for (long kk = 0; kk < root.k(); ++kk) acc += double(a.at(i, kk)) * double(b.at(kk, j));
            c.at(i, j) = static_cast<float>(acc);
        }
    return c;
}

}  // namespace

int main(int argc, char** argv) {
    const Args a = parse_args(argc, argv);
    try {
        if (a.cmd == "elaborate") {
            ParsedScript s = load(a);
            std::cout << render_trace(elaborate(s.root, s.tree, s.micro_kernels), a.dump_trace);
            return 0;
        }
        if (a.cmd == "codegen") {
            ParsedScript s = load(a);
            const KernelSource ks = generate(s.root, s.tree, s.micro_kernels);
            if (a.out.empty()) {
                std::cout << ks.source;
            } else {
                std::ofstream o(a.out);
                if (!o) fail(ErrorKind::IoError, "cannot write '" + a.out + "'");
                o << ks.source;
            }
            return 0;
        }
        if (a.cmd == "check-async") {  // CPU protocol check of the tcgen05 launch (no GPU)
            ParsedScript s = load(a);
            AsyncCheckOptions o;
            o.gated_chunks = a.gated_chunks;
            o.gated_first = a.gated_first;
            const AsyncReport r = check_async(s.root, s.tree, o, s.micro_kernels);
            std::cout << r.to_string();
            return r.ok() ? 0 : 1;
        }
        if (a.cmd == "simulate" || a.cmd == "verify") {
            ParsedScript s = load(a);
            auto plan = Plan::create(s.root, s.tree, s.micro_kernels);
            Inputs in = make_inputs(s, a);
            RunResult r = plan->run_host(in.a, in.has_b ? &in.b : nullptr);
            if (a.cmd == "simulate") {
                if (!a.dump_c.empty()) write_matrix(a.dump_c, r.output);
                double max_abs = 0.0;
                for (long i = 0; i < r.output.rows; ++i)
                    for (long j = 0; j < r.output.cols; ++j) max_abs = std::max(max_abs, std::fabs(double(r.output.at(i, j))));
                std::printf("c %ldx%ld digest=0x%016llx max_abs=%g races=%ld device_ms=%.4f\n", r.output.rows,
                            r.output.cols, static_cast<unsigned long long>(digest(r.output)), max_abs, r.races.total,
                            r.device_ms);
                return 0;
            }
            const Matrix want = oracle(s, in);
            double err = 0.0;
            for (long i = 0; i < want.rows; ++i)
                for (long j = 0; j < want.cols; ++j)
                    err = std::max(err, std::fabs(double(r.output.at(i, j)) - double(want.at(i, j))));
            const double tol = a.tolerance >= 0 ? a.tolerance : (a.float_mode ? 1e-3 : 0.0);
            const bool ok = err <= tol;
            std::printf("%s max_error=%g tolerance=%g races=0 ownership_violations=0 backend=%s\n", ok ? "PASS" : "FAIL",
                        err, tol, plan->info().kind == 1 ? "tcgen05" : "generic");
            return ok ? 0 : 1;
        }
        usage();
    } catch (const Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
