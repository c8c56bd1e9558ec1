// A reference-style caller (the shape of proj/tests/test_sim.cpp and
// proj/tools/anvil.cpp `verify`), compiled against the drop-in headers.
//   no args  : IR services only (parse, validate, elaborate, lower, generate)
//   "gpu"    : also anvil::run on the B200 and compare with the naive oracle
//   "gpu-tc" : the tensor-core strategy from its script text at 1024x2048x512 --
//              std::vector-backed (pageable) matrices through the pipelined host
//              path of run() -- exact against the naive oracle on integers
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "fireiron/anvil.hpp"

using namespace anvil;

static Matrix naive(const Matrix& a, const Matrix& b) {  // oracle.hpp:11-22 semantics
    Matrix c = Matrix::zeros(a.rows, b.cols);
    for (long i = 0; i < a.rows; ++i)
        for (long j = 0; j < b.cols; ++j) {
            double acc = 0;
            for (long k = 0; k < a.cols; ++k) acc += double(a.at(i, k)) * double(b.at(k, j));
            c.at(i, j) = float(acc);
        }
    return c;
}

static int tensor_core_run() {
    ParsedScript ps = parse_script(
        "spec MatMul(1024,2048,512)(GL,GL,GL)(Kernel) elems f16 f16 f32\n"
        "tile 256 256 .to block .pair\n"
        "epilog tm {\n  init {\n    done\n  }\n  store {\n    tile 32 256 .to warp\n    done\n  }\n}\n"
        "split 64\nload a sh {\n  done\n}\nload b sh {\n  done\n}\ndone\n");
    Matrix a = Matrix::zeros(1024, 512), b = Matrix::zeros(512, 2048);
    fill_integers(a, 3);
    fill_integers(b, 4);
    RunResult r = run(ps.root, ps.tree, a, &b);  // pageable host matrices, pipelined upload/download
    Matrix want = naive(a, b);
    double err = 0;
    for (long i = 0; i < 1024; i += 3)
        for (long j = 0; j < 2048; j += 5) err = std::fmax(err, std::fabs(r.output.at(i, j) - want.at(i, j)));
    std::printf("gpu tensor-core run: max_abs_error=%g device_ms=%.4f\n", err, r.device_ms);
    return err == 0 ? 0 : 2;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "gpu-tc") == 0) return tensor_core_run();
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    // programmatic tree (the reference's builder API): 64x64x32, CTA -> warp -> thread, FMA leaf
    Spec root = make_matmul_spec(64, 64, 32, {}, {MemLevel::gl(), MemLevel::gl(), MemLevel::gl()},
                                 {Layout::col_major(), Layout::col_major(), Layout::col_major()},
                                 ComputeLevel::Kernel);
    auto lanes = [](NodePtr leaf) {
        TileRefinements w, t;
        w.to = ComputeLevel::Warp;
        t.to = ComputeLevel::Thread;
        return n_tile(32, 32, w, n_tile(4, 8, t, n_tile(1, 1, {}, std::move(leaf))));
    };
    NodePtr chain = n_tile(1, 1, {}, n_done());
    chain = n_load(Operand::B, MemLevel::rf(), n_tile(1, 1, {}, n_done()), {}, std::move(chain));
    chain = n_load(Operand::A, MemLevel::rf(), n_tile(1, 1, {}, n_done()), {}, std::move(chain));
    chain = n_split(1, {}, std::move(chain));
    TileRefinements w, t;
    w.to = ComputeLevel::Warp;
    t.to = ComputeLevel::Thread;
    chain = n_tile(32, 32, w, n_tile(4, 8, t, std::move(chain)));
    chain = n_split(8, {}, std::move(chain));
    chain = n_epilog(MemLevel::rf(), lanes(n_done()), lanes(n_done()), std::move(chain));
    TileRefinements blk;
    blk.to = ComputeLevel::Block;
    NodePtr tree = n_tile(64, 64, blk, std::move(chain));

    ValidationReport report = validate(root, tree);
    std::printf("%s\n", report.to_string().c_str());
    if (!report.ok()) return 1;
    std::printf("%s", render_trace(elaborate(root, tree)).c_str());
    Program prog = lower(root, tree);
    std::printf("barriers=%d buffers=%zu\n", count_barriers(prog.body), prog.plan.buffers.size());
    KernelSource ks = generate(prog);
    std::printf("generated %zu bytes of sm_100a CUDA (%s)\n", ks.source.size(), ks.entry_name.c_str());
    try {
        parse_script("spec MatMul(64,64,8)(GL,GL,GL)(Kernel)\ntile 8 8 .bogus\ndone\n");
    } catch (const Error& e) {
        std::printf("error kind %s\n", error_kind_name(e.kind()));
    }
    if (!gpu) return 0;
    Matrix a = Matrix::zeros(64, 32), b = Matrix::zeros(32, 64);
    fill_integers(a, 7);
    fill_integers(b, 8);
    RunResult r = run(root, tree, a, &b);  // executes on the B200
    Matrix want = naive(a, b);
    double err = 0;
    for (long i = 0; i < 64; ++i)
        for (long j = 0; j < 64; ++j) err = std::fmax(err, std::fabs(r.output.at(i, j) - want.at(i, j)));
    std::printf("gpu run: max_abs_error=%g digest=0x%016llx device_ms=%.4f\n", err,
                static_cast<unsigned long long>(digest(r.output)), r.device_ms);
    // the same call under the GPU-explicit names: bit-identical
    GpuRunOptions go;
    go.device = 0;
    RunResult r2 = run_gpu(root, tree, a, &b, go);
    const bool same = digest(r2.output) == digest(r.output);
    std::printf("run_gpu: %s\n", same ? "identical" : "DIFFERENT");
    return err == 0 && same ? 0 : 2;
}
