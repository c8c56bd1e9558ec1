// Built-in leaves and residual matching (reference: proj/include/anvil/exec.hpp).
#include "fireiron/exec.hpp"

namespace fireiron {

bool OperandPattern::matches(const MatrixRef& m) const {
    if (rows && *rows != m.rows) return false;
    if (cols && *cols != m.cols) return false;
    if (elem && *elem != m.elem) return false;
    if (!mems.empty()) {
        bool any = false;
        for (MemKind k : mems) any = any || k == m.mem.kind;
        if (!any) return false;
    }
    return !major || *major == m.layout.major;
}

bool Instruction::matches(const Spec& s) const {
    if (s.kind != kind || s.level != level) return false;
    if (s.is_matmul()) return a.matches(s.mm().a) && b.matches(s.mm().b) && c.matches(s.mm().c);
    return a.matches(s.mv().src) && c.matches(s.mv().dst);
}

std::string Instruction::pattern_short_form() const {
    auto d = [](const std::optional<long>& v) { return v ? std::to_string(*v) : std::string("_"); };
    if (kind == Spec::Kind::MatMul)
        return "MatMul(" + d(c.rows) + "," + d(c.cols) + "," + d(a.cols) + ")(...)(" +
               level_name(level) + ")";
    auto one_mem = [](const OperandPattern& p) {
        return p.mems.size() == 1 ? mem_name(MemLevel{p.mems[0]}) : std::string("_");
    };
    return "Move(" + d(c.rows) + "x" + d(c.cols) + ")(" + one_mem(a) + "->" + one_mem(c) + ")(" +
           level_name(level) + ")";
}

bool Instruction::is_tensor_core_sm100() const {
    return sim == SimSemantics::TMA_LOAD || sim == SimSemantics::UMMA ||
           sim == SimSemantics::TMEM_ZERO || sim == SimSemantics::TMEM_STORE;
}

namespace {

OperandPattern pat(std::optional<long> r, std::optional<long> c, std::optional<ElemType> e,
                   std::vector<MemKind> mems, std::optional<Major> mj = std::nullopt) {
    OperandPattern p;
    p.rows = r;
    p.cols = c;
    p.elem = e;
    p.mems = std::move(mems);
    p.major = mj;
    return p;
}

Instruction make(std::string name, Spec::Kind kind, ComputeLevel level, OperandPattern a,
                 OperandPattern b, OperandPattern c, SimSemantics sim, std::string emission = "") {
    Instruction i;
    i.name = std::move(name);
    i.kind = kind;
    i.level = level;
    i.a = std::move(a);
    i.b = std::move(b);
    i.c = std::move(c);
    i.sim = sim;
    i.emission = std::move(emission);
    return i;
}

std::vector<Instruction> build_builtins() {
    using K = Spec::Kind;
    using L = ComputeLevel;
    const auto RF = MemKind::RF, FR = MemKind::FR, GL = MemKind::GL, SH = MemKind::SH,
               TM = MemKind::TM;
    std::vector<Instruction> v;
    // the reference's seven leaves (exec.hpp:76-148)
    v.push_back(make("FMA", K::MatMul, L::Thread, pat(1, 1, ElemType::F32, {RF}),
                     pat(1, 1, ElemType::F32, {RF}), pat(1, 1, ElemType::F32, {RF}),
                     SimSemantics::FMA, "{C} += {A} * {B};"));
    v.push_back(make("HFMA", K::MatMul, L::Thread, pat(1, 1, ElemType::F16, {RF}),
                     pat(1, 1, ElemType::F16, {RF}), pat(1, 1, ElemType::F16, {RF}),
                     SimSemantics::FMA, "{C} += {A} * {B};"));
    v.push_back(make("COPY", K::Move, L::Thread, pat(1, 1, std::nullopt, {}), {},
                     pat(1, 1, std::nullopt, {}), SimSemantics::FMA, "{DST} = {SRC};"));
    v.push_back(make("WMMA_MMA", K::MatMul, L::Warp, pat(16, 16, ElemType::F16, {FR}),
                     pat(16, 16, ElemType::F16, {FR}), pat(16, 16, std::nullopt, {FR}),
                     SimSemantics::WMMA_MMA));
    v.push_back(make("WMMA_LOAD", K::Move, L::Warp, pat(16, 16, std::nullopt, {}), {},
                     pat(16, 16, std::nullopt, {FR}), SimSemantics::WMMA_LOAD));
    v.push_back(make("WMMA_STORE", K::Move, L::Warp, pat(16, 16, std::nullopt, {FR}), {},
                     pat(16, 16, std::nullopt, {GL, SH, RF}), SimSemantics::WMMA_STORE));
    v.push_back(make("HMMA.884.F16.TN", K::MatMul, L::Thread,
                     pat(1, 4, ElemType::F16, {RF}, Major::RowMajor),
                     pat(4, 1, ElemType::F16, {RF}, Major::ColMajor),
                     pat(1, 8, ElemType::F16, {RF}, Major::ColMajor), SimSemantics::OPAQUE));
    // sm_100a tensor-core leaves
    v.push_back(make("TMA_LOAD", K::Move, L::Block, pat(std::nullopt, std::nullopt, std::nullopt, {GL}),
                     {}, pat(std::nullopt, std::nullopt, std::nullopt, {SH}), SimSemantics::TMA_LOAD,
                     "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"));
    for (ElemType e : {ElemType::F16, ElemType::BF16})
        v.push_back(make(e == ElemType::F16 ? "UMMA.F16" : "UMMA.BF16", K::MatMul, L::Block,
                         pat(std::nullopt, std::nullopt, e, {SH}),
                         pat(std::nullopt, std::nullopt, e, {SH}),
                         pat(std::nullopt, std::nullopt, ElemType::F32, {TM}), SimSemantics::UMMA,
                         "tcgen05.mma.cta_group::{1|2}.kind::f16"));
    v.push_back(make("TMEM_ZERO", K::Move, L::Block, pat(std::nullopt, std::nullopt, std::nullopt, {TM}),
                     {}, pat(std::nullopt, std::nullopt, std::nullopt, {TM}), SimSemantics::TMEM_ZERO,
                     "first tcgen05.mma with enable-input-d = 0"));
    v.push_back(make("TMEM_STORE", K::Move, L::Warp, pat(32, std::nullopt, std::nullopt, {TM}), {},
                     pat(32, std::nullopt, std::nullopt, {GL}), SimSemantics::TMEM_STORE,
                     "tcgen05.ld.sync.aligned.32x32b + st.global"));
    return v;
}

}  // namespace

const std::vector<Instruction>& builtin_instructions() {
    static const std::vector<Instruction> set = build_builtins();
    return set;
}

bool spec_equal(const Spec& x, const Spec& y) {
    if (x.kind != y.kind || x.level != y.level) return false;
    auto same = [](const MatrixRef& p, const MatrixRef& q) {
        return p.rows == q.rows && p.cols == q.cols && p.elem == q.elem && p.mem == q.mem &&
               p.layout.major == q.layout.major;
    };
    if (x.is_matmul())
        return same(x.mm().a, y.mm().a) && same(x.mm().b, y.mm().b) && same(x.mm().c, y.mm().c);
    return same(x.mv().src, y.mv().src) && same(x.mv().dst, y.mv().dst);
}

bool MicroKernel::matches(const Spec& s) const { return spec_equal(pattern, s); }

void MicroKernelSet::register_kernel(MicroKernel mk) {
    for (const auto& k : kernels)
        if (spec_equal(k.pattern, mk.pattern))
            fail(ErrorKind::DuplicatePattern, "micro-kernels '" + k.name + "' and '" + mk.name +
                                                  "' share the pattern " + spec_short_form(mk.pattern));
    kernels.push_back(std::move(mk));
}

const MicroKernel* MicroKernelSet::find(const std::string& name) const {
    for (const auto& k : kernels)
        if (k.name == name) return &k;
    return nullptr;
}

std::string Match::name() const {
    if (micro_kernel) return micro_kernel->name;
    if (instruction) return instruction->name;
    return "";
}

Match match_executable(const Spec& s, const std::vector<Instruction>& instrs,
                       const MicroKernelSet& mks) {
    for (const auto& mk : mks.kernels)
        if (mk.matches(s)) return Match{nullptr, &mk};
    const Instruction* found = nullptr;
    for (const auto& ins : instrs) {
        if (!ins.matches(s)) continue;
        if (found)
            fail(ErrorKind::AmbiguousMatch, "built-ins '" + found->name + "' and '" + ins.name +
                                                "' both match " + spec_short_form(s));
        found = &ins;
    }
    return Match{found, nullptr};
}

Match match_executable(const Spec& s) {
    static const MicroKernelSet empty;
    return match_executable(s, builtin_instructions(), empty);
}

}  // namespace fireiron
