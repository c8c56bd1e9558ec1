// Executable leaves: built-in instructions and user micro-kernels, and the
// residual-spec matcher. Same matching rules as the reference
// (proj/include/anvil/exec.hpp:20-237): micro-kernels take precedence, two
// matching built-ins are AmbiguousMatch, duplicate micro-kernel patterns are
// rejected at registration.
//
// The built-in set keeps the reference's seven leaves (FMA, HFMA, COPY,
// WMMA_MMA, WMMA_LOAD, WMMA_STORE, HMMA.884.F16.TN) and adds the sm_100a
// leaves the tensor-core strategies bind:
//   TMA_LOAD     Move(_x_)(GL->SH)(Block)           cp.async.bulk.tensor + mbarrier
//   UMMA.F16     MatMul(_,_,_)(SH,SH,TM)(Block) f16  tcgen05.mma kind::f16
//   UMMA.BF16    MatMul(_,_,_)(SH,SH,TM)(Block) bf16
//   TMEM_ZERO    Move(_x_)(TM->TM)(Block)            accumulate=0 on the first MMA
//   TMEM_STORE   Move(32x_)(TM->GL)(Warp)            tcgen05.ld 32x32b + st.global
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "fireiron/types.hpp"

namespace fireiron {

enum class SimSemantics {
    FMA,
    WMMA_MMA,
    WMMA_LOAD,
    WMMA_STORE,
    OPAQUE,
    // sm_100a tensor-core leaves (executed only by the tcgen05 kernel family)
    TMA_LOAD,
    UMMA,
    TMEM_ZERO,
    TMEM_STORE,
};

// One operand slot; unset fields are wildcards, mems is a set (empty = any).
struct OperandPattern {
    std::optional<long> rows, cols;
    std::optional<ElemType> elem;
    std::vector<MemKind> mems;
    std::optional<Major> major;

    bool matches(const MatrixRef& m) const;
};

struct Instruction {
    std::string name;
    Spec::Kind kind = Spec::Kind::MatMul;
    ComputeLevel level = ComputeLevel::Thread;
    OperandPattern a, b, c;  // MatMul: a,b,c; Move: a = src, c = dst
    std::string emission;
    SimSemantics sim = SimSemantics::FMA;

    bool matches(const Spec& s) const;
    std::string pattern_short_form() const;
    bool is_tensor_core_sm100() const;
};

const std::vector<Instruction>& builtin_instructions();

struct MicroKernel {
    std::string name;
    Spec pattern;
    std::string body;
    std::vector<std::string> declared_vars;

    bool matches(const Spec& s) const;
};

bool spec_equal(const Spec& x, const Spec& y);

struct MicroKernelSet {
    std::vector<MicroKernel> kernels;
    void register_kernel(MicroKernel mk);
    const MicroKernel* find(const std::string& name) const;
};

struct Match {
    const Instruction* instruction = nullptr;
    const MicroKernel* micro_kernel = nullptr;
    explicit operator bool() const { return instruction || micro_kernel; }
    std::string name() const;
};

Match match_executable(const Spec& s, const std::vector<Instruction>& instrs,
                       const MicroKernelSet& mks);
Match match_executable(const Spec& s);

struct ResidualBinding {
    Spec residual;
    Match match;
};

}  // namespace fireiron
