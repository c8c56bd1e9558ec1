// Spec core: element types, memory / compute hierarchies, layouts and the
// MatMul / Move specs every decomposition transforms. API-compatible with the
// reference (proj/include/anvil/types.hpp:15-226), extended for sm_100a:
//   ElemType::BF16          (the reference only knows F32/F16, types.hpp:15)
//   MemKind::TM             (tensor memory: tcgen05 accumulators)
//   kSharedMemoryBudgetSm100 (227 KiB opt-in per CTA, vs the 48 KiB default)
#pragma once

#include <string>
#include <variant>

#include "fireiron/error.hpp"

namespace fireiron {

enum class ElemType { F32, F16, BF16 };

int bit_width(ElemType t);
int byte_width(ElemType t);
const char* elem_name(ElemType t);     // "f32" | "f16" | "bf16"
const char* elem_c_type(ElemType t);   // "float" | "__half" | "__nv_bfloat16"

// GL > SH > { RF, FR, TM }. Loads move data strictly downward in rank.
enum class MemKind { GL, SH, RF, FR, TM };

struct MemLevel {
    MemKind kind = MemKind::GL;
    int fr_m = 16, fr_n = 16, fr_k = 16;  // fragment geometry (FR only)

    static MemLevel gl() { return {MemKind::GL}; }
    static MemLevel sh() { return {MemKind::SH}; }
    static MemLevel rf() { return {MemKind::RF}; }
    static MemLevel fr(int m = 16, int n = 16, int k = 16) { return {MemKind::FR, m, n, k}; }
    static MemLevel tm() { return {MemKind::TM}; }

    bool operator==(const MemLevel& o) const;
    bool operator!=(const MemLevel& o) const { return !(*this == o); }
};

int mem_rank(MemKind k);
std::string mem_name(const MemLevel& m);

// Total order Kernel > Block > Warp > Thread (decomposition paths descend).
enum class ComputeLevel { Kernel = 0, Block = 1, Warp = 2, Thread = 3 };
const char* level_name(ComputeLevel l);

constexpr int kWarpWidth = 32;
constexpr long kSharedMemoryBudget = 48 * 1024;         // reference default (types.hpp:87)
constexpr long kSharedMemoryBudgetSm100 = 227 * 1024;   // B200 opt-in per CTA
constexpr int kTmemColumns = 512;                       // 128 lanes x 512 x 32-bit per SM

enum class Major { RowMajor, ColMajor };
const char* major_name(Major m);

struct Layout {
    Major major = Major::ColMajor;
    long pad_cols = 0;  // extra elements appended to the minor dimension

    static Layout row_major(long pad = 0) { return {Major::RowMajor, pad}; }
    static Layout col_major(long pad = 0) { return {Major::ColMajor, pad}; }

    long row_stride(long rows, long cols) const;
    long col_stride(long rows, long cols) const;
    long extent(long rows, long cols) const;
    // physical leading dimension (stride of the major dimension)
    long leading_dim(long rows, long cols) const;
    bool operator==(const Layout& o) const { return major == o.major && pad_cols == o.pad_cols; }
};

struct MatrixRef {
    std::string name;
    long rows = 0, cols = 0;
    ElemType elem = ElemType::F32;
    MemLevel mem = MemLevel::gl();
    Layout layout = Layout::col_major();
};

MatrixRef make_matrix(std::string name, long rows, long cols, ElemType elem, MemLevel mem,
                      Layout layout);

struct MatMulOp {
    MatrixRef a, b, c;
};
struct MoveOp {
    MatrixRef src, dst;
};

// The computation left to implement: operation, operands and the compute level
// responsible for it.
struct Spec {
    enum class Kind { MatMul, Move };
    Kind kind = Kind::MatMul;
    ComputeLevel level = ComputeLevel::Kernel;
    std::variant<MatMulOp, MoveOp> op;
    bool accumulate = false;  // set by epilog: the residual computes C += A*B

    const MatMulOp& mm() const { return std::get<MatMulOp>(op); }
    MatMulOp& mm() { return std::get<MatMulOp>(op); }
    const MoveOp& mv() const { return std::get<MoveOp>(op); }
    MoveOp& mv() { return std::get<MoveOp>(op); }
    bool is_matmul() const { return kind == Kind::MatMul; }
    bool is_move() const { return kind == Kind::Move; }
    long m() const { return is_matmul() ? mm().c.rows : mv().dst.rows; }
    long n() const { return is_matmul() ? mm().c.cols : mv().dst.cols; }
    long k() const { return is_matmul() ? mm().a.cols : 1; }
};

struct ElemTriple {
    ElemType a = ElemType::F32, b = ElemType::F32, c = ElemType::F32;
};
struct MemTriple {
    MemLevel a, b, c;
};
struct LayoutTriple {
    Layout a, b, c;
};

Spec make_matmul_spec(long m, long n, long k, ElemTriple elems, MemTriple mems,
                      LayoutTriple layouts, ComputeLevel level);
Spec make_move_spec(MatrixRef src, MatrixRef dst, ComputeLevel level);

// MatMul(M,N,K)(memA,memB,memC)(Level) or Move(RxC)(memSrc->memDst)(Level)
std::string spec_short_form(const Spec& s);

}  // namespace fireiron
