// Lowered kernel program: buffer plan + statement list with symbolic index
// expressions. Same lowering rules as the reference
// (proj/include/anvil/program.hpp:17-693) -- thread mapping (unit_coords),
// K-chunk loops, staging buffers with barriers, epilog init/compute/store,
// reuseBuffer aliasing and the shared-byte plan -- plus the sm_100a leaf
// statements (TMA tile loads, UMMA, TMEM zero/store) and pipelined loops.
#pragma once

#include <string>
#include <variant>
#include <vector>

#include "fireiron/decomp.hpp"

namespace fireiron {

enum class BufferRole { RootA, RootB, RootC, RootSrc, RootDst, OperandA, OperandB, Accum, Staging };

struct BufferDecl {
    int id = -1;
    std::string name;
    MemLevel mem;
    ElemType elem = ElemType::F32;
    long rows = 0, cols = 0;
    Layout layout;
    long align_bytes = 4;
    ComputeLevel home = ComputeLevel::Kernel;
    BufferRole role = BufferRole::Staging;
    bool is_root = false;
    bool reuse_requested = false;
    int alias_of = -1;
    long local_rows = 0, local_cols = 0;

    long row_stride() const { return layout.row_stride(rows, cols); }
    long col_stride() const { return layout.col_stride(rows, cols); }
    long extent() const { return layout.extent(rows, cols); }
    long local_row_stride() const { return layout.major == Major::RowMajor ? local_cols : 1; }
    long local_col_stride() const { return layout.major == Major::ColMajor ? local_rows : 1; }
    long local_extent() const { return local_rows * local_cols; }
    bool distributed_rf() const {
        return !is_root && mem.kind == MemKind::RF && home < ComputeLevel::Thread;
    }
    bool is_fragment() const { return !is_root && mem.kind == MemKind::FR; }
};

struct BufferPlan {
    std::vector<BufferDecl> buffers;
    long shared_bytes = 0;
    const BufferDecl& at(int id) const { return buffers[static_cast<size_t>(id)]; }
    int storage_root(int id) const;
};

struct ElemRef {
    int buf = -1;
    Expr row, col;    // logical coordinates in the buffer
    Expr lrow, lcol;  // per-owning-unit coordinates (distributed buffers)
};
struct FragRef {
    int buf = -1;
    Expr row, col;
    Expr lrow, lcol;
};

struct Stmt;
using StmtList = std::vector<Stmt>;

struct LoopStmt {
    std::string var;
    long count = 0;
    StmtList body;
    int stages = 0;         // sm_100a pipelined K loop (split .stages)
    bool splitk = false;    // sm_100a parallel split across cluster CTAs
};
struct BarrierStmt {};
struct CopyStmt { ElemRef dst, src; };
struct ZeroStmt { ElemRef dst; };
struct FmaStmt { ElemRef c, a, b; };
struct WmmaFillStmt { FragRef frag; };
struct WmmaLoadStmt { FragRef frag; ElemRef src; };
struct WmmaStoreStmt { ElemRef dst; FragRef frag; };
struct WmmaMmaStmt { FragRef c, a, b; };
struct MicroKernelStmt {
    const MicroKernel* mk = nullptr;
    std::vector<std::pair<std::string, ElemRef>> operands;
    long m = 0, n = 0, k = 0;
};
struct HmmaStmt { ElemRef a, b, c; };
// sm_100a leaves: whole-tile statements at Block / Warp level
struct TmaLoadStmt { ElemRef dst, src; long rows = 0, cols = 0; };
struct UmmaStmt { ElemRef c, a, b; long m = 0, n = 0, k = 0; };
struct TmemZeroStmt { ElemRef dst; long rows = 0, cols = 0; };
struct TmemStoreStmt { ElemRef dst, src; long rows = 0, cols = 0; };

struct Stmt {
    std::variant<LoopStmt, BarrierStmt, CopyStmt, ZeroStmt, FmaStmt, WmmaFillStmt, WmmaLoadStmt,
                 WmmaStoreStmt, WmmaMmaStmt, MicroKernelStmt, HmmaStmt, TmaLoadStmt, UmmaStmt,
                 TmemZeroStmt, TmemStoreStmt>
        v;
};

struct Program {
    Spec root;
    LaunchConfig launch;
    BufferPlan plan;
    StmtList body;
    std::string entry_name;
    bool simulatable = true;  // false once a micro-kernel / opaque / sm100 leaf is bound
    bool uses_wmma = false;
    bool uses_tcgen05 = false;  // sm_100a tensor-core leaves present
    bool uses_micro_kernel = false;
    bool uses_hmma = false;
    NodePtr tree;  // snapshot of the lowered strategy (the tcgen05 planner reads it)
};

int count_barriers(const StmtList& body);

Program lower(const Spec& root, const NodePtr& tree, const MicroKernelSet& mks = MicroKernelSet{});
ValidationReport validate_with_plan(const Spec& root, const NodePtr& tree,
                                    const MicroKernelSet& mks = MicroKernelSet{});

}  // namespace fireiron
