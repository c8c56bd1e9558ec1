// Decomposition trees (Fireiron strategies), spec transforms, leaf binding,
// validation with launch derivation, and elaboration traces. Semantics follow
// the reference (proj/include/anvil/decomp.hpp:17-770); the sm_100a
// refinements are additions:
//   tile ... .to block .pair   -> the block unit is a CTA pair (tcgen05 cta_group::2)
//   tile ... .to block .pair .multicast -> two neighbouring pair units (along N) form a
//                                 cluster and receive each A stage by one TMA multicast
//   split K .stages S          -> S-deep TMA/MMA mbarrier pipeline over the K loop
//   split K .splitk            -> the split's chunks run in parallel on the CTAs
//   split K .prefetchLoads / .doubleBufferLoop, load .. .doubleBuffer / .postponed
//                              -> the paper's pipelining refinements: the
//                                 deepest / a 2-stage TMA ring; postponed loads are what the
//                                 warp-specialised producer does. Scheduling only.
//                                 of a cluster; the following epilog reduces the
//                                 partial accumulators on chip (paper's splitK,
//                                 PAPER.md:67-127)
//   epilog tm                  -> accumulator in tensor memory
#pragma once

#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "fireiron/exec.hpp"
#include "fireiron/index_expr.hpp"
#include "fireiron/types.hpp"

namespace fireiron {

enum class Operand { A, B, Src };
const char* operand_name(Operand o);

struct TileRefinements {
    std::optional<ComputeLevel> to;
    bool unroll = false;
    std::optional<Major> layout;  // unit id -> tile coordinate order
    Expr swizzle;                 // over the free variable "id"
    bool pair = false;            // sm_100a: block unit = CTA pair
    bool multicast = false;       // sm_100a: two neighbouring block units along N share A by TMA multicast
};

struct LoadRefinements {
    bool no_sync = false;
    std::optional<Major> storage_layout;
    long pad = 0;
    std::optional<long> align;
    bool reuse_buffer = false;
    // paper appendix, scheduling only -- results are unchanged:
    bool double_buffer = false;   // .doubleBuffer: two staging buffers (sm_100a SH loads: a 2-stage TMA ring)
    bool postponed = false;       // .postponed: the next step's loads complete behind this step's MMA
                                  // (sm_100a: the TMA producer warp always runs ahead of the MMA warp)
};

struct SplitRefinements {
    bool unroll = false;
    bool sync = false;
    int stages = 0;        // sm_100a: pipeline depth (0 = default)
    bool splitk = false;   // sm_100a: parallel split with on-chip reduction
    // paper appendix, scheduling only:
    bool prefetch = false;       // .prefetchLoads: loads of later steps in flight (the deepest ring, stages 0)
    bool double_buffer = false;  // .doubleBufferLoop: two stages (normalised to stages = 2)
};

enum class NodeKind { Tile, Split, Load, Epilog, MmaTile, Done };

struct DecompNode;
using NodePtr = std::shared_ptr<DecompNode>;

struct DecompNode {
    NodeKind kind = NodeKind::Done;
    int src_line = 0;

    long tile_r = 0, tile_c = 0;  // Tile
    TileRefinements tile_ref;

    long split_k = 0;  // Split
    SplitRefinements split_ref;

    Operand operand = Operand::A;  // Load
    MemLevel target;
    NodePtr move_decomp;
    LoadRefinements load_ref;

    MemLevel acc_level;  // Epilog
    NodePtr init_decomp, store_decomp;

    std::string micro_kernel;  // Done: empty = match built-ins

    NodePtr child;
};

void check_tile_refinements(const TileRefinements& r);
void check_load_refinements(const LoadRefinements& r, const MemLevel& target, ElemType elem);

NodePtr n_done(std::string micro_kernel = "", int line = 0);
NodePtr n_tile(long r, long c, TileRefinements ref, NodePtr child, int line = 0);
NodePtr n_tile(long r, long c, NodePtr child);
NodePtr n_split(long k, SplitRefinements ref, NodePtr child, int line = 0);
NodePtr n_load(Operand op, MemLevel target, NodePtr move_decomp, LoadRefinements ref, NodePtr child,
               ElemType elem = ElemType::F32, int line = 0);
NodePtr n_epilog(MemLevel acc, NodePtr init_decomp, NodePtr store_decomp, NodePtr child,
                 int line = 0);
NodePtr n_mma_tile(NodePtr child, int line = 0);

// --- spec transforms, one per decomposition rule ---------------------------
Spec after_tile(const Spec& s, long r, long c);
Spec after_to(const Spec& s, ComputeLevel level);
Spec after_split(const Spec& s, long k_block);
const MatrixRef& operand_ref(const Spec& s, Operand op);
MatrixRef& operand_ref(Spec& s, Operand op);
Spec after_load(const Spec& s, Operand op, MemLevel target, Layout dst_layout = Layout::col_major());
Spec induced_move_spec(const Spec& s, Operand op, MemLevel target,
                       Layout dst_layout = Layout::col_major());
Spec after_epilog(const Spec& s, MemLevel acc);
Spec induced_init_move(const Spec& s, MemLevel acc);
Spec induced_store_move(const Spec& s, MemLevel acc);
Spec hmma_residual_spec();
Spec after_mma_tile(const Spec& s);

ResidualBinding bind_done(const Spec& residual, const std::string& mk_name,
                          const MicroKernelSet& mks,
                          const std::vector<Instruction>& instrs = builtin_instructions());

// --- validation ------------------------------------------------------------
struct Violation {
    ErrorKind kind;
    int step = 0;  // preorder node index
    int line = 0;  // script line when known
    std::string message;
};

struct LaunchConfig {
    long grid_x = 1, grid_y = 1;
    long warps_per_block = 1;
    long block_threads = 1;
};

struct ValidationReport {
    std::vector<Violation> violations;
    LaunchConfig launch;
    long shared_bytes = 0;
    bool ok() const { return violations.empty(); }
    std::string to_string() const;
};

ValidationReport validate(const Spec& root, const NodePtr& tree,
                          const MicroKernelSet& mks = MicroKernelSet{});

// --- elaboration -----------------------------------------------------------
struct TraceEntry {
    std::string label;
    Spec spec;
    std::vector<std::pair<std::string, std::vector<TraceEntry>>> subs;
};

std::vector<TraceEntry> elaborate(const Spec& root, const NodePtr& tree,
                                  const MicroKernelSet& mks = MicroKernelSet{});
void render_trace(const std::vector<TraceEntry>& trace, std::string& out, int indent,
                  bool with_subs);
std::string render_trace(const std::vector<TraceEntry>& trace, bool with_subs = false);

// Deep copy of a tree (trees are mutable shared structures).
NodePtr clone_tree(const NodePtr& n);

}  // namespace fireiron
