// sm_100a code generation (the re-targeted anvil::generate seam,
// proj/include/anvil/codegen.hpp:18-298).
//
// Generic trees are emitted statement by statement from the Program; the
// emitted TU is self-contained CUDA for NVRTC (--gpu-architecture=sm_100a
// --fmad=false). Differences from the reference's Volta-era text, all needed
// to compile and to reproduce the simulator's numerics:
//   * every root is a kernel pointer parameter (the simulator ingests inputs
//     into roots whatever their declared level, sim.hpp:462-474);
//   * elements load as fp32 and store with round-to-nearest into the buffer
//     type (__half / __nv_bfloat16), as the simulator's store() does;
//   * the FMA leaf is `c = c + a*b` with contraction disabled (FMUL + FADD),
//     bit-exact with the simulator's unfused fp32 (sim.hpp:370-376);
//   * shared buffers live in one dynamic allocation (up to 227 KiB);
//   * WMMA fragments take their layout from the buffer they are loaded from.
// Tensor-core trees are recognised (match_tc_strategy) and emitted as a
// parameterised instantiation of the hand-written tcgen05 kernel family.
#include <algorithm>
#include <map>
#include <set>
#include <sstream>

#include "fireiron/backend.hpp"

namespace fireiron {

namespace {

const char* storage_type(ElemType e) { return elem_c_type(e); }

struct Emitter {
    const Program& prog;
    std::string out;
    int indent = 0;
    std::map<int, Major> frag_major;  // WMMA matrix_a/b fragment layout by buffer
    std::map<int, long> sh_offset;    // storage root -> byte offset in dynamic smem
    long sh_bytes = 0;

    explicit Emitter(const Program& p) : prog(p) {}

    void line(const std::string& s) {
        if (!s.empty()) out.append(static_cast<size_t>(indent) * 2, ' ');
        out += s;
        out += '\n';
    }
    const BufferDecl& buf(int id) const { return prog.plan.at(id); }
    std::string storage_name(int id) const { return buf(prog.plan.storage_root(id)).name; }

    std::string offset_text(const ElemRef& r) const {
        const BufferDecl& b = buf(r.buf);
        Expr row = r.row, col = r.col;
        long rs = b.row_stride(), cs = b.col_stride();
        if (b.distributed_rf()) {
            row = r.lrow;
            col = r.lcol;
            rs = b.local_row_stride();
            cs = b.local_col_stride();
        }
        return emit_c(simplify(iadd(imul(row, iconst(rs)), imul(col, iconst(cs)))));
    }
    // every shared buffer, aliases included, is a pointer of its own element
    // type into its storage root (sim.hpp:314-320 indexes an alias by element
    // in its own geometry; its stores round by its own type, sim.hpp:336-339)
    std::string ref_text(const ElemRef& r) const { return buf(r.buf).name + "[" + offset_text(r) + "]"; }
    std::string load_text(const ElemRef& r) const { return "fi_ld(" + ref_text(r) + ")"; }
    std::string store_text(const ElemRef& r, const std::string& value) const {
        return ref_text(r) + " = fi_st<" + std::string(storage_type(buf(r.buf).elem)) + ">(" + value + ");";
    }

    std::string frag_text(const FragRef& f) const {
        const BufferDecl& b = buf(f.buf);
        const long tiles_n = std::max<long>(1, b.local_cols / 16);
        Expr idx = iadd(imul(idiv(f.lrow, iconst(16)), iconst(tiles_n)), idiv(f.lcol, iconst(16)));
        return b.name + "[" + emit_c(simplify(idx)) + "]";
    }

    void scan_fragments(const StmtList& body) {
        for (const auto& s : body) {
            if (const auto* l = std::get_if<LoopStmt>(&s.v)) scan_fragments(l->body);
            if (const auto* w = std::get_if<WmmaLoadStmt>(&s.v)) {
                const Major src = buf(w->src.buf).layout.major;
                auto it = frag_major.find(w->frag.buf);
                if (it != frag_major.end() && it->second != src)
                    throw BackendError(103, "fragment " + buf(w->frag.buf).name +
                                                " is loaded from buffers of different layouts");
                frag_major[w->frag.buf] = src;
            }
        }
    }

    void stmt(const Stmt& s) {
        if (const auto* l = std::get_if<LoopStmt>(&s.v)) {
            line("for (int " + l->var + " = 0; " + l->var + " < " + std::to_string(l->count) + "; ++" +
                 l->var + ") {");
            ++indent;
            for (const auto& inner : l->body) stmt(inner);
            --indent;
            line("}");
            return;
        }
        if (std::holds_alternative<BarrierStmt>(s.v)) return line("__syncthreads();");
        if (const auto* c = std::get_if<CopyStmt>(&s.v)) return line(store_text(c->dst, load_text(c->src)));
        if (const auto* z = std::get_if<ZeroStmt>(&s.v)) return line(store_text(z->dst, "0.0f"));
        if (const auto* f = std::get_if<FmaStmt>(&s.v))
            return line(store_text(f->c, "fi_fma_unfused(" + load_text(f->c) + ", " + load_text(f->a) +
                                             ", " + load_text(f->b) + ")"));
        if (const auto* w = std::get_if<WmmaFillStmt>(&s.v))
            return line("wmma::fill_fragment(" + frag_text(w->frag) + ", 0.0f);");
        if (const auto* w = std::get_if<WmmaLoadStmt>(&s.v)) {
            const BufferDecl& src = buf(w->src.buf);
            const long ld = src.layout.major == Major::RowMajor ? src.row_stride() : src.col_stride();
            const BufferDecl& dst = buf(w->frag.buf);
            if (dst.role == BufferRole::OperandA || dst.role == BufferRole::OperandB)
                return line("wmma::load_matrix_sync(" + frag_text(w->frag) + ", &" + ref_text(w->src) + ", " +
                            std::to_string(ld) + ");");
            const char* mem = src.layout.major == Major::RowMajor ? "wmma::mem_row_major" : "wmma::mem_col_major";
            return line("wmma::load_matrix_sync(" + frag_text(w->frag) + ", &" + ref_text(w->src) + ", " +
                        std::to_string(ld) + ", " + mem + ");");
        }
        if (const auto* w = std::get_if<WmmaStoreStmt>(&s.v)) {
            const BufferDecl& dst = buf(w->dst.buf);
            const long ld = dst.layout.major == Major::RowMajor ? dst.row_stride() : dst.col_stride();
            const char* mem = dst.layout.major == Major::RowMajor ? "wmma::mem_row_major" : "wmma::mem_col_major";
            return line("wmma::store_matrix_sync(&" + ref_text(w->dst) + ", " + frag_text(w->frag) + ", " +
                        std::to_string(ld) + ", " + mem + ");");
        }
        if (const auto* w = std::get_if<WmmaMmaStmt>(&s.v)) {
            const std::string c = frag_text(w->c);
            return line("wmma::mma_sync(" + c + ", " + frag_text(w->a) + ", " + frag_text(w->b) + ", " + c + ");");
        }
        if (const auto* m = std::get_if<MicroKernelStmt>(&s.v)) return micro_kernel(*m);
        if (const auto* h = std::get_if<HmmaStmt>(&s.v)) {
            line("// HMMA.884.F16.TN (Volta quad-pair leaf): emitted for inspection only");
            line("asm volatile(\"mma.sync.aligned.m8n8k4.row.col.f16.f16.f16.f16 {%0,%1,%2,%3}, {%4,%5}, {%6,%7}, {%0,%1,%2,%3};\"");
            line("    : \"+r\"(((unsigned*)&" + ref_text(h->c) + ")[0]), \"+r\"(((unsigned*)&" + ref_text(h->c) +
                 ")[1]), \"+r\"(((unsigned*)&" + ref_text(h->c) + ")[2]), \"+r\"(((unsigned*)&" + ref_text(h->c) + ")[3])");
            line("    : \"r\"(((const unsigned*)&" + ref_text(h->a) + ")[0]), \"r\"(((const unsigned*)&" +
                 ref_text(h->a) + ")[1]), \"r\"(((const unsigned*)&" + ref_text(h->b) + ")[0]), \"r\"(((const unsigned*)&" +
                 ref_text(h->b) + ")[1]));");
            return;
        }
        // sm_100a leaves have no per-statement form: the tcgen05 family implements them
        if (std::holds_alternative<TmaLoadStmt>(s.v) || std::holds_alternative<UmmaStmt>(s.v) ||
            std::holds_alternative<TmemZeroStmt>(s.v) || std::holds_alternative<TmemStoreStmt>(s.v))
            throw BackendError(103, "tensor-core leaves are emitted through the tcgen05 kernel family");
    }

    void micro_kernel(const MicroKernelStmt& m) {  // codegen.hpp:128-174 substitution rules
        std::string body = m.mk->body;
        auto replace_all = [&body](const std::string& from, const std::string& to) {
            for (size_t p = 0; (p = body.find(from, p)) != std::string::npos; p += to.size())
                body.replace(p, from.size(), to);
        };
        for (const std::string& var : m.mk->declared_vars) {
            std::string value;
            if (var == "M") value = std::to_string(m.m);
            else if (var == "N") value = std::to_string(m.n);
            else if (var == "K") value = std::to_string(m.k);
            else {
                std::string base = var, field;
                if (auto dot = var.find('.'); dot != std::string::npos) {
                    base = var.substr(0, dot);
                    field = var.substr(dot + 1);
                }
                const ElemRef* r = nullptr;
                for (const auto& [name, er] : m.operands)
                    if (name == base) r = &er;
                if (!r) continue;
                const BufferDecl& b = buf(r->buf);
                const bool local = b.distributed_rf();
                if (field.empty()) value = ref_text(*r);
                else if (field == "base") value = b.name;
                else if (field == "off") value = offset_text(*r);
                else if (field == "rs") value = std::to_string(local ? b.local_row_stride() : b.row_stride());
                else if (field == "cs") value = std::to_string(local ? b.local_col_stride() : b.col_stride());
                else continue;
            }
            replace_all("{" + var + "}", value);
        }
        line("{");
        ++indent;
        for (size_t start = 0; start < body.size();) {
            size_t end = body.find('\n', start);
            if (end == std::string::npos) end = body.size();
            const std::string ln = body.substr(start, end - start);
            if (!ln.empty()) line(ln);
            start = end + 1;
        }
        --indent;
        line("}");
    }

    void declarations() {
        // shared storage roots: one dynamic allocation, each root aligned
        for (const auto& b : prog.plan.buffers) {
            if (b.is_root || b.mem.kind != MemKind::SH || b.alias_of >= 0) continue;
            long bytes = 0, align = 16;
            for (const auto& m : prog.plan.buffers)
                if (m.mem.kind == MemKind::SH && !m.is_root && prog.plan.storage_root(m.id) == b.id) {
                    bytes = std::max(bytes, m.extent() * byte_width(m.elem));
                    align = std::max(align, m.align_bytes);
                }
            sh_bytes = (sh_bytes + align - 1) / align * align;
            sh_offset[b.id] = sh_bytes;
            sh_bytes += bytes;
        }
        if (!sh_offset.empty()) line("extern __shared__ __align__(128) unsigned char fi_smem[];");
        for (const auto& b : prog.plan.buffers) {
            if (b.is_root) continue;
            const std::string t = storage_type(b.elem);
            switch (b.mem.kind) {
                case MemKind::SH:
                    if (b.alias_of >= 0)
                        line("// " + b.name + " aliases " + storage_name(b.id) + " (reuseBuffer)");
                    line(t + "* const " + b.name + " = reinterpret_cast<" + t + "*>(fi_smem + " +
                         std::to_string(sh_offset[prog.plan.storage_root(b.id)]) + ");");
                    break;
                case MemKind::RF:
                    line(t + " " + b.name + "[" + std::to_string(b.distributed_rf() ? b.local_extent() : b.extent()) +
                         "];");
                    break;
                case MemKind::FR: {
                    const long count = std::max<long>(1, (b.local_rows / 16) * (b.local_cols / 16));
                    std::string kind;
                    if (b.role == BufferRole::OperandA || b.role == BufferRole::OperandB) {
                        if (b.elem != ElemType::F16)
                            throw BackendError(103, "WMMA operand fragments must be f16");
                        const Major mj = frag_major.count(b.id) ? frag_major[b.id] : b.layout.major;
                        kind = std::string(b.role == BufferRole::OperandA ? "wmma::matrix_a" : "wmma::matrix_b") +
                               ", 16, 16, 16, __half, " +
                               (mj == Major::RowMajor ? "wmma::row_major" : "wmma::col_major");
                    } else {
                        kind = std::string("wmma::accumulator, 16, 16, 16, ") +
                               (b.elem == ElemType::F16 ? "__half" : "float");
                    }
                    line("wmma::fragment<" + kind + "> " + b.name + "[" + std::to_string(count) + "];");
                    break;
                }
                default: throw BackendError(103, "buffer " + b.name + " in " + mem_name(b.mem) + " has no generic lowering");
            }
        }
    }

    std::string params() const {
        std::string p;
        for (const auto& b : prog.plan.buffers) {
            if (!b.is_root) continue;
            const bool out_param = b.role == BufferRole::RootC || b.role == BufferRole::RootDst;
            if (!p.empty()) p += ", ";
            p += std::string(out_param ? "" : "const ") + storage_type(b.elem) + "* __restrict__ " + b.name;
        }
        return p;
    }

    std::string run() {
        scan_fragments(prog.body);
        line("// " + spec_short_form(prog.root));
        line("// grid " + std::to_string(prog.launch.grid_x) + "x" + std::to_string(prog.launch.grid_y) + ", " +
             std::to_string(prog.launch.block_threads) + " threads per block; sm_100a, compile with --fmad=false");
        line("#include <cuda_fp16.h>");
        line("#include <cuda_bf16.h>");
        if (prog.uses_wmma) {
            line("#include <mma.h>");
            line("using namespace nvcuda;");
        }
        line("");
        line("__device__ __forceinline__ float fi_ld(float v) { return v; }");
        line("__device__ __forceinline__ float fi_ld(__half v) { return __half2float(v); }");
        line("__device__ __forceinline__ float fi_ld(__nv_bfloat16 v) { return __bfloat162float(v); }");
        line("template <typename T> __device__ __forceinline__ T fi_st(float v);");
        line("template <> __device__ __forceinline__ float fi_st<float>(float v) { return v; }");
        line("// round_to_f16 saturates at +-65504 above 2^16 (anvil matrix.hpp:76)");
        line("template <> __device__ __forceinline__ __half fi_st<__half>(float v) {");
        line("  return __float2half_rn(fabsf(v) >= 65536.0f && fabsf(v) <= 3.40282347e38f ? copysignf(65504.0f, v) : v);");
        line("}");
        line("template <> __device__ __forceinline__ __nv_bfloat16 fi_st<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }");
        line("// the FMA leaf: product and sum each rounded to fp32 (sim.hpp:370-376)");
        line("__device__ __forceinline__ float fi_fma_unfused(float c, float a, float b) {");
        line("  return __fadd_rn(c, __fmul_rn(a, b));");
        line("}");
        line("");
        line("extern \"C\" __global__ void __launch_bounds__(" + std::to_string(std::max<long>(1, prog.launch.block_threads)) +
             ") " + prog.entry_name + "(" + params() + ") {");
        ++indent;
        if (prog.root.is_matmul())
            line("constexpr int M = " + std::to_string(prog.root.m()) + ", N = " + std::to_string(prog.root.n()) +
                 ", K = " + std::to_string(prog.root.k()) + ";");
        else
            line("constexpr int R = " + std::to_string(prog.root.mv().src.rows) + ", C = " +
                 std::to_string(prog.root.mv().src.cols) + ";");
        declarations();
        line("");
        for (const auto& s : prog.body) stmt(s);
        --indent;
        line("}");
        return out;
    }
};

// Follows `c` through the chain; returns nodes in order.
std::vector<const DecompNode*> chain_nodes(const NodePtr& n) {
    std::vector<const DecompNode*> v;
    for (const DecompNode* p = n.get(); p; p = p->child.get()) v.push_back(p);
    return v;
}

}  // namespace

long generic_shared_bytes(const Program& prog);

KernelSource generate(const Program& prog) {
    KernelSource ks;
    ks.launch = prog.launch;
    ks.plan = prog.plan;
    ks.entry_name = prog.entry_name;
    if (prog.uses_tcgen05) {
        TcStrategy tc = match_tc_strategy(prog.root, prog.tree);
        if (!tc.matched) throw BackendError(103, "tensor-core tree has no sm_100a lowering: " + tc.why_not);
        const auto& mm = prog.root.mm();
        std::ostringstream o;
        o << "// " << spec_short_form(prog.root) << "\n"
          << "// tcgen05 strategy: block tile " << tc.tile_m << "x" << tc.tile_n << " (cta_group::" << tc.cta_group
          << "), K block " << tc.tile_k << ", split-K " << tc.split_k << ", stages "
          << (tc.stages ? std::to_string(tc.stages) : std::string("max")) << "\n"
          << "// warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7 epilogue (TMEM->RF->GL)\n"
          << "#include \"sm100/gemm_kernel.cuh\"\n\n"
          << "namespace fi_generated {\n"
          << "using namespace fireiron::sm100;\n"
          << "constexpr int kCtaGroup = " << tc.cta_group << ", kMmaN = " << (tc.tile_n == 512 ? 256 : tc.tile_n)
          << ", kSplitK = " << tc.split_k
          << ", kSlabs = " << tc.tile_m / (128 * tc.cta_group) << ", kNHalves = " << (tc.tile_n == 512 ? 2 : 1)
          << ", kMcast = " << tc.mcast << ";\n"
          << "using Shape = GemmShape<kCtaGroup, kMmaN, kSplitK, kSlabs, kNHalves>;\n"
          << "// grid: one persistent CTA per SM (clusters of kCtaGroup*kSplitK), "
          << "dynamic smem Shape::SMEM_BYTES\n"
          << "inline GemmArgs " << prog.entry_name << "_args(void* C) {\n"
          << "  GemmArgs a;\n"
          << "  a.C = C;\n"
          << "  a.M = " << prog.root.m() << "; a.N = " << prog.root.n() << "; a.K = " << prog.root.k() << ";\n"
          << "  a.ldc = " << mm.c.layout.leading_dim(mm.c.rows, mm.c.cols) << ";\n"
          << "  a.tiles_m = " << prog.root.m() / tc.tile_m << "; a.tiles_n = " << prog.root.n() / (tc.tile_n * tc.mcast)
          << ";\n"
          << "  a.k_blocks = " << prog.root.k() / tc.tile_k / tc.split_k << ";\n"
          << "  a.ab_format = " << (mm.a.elem == ElemType::BF16 ? 1 : 0) << ";  // " << elem_name(mm.a.elem) << "\n"
          << "  a.a_mn_major = " << (mm.a.layout.major == Major::ColMajor ? 1 : 0) << ";\n"
          << "  a.b_mn_major = " << (mm.b.layout.major == Major::RowMajor ? 1 : 0) << ";\n"
          << "  a.c_row_major = " << (mm.c.layout.major == Major::RowMajor ? 1 : 0) << ";\n"
          << "  a.out_type = " << (mm.c.elem == ElemType::F32 ? 0 : mm.c.elem == ElemType::F16 ? 1 : 2) << ";\n"
          << "  return a;\n"
          << "}\n"
          << "__global__ void __launch_bounds__(256, 1) " << prog.entry_name
          << "(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,\n"
          << "    const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,\n"
          << "    const __grid_constant__ CUtensorMap tmC2,\n"
          << "    const __grid_constant__ GemmArgs args) {\n"
          << "  fi_sm100_gemm_body<kCtaGroup, kMmaN, kSplitK, kSlabs, kNHalves, kMcast>(tmA, tmB, tmB2, tmC, tmC2, args);\n"
          << "}\n"
          << "}  // namespace fi_generated\n";
        ks.source = o.str();
        return ks;
    }
    if (generic_shared_bytes(prog) > kSharedMemoryBudgetSm100)
        fail(ErrorKind::CapacityExceeded, "plan needs " + std::to_string(generic_shared_bytes(prog)) +
                                              " shared bytes per block; the sm_100a budget is " +
                                              std::to_string(kSharedMemoryBudgetSm100));
    Emitter em(prog);
    ks.source = em.run();
    return ks;
}

KernelSource generate(const Spec& root, const NodePtr& tree, const MicroKernelSet& mks) {
    return generate(lower(root, tree, mks));
}

// Bytes of the generic kernel's dynamic shared allocation (storage roots,
// aligned), as laid out by the emitter.
long generic_shared_bytes(const Program& prog) {
    long total = 0;
    for (const auto& b : prog.plan.buffers) {
        if (b.is_root || b.mem.kind != MemKind::SH || b.alias_of >= 0) continue;
        long bytes = 0, align = 16;
        for (const auto& m : prog.plan.buffers)
            if (m.mem.kind == MemKind::SH && !m.is_root && prog.plan.storage_root(m.id) == b.id) {
                bytes = std::max(bytes, m.extent() * byte_width(m.elem));
                align = std::max(align, m.align_bytes);
            }
        total = (total + align - 1) / align * align + bytes;
    }
    return total;
}

// ---------------------------------------------------------------- tcgen05 recognizer
// The canonical sm_100a strategy (see fireiron/decomp.hpp):
//   tile BM BN .to block [.pair] [.swizzle e] [.layout l]
//   [split KC .splitk]
//   epilog tm { init { done } store { tile 32 BN .to warp ; done } }
//   split 64 [.stages S]
//   load a sh { done }   load b sh { done }      (either order)
//   done                                          -> UMMA.F16 | UMMA.BF16
TcStrategy match_tc_strategy(const Spec& root, const NodePtr& tree, const MicroKernelSet& mks) {
    TcStrategy tc;
    auto reject = [&](const std::string& why) {
        tc.matched = false;
        tc.why_not = why;
        return tc;
    };
    if (!root.is_matmul() || root.level != ComputeLevel::Kernel) return reject("root must be a Kernel-level MatMul");
    const auto& mm = root.mm();
    if (mm.a.mem.kind != MemKind::GL || mm.b.mem.kind != MemKind::GL || mm.c.mem.kind != MemKind::GL)
        return reject("operands must start in GL");
    if (mm.a.elem != mm.b.elem || (mm.a.elem != ElemType::F16 && mm.a.elem != ElemType::BF16))
        return reject("A and B must both be f16 or both bf16");
    auto nodes = chain_nodes(tree);
    size_t i = 0;
    auto at = [&](size_t j) -> const DecompNode* { return j < nodes.size() ? nodes[j] : nullptr; };
    const DecompNode* blk = at(i++);
    if (!blk || blk->kind != NodeKind::Tile || !blk->tile_ref.to || *blk->tile_ref.to != ComputeLevel::Block)
        return reject("first step must be the block tile (.to block)");
    tc.cta_group = blk->tile_ref.pair ? 2 : 1;
    tc.mcast = blk->tile_ref.multicast ? 2 : 1;
    tc.tile_m = static_cast<int>(blk->tile_r);
    tc.tile_n = static_cast<int>(blk->tile_c);
    // one TMEM lane per row: 128, 256 with .pair, or 512 with .pair and N = 256
    // (two A slabs per CTA sharing B, the whole TMEM per accumulator)
    if (tc.tile_m != 128 * tc.cta_group && !(tc.cta_group == 2 && tc.tile_m == 512))
        return reject("block tile M must be 128, 256 with .pair, or 512 with .pair and N 256");
    if (tc.tile_n != 64 && tc.tile_n != 128 && tc.tile_n != 256 && !(tc.tile_n == 512 && tc.cta_group == 2 && tc.tile_m == 256))
        return reject("block tile N must be 64, 128 or 256 (512 with .pair and M 256: two N halves sharing A)");
    const DecompNode* nx = at(i++);
    if (nx && nx->kind == NodeKind::Split && nx->split_ref.splitk) {
        tc.split_k = static_cast<int>(root.k() / nx->split_k);
        nx = at(i++);
    }
    if (!nx || nx->kind != NodeKind::Epilog || nx->acc_level.kind != MemKind::TM)
        return reject("expected 'epilog tm' after the block tile");
    {
        auto init = chain_nodes(nx->init_decomp);
        if (init.size() != 1 || init[0]->kind != NodeKind::Done || !init[0]->micro_kernel.empty())
            return reject("epilog init must be a single TMEM_ZERO leaf");
        auto store = chain_nodes(nx->store_decomp);
        if (store.size() != 2 || store[0]->kind != NodeKind::Tile || !store[0]->tile_ref.to ||
            *store[0]->tile_ref.to != ComputeLevel::Warp || store[0]->tile_r != 32 ||
            store[0]->tile_c != tc.tile_n || store[0]->tile_ref.swizzle || store[0]->tile_ref.layout ||
            store[1]->kind != NodeKind::Done)
            return reject("epilog store must be 'tile 32 BN .to warp' then the TMEM_STORE leaf");
    }
    const DecompNode* kl = at(i++);
    if (!kl || kl->kind != NodeKind::Split || kl->split_ref.splitk || kl->split_ref.unroll)
        return reject("expected the pipelined K split after the epilog");
    if (kl->split_k != 64) return reject("the K block must be 64 (one 128B swizzle span of 16-bit elements)");
    tc.tile_k = 64;
    tc.stages = kl->split_ref.stages;  // .prefetchLoads: 0 = the deepest ring that fits
    bool have_a = false, have_b = false;
    for (int j = 0; j < 2; ++j) {
        const DecompNode* ld = at(i++);
        if (!ld || ld->kind != NodeKind::Load || ld->target.kind != MemKind::SH)
            return reject("expected loads of A and B into SH");
        // A and B share each ring stage: a double-buffered operand makes the ring 2 deep
        if (ld->load_ref.double_buffer) {
            if (tc.stages != 0 && tc.stages != 2)
                return reject("load .doubleBuffer is a 2-stage TMA ring; it conflicts with .stages " +
                              std::to_string(tc.stages));
            if (kl->split_ref.prefetch) return reject("load .doubleBuffer conflicts with .prefetchLoads");
            tc.stages = 2;
        }
        if (ld->load_ref.pad || ld->load_ref.storage_layout || ld->load_ref.reuse_buffer || ld->load_ref.align)
            return reject("TMA loads use the 128B-swizzled layout; pad/storagelayout/align/reusebuffer do not apply");
        auto mv = chain_nodes(ld->move_decomp);
        if (mv.size() != 1 || mv[0]->kind != NodeKind::Done || !mv[0]->micro_kernel.empty())
            return reject("operand loads must bind the TMA_LOAD leaf directly");
        (ld->operand == Operand::A ? have_a : have_b) = true;
    }
    if (!have_a || !have_b) return reject("both A and B must be staged in SH");
    const DecompNode* leaf = at(i++);
    if (!leaf || leaf->kind != NodeKind::Done || at(i)) return reject("the chain must end in the UMMA leaf");
    // the residuals must bind the sm_100a leaves (validates leaf matching end to end)
    try {
        auto trace = elaborate(root, tree, mks);
        const Spec& last = trace.back().spec;
        ResidualBinding b = bind_done(last, leaf->micro_kernel, mks);
        if (!b.match.instruction || b.match.instruction->sim != SimSemantics::UMMA)
            return reject("leaf does not bind UMMA");
    } catch (const Error& e) {
        return reject(e.what());
    }
    if (tc.mcast > 1 && (tc.tile_m != 256 || tc.tile_n > 256 || tc.split_k > 1 || root.n() % (2L * tc.tile_n)))
        return reject("multicast pairs need 256-row tiles of N <= 256, no split-K, and N a multiple of 2 tiles");
    if ((tc.tile_m == 512 || tc.tile_n == 512) && tc.tile_m * tc.tile_n != 512 * 256)
        return reject("block tile M 512 needs N 256 (two A slabs sharing B), N 512 needs M 256 (two N halves sharing A)");
    if ((tc.tile_m == 512 || tc.tile_n == 512) && tc.split_k > 1)
        return reject("512 x 256 / 256 x 512 pair tiles take no split-K (their accumulator fills TMEM)");
    if (tc.split_k > 1) {
        const int cluster = tc.split_k * tc.cta_group;
        if (cluster > 8 || (tc.split_k != 2 && tc.split_k != 4))
            return reject("split-K ranks must be 2 or 4 with at most 8 CTAs per cluster");
        if (root.k() % (64L * tc.split_k)) return reject("K must split into 64-wide blocks per rank");
    }
    // Block .swizzle / .layout: an explicit schedule (tile_order[t] = RowMajor unit id)
    if (blk->tile_ref.swizzle || blk->tile_ref.layout.value_or(Major::RowMajor) == Major::ColMajor) {
        const long tiles_m = root.m() / tc.tile_m, tiles_n = root.n() / tc.tile_n, units = tiles_m * tiles_n;
        tc.tile_order.resize(static_cast<size_t>(units));
        for (long t = 0; t < units; ++t) {
            const long id = blk->tile_ref.swizzle ? apply_swizzle(blk->tile_ref.swizzle, t) : t;
            long row, col;
            if (blk->tile_ref.layout.value_or(Major::RowMajor) == Major::RowMajor) {
                row = id % tiles_m;
                col = id / tiles_m;
            } else {
                col = id % tiles_n;
                row = id / tiles_n;
            }
            tc.tile_order[static_cast<size_t>(t)] = static_cast<int32_t>(row + col * tiles_m);
        }
    }
    tc.matched = true;
    return tc;
}

}  // namespace fireiron
