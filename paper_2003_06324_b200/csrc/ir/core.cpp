// Spec core, index algebra and host matrices of the strategy IR.
// Semantics cite the reference (paths relative to /root/reference/proj).
#include <cmath>
#include <cstring>
#include <fstream>

#include "fireiron/error.hpp"
#include "fireiron/index_expr.hpp"
#include "fireiron/matrix.hpp"
#include "fireiron/types.hpp"

namespace fireiron {

// ---------------------------------------------------------------- errors
const char* error_kind_name(ErrorKind k) {
    static const char* const names[] = {
        "ZeroDim",           "ShapeMismatch",       "NonDivisible",        "NotMatMul",
        "CNotInGL",          "HierarchyViolation",  "UnitCountMismatch",   "UpwardLoad",
        "InvalidMoveDecomp", "PatternMismatch",     "NoExecutableMatch",   "AmbiguousMatch",
        "DuplicatePattern",  "SwizzleNotBijective", "InvalidRefinement",   "UnboundVar",
        "DivisionByZero",    "CapacityExceeded",    "ReuseBufferUnavailable",
        "OwnershipViolation", "UnsimulatableResidual", "ParseError",       "InvalidTree",
        "IoError"};
    const int i = static_cast<int>(k);
    return (i >= 0 && i < static_cast<int>(sizeof(names) / sizeof(names[0]))) ? names[i] : "Unknown";
}

Error::Error(ErrorKind kind, const std::string& msg)
    : std::runtime_error(std::string(error_kind_name(kind)) + ": " + msg), kind_(kind) {}

void fail(ErrorKind kind, const std::string& msg) { throw Error(kind, msg); }

// ---------------------------------------------------------------- types
int bit_width(ElemType t) { return t == ElemType::F32 ? 32 : 16; }
int byte_width(ElemType t) { return bit_width(t) / 8; }
const char* elem_name(ElemType t) {
    switch (t) {
        case ElemType::F32: return "f32";
        case ElemType::F16: return "f16";
        case ElemType::BF16: return "bf16";
    }
    return "?";
}
const char* elem_c_type(ElemType t) {
    switch (t) {
        case ElemType::F32: return "float";
        case ElemType::F16: return "__half";
        case ElemType::BF16: return "__nv_bfloat16";
    }
    return "?";
}

bool MemLevel::operator==(const MemLevel& o) const {
    if (kind != o.kind) return false;
    return kind != MemKind::FR || (fr_m == o.fr_m && fr_n == o.fr_n && fr_k == o.fr_k);
}

int mem_rank(MemKind k) {
    // types.hpp:48-56; TM sits with the per-unit storage levels
    return k == MemKind::GL ? 0 : k == MemKind::SH ? 1 : 2;
}

std::string mem_name(const MemLevel& m) {
    switch (m.kind) {
        case MemKind::GL: return "GL";
        case MemKind::SH: return "SH";
        case MemKind::RF: return "RF";
        case MemKind::FR: return "FR";
        case MemKind::TM: return "TM";
    }
    return "?";
}

const char* level_name(ComputeLevel l) {
    switch (l) {
        case ComputeLevel::Kernel: return "Kernel";
        case ComputeLevel::Block: return "Block";
        case ComputeLevel::Warp: return "Warp";
        case ComputeLevel::Thread: return "Thread";
    }
    return "?";
}

const char* major_name(Major m) { return m == Major::RowMajor ? "RowMajor" : "ColMajor"; }

// types.hpp:102-114: the pad extends the minor (contiguous) dimension
long Layout::row_stride(long, long cols) const {
    return major == Major::RowMajor ? cols + pad_cols : 1;
}
long Layout::col_stride(long rows, long) const {
    return major == Major::ColMajor ? rows + pad_cols : 1;
}
long Layout::extent(long rows, long cols) const {
    return major == Major::RowMajor ? rows * (cols + pad_cols) : cols * (rows + pad_cols);
}
long Layout::leading_dim(long rows, long cols) const {
    return major == Major::RowMajor ? cols + pad_cols : rows + pad_cols;
}

MatrixRef make_matrix(std::string name, long rows, long cols, ElemType elem, MemLevel mem,
                      Layout layout) {
    if (rows < 1 || cols < 1)
        fail(ErrorKind::ZeroDim, "matrix '" + name + "' has degenerate shape " +
                                     std::to_string(rows) + "x" + std::to_string(cols));
    MatrixRef r;
    r.name = std::move(name);
    r.rows = rows;
    r.cols = cols;
    r.elem = elem;
    r.mem = mem;
    r.layout = layout;
    return r;
}

Spec make_matmul_spec(long m, long n, long k, ElemTriple elems, MemTriple mems,
                      LayoutTriple layouts, ComputeLevel level) {
    if (m < 1 || n < 1 || k < 1)
        fail(ErrorKind::ZeroDim, "matmul dims must be positive, got " + std::to_string(m) + "x" +
                                     std::to_string(n) + "x" + std::to_string(k));
    Spec s;
    s.kind = Spec::Kind::MatMul;
    s.level = level;
    s.op = MatMulOp{make_matrix("A", m, k, elems.a, mems.a, layouts.a),
                    make_matrix("B", k, n, elems.b, mems.b, layouts.b),
                    make_matrix("C", m, n, elems.c, mems.c, layouts.c)};
    return s;
}

Spec make_move_spec(MatrixRef src, MatrixRef dst, ComputeLevel level) {
    if (src.rows != dst.rows || src.cols != dst.cols)
        fail(ErrorKind::ShapeMismatch, "move endpoints differ in shape: " + std::to_string(src.rows) +
                                           "x" + std::to_string(src.cols) + " vs " +
                                           std::to_string(dst.rows) + "x" + std::to_string(dst.cols));
    if (src.elem != dst.elem) fail(ErrorKind::ShapeMismatch, "move endpoints differ in element type");
    Spec s;
    s.kind = Spec::Kind::Move;
    s.level = level;
    s.op = MoveOp{std::move(src), std::move(dst)};
    return s;
}

std::string spec_short_form(const Spec& s) {
    const std::string lv = std::string("(") + level_name(s.level) + ")";
    if (s.is_matmul()) {
        const auto& o = s.mm();
        return "MatMul(" + std::to_string(s.m()) + "," + std::to_string(s.n()) + "," +
               std::to_string(s.k()) + ")(" + mem_name(o.a.mem) + "," + mem_name(o.b.mem) + "," +
               mem_name(o.c.mem) + ")" + lv;
    }
    const auto& o = s.mv();
    return "Move(" + std::to_string(o.src.rows) + "x" + std::to_string(o.src.cols) + ")(" +
           mem_name(o.src.mem) + "->" + mem_name(o.dst.mem) + ")" + lv;
}

// ---------------------------------------------------------------- index algebra
Expr iconst(long v) {
    auto n = std::make_shared<ExprNode>();
    n->op = ExprOp::Const;
    n->value = v;
    return n;
}
Expr ivar(std::string name) {
    auto n = std::make_shared<ExprNode>();
    n->op = ExprOp::Var;
    n->name = std::move(name);
    return n;
}
Expr ibin(ExprOp op, Expr a, Expr b) {
    auto n = std::make_shared<ExprNode>();
    n->op = op;
    n->lhs = std::move(a);
    n->rhs = std::move(b);
    return n;
}
bool is_const(const Expr& e, long v) { return e->op == ExprOp::Const && e->value == v; }

namespace {
long apply_op(ExprOp op, long a, long b, bool strict) {
    switch (op) {
        case ExprOp::Add: return a + b;
        case ExprOp::Mul: return a * b;
        case ExprOp::Div:
            if (b == 0) {
                if (strict) fail(ErrorKind::DivisionByZero, "division by zero");
                return 0;
            }
            return a / b;
        case ExprOp::Mod:
            if (b == 0) {
                if (strict) fail(ErrorKind::DivisionByZero, "modulo by zero");
                return 0;
            }
            return a % b;
        case ExprOp::Shr: return a >> b;
        case ExprOp::Shl: return a << b;
        case ExprOp::BitAnd: return a & b;
        case ExprOp::BitOr: return a | b;
        default: break;
    }
    fail(ErrorKind::UnboundVar, "malformed expression node");
}
bool commutes(ExprOp op) {
    return op == ExprOp::Add || op == ExprOp::Mul || op == ExprOp::BitAnd || op == ExprOp::BitOr;
}
}  // namespace

long eval(const Expr& e, const Env& env) {
    if (e->op == ExprOp::Const) return e->value;
    if (e->op == ExprOp::Var) {
        auto it = env.find(e->name);
        if (it == env.end()) fail(ErrorKind::UnboundVar, "no binding for '" + e->name + "'");
        return it->second;
    }
    const long a = eval(e->lhs, env);
    const long b = eval(e->rhs, env);
    return apply_op(e->op, a, b, true);
}

// index_expr.hpp:115-191: a fixed rewrite list applied bottom-up, constants
// canonicalised to the right of commutative operators.
Expr simplify(const Expr& e) {
    if (e->op == ExprOp::Const || e->op == ExprOp::Var) return e;
    Expr a = simplify(e->lhs);
    Expr b = simplify(e->rhs);
    const ExprOp op = e->op;
    for (int guard = 0; guard < 8; ++guard) {
        if (a->op == ExprOp::Const && b->op == ExprOp::Const)
            return iconst(apply_op(op, a->value, b->value, false));
        if (commutes(op) && a->op == ExprOp::Const) std::swap(a, b);
        if (b->op == ExprOp::Const) {
            const long c = b->value;
            const bool a_scaled = a->op == ExprOp::Mul && a->rhs->op == ExprOp::Const;
            bool again = false;
            switch (op) {
                case ExprOp::Add:
                    if (c == 0) return a;
                    if (a->op == ExprOp::Add && a->rhs->op == ExprOp::Const) {
                        b = iconst(a->rhs->value + c);
                        a = a->lhs;
                        again = true;
                    }
                    break;
                case ExprOp::Mul:
                    if (c == 0) return iconst(0);
                    if (c == 1) return a;
                    if (a_scaled) {
                        b = iconst(a->rhs->value * c);
                        a = a->lhs;
                        again = true;
                    }
                    break;
                case ExprOp::Div:
                    if (c == 1) return a;
                    if (a_scaled && c != 0 && a->rhs->value % c == 0)
                        return simplify(imul(a->lhs, iconst(a->rhs->value / c)));
                    break;
                case ExprOp::Mod:
                    if (c == 1) return iconst(0);
                    if (a_scaled && c != 0 && a->rhs->value % c == 0) return iconst(0);
                    break;
                case ExprOp::Shr:
                case ExprOp::Shl:
                case ExprOp::BitOr:
                    if (c == 0) return a;
                    break;
                case ExprOp::BitAnd:
                    if (c == 0) return iconst(0);
                    break;
                default: break;
            }
            if (again) continue;
        }
        if (is_const(a, 0) && (op == ExprOp::Div || op == ExprOp::Mod || op == ExprOp::Shr ||
                               op == ExprOp::Shl))
            return iconst(0);
        break;
    }
    return ibin(op, a, b);
}

namespace {
const char* op_text(ExprOp op) {
    switch (op) {
        case ExprOp::Add: return "+";
        case ExprOp::Mul: return "*";
        case ExprOp::Div: return "/";
        case ExprOp::Mod: return "%";
        case ExprOp::Shr: return ">>";
        case ExprOp::Shl: return "<<";
        case ExprOp::BitAnd: return "&";
        case ExprOp::BitOr: return "|";
        default: return "?";
    }
}
}  // namespace

std::string emit_c(const Expr& e) {
    if (e->op == ExprOp::Const) return std::to_string(e->value);
    if (e->op == ExprOp::Var) return e->name;
    return "(" + emit_c(e->lhs) + " " + op_text(e->op) + " " + emit_c(e->rhs) + ")";
}

long apply_swizzle(const Expr& s, long id) { return eval(s, Env{{"id", id}}); }

Expr subst_var(const Expr& e, const std::string& name, const Expr& repl) {
    if (e->op == ExprOp::Const) return e;
    if (e->op == ExprOp::Var) return e->name == name ? repl : e;
    return ibin(e->op, subst_var(e->lhs, name, repl), subst_var(e->rhs, name, repl));
}

bool structurally_equal(const Expr& a, const Expr& b) {
    if (a.get() == b.get()) return true;
    if (a->op != b->op) return false;
    if (a->op == ExprOp::Const) return a->value == b->value;
    if (a->op == ExprOp::Var) return a->name == b->name;
    return structurally_equal(a->lhs, b->lhs) && structurally_equal(a->rhs, b->rhs);
}

// ---------------------------------------------------------------- matrices
Matrix Matrix::zeros(long r, long c, Layout l) {
    Matrix m;
    m.rows = r;
    m.cols = c;
    m.layout = l;
    m.data.assign(static_cast<size_t>(l.extent(r, c)), 0.0f);
    return m;
}

uint64_t Rng::next() {  // splitmix64, matrix.hpp:37-46
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

void fill_integers(Matrix& m, uint64_t seed, long lo, long hi) {
    Rng rng(seed);
    const uint64_t span = static_cast<uint64_t>(hi - lo + 1);
    for (long r = 0; r < m.rows; ++r)
        for (long c = 0; c < m.cols; ++c)
            m.at(r, c) = static_cast<float>(lo + static_cast<long>(rng.next() % span));
}

void fill_uniform(Matrix& m, uint64_t seed) {
    Rng rng(seed);
    for (long r = 0; r < m.rows; ++r)
        for (long c = 0; c < m.cols; ++c) {
            const double u = static_cast<double>(rng.next() >> 11) * 0x1.0p-53;
            m.at(r, c) = static_cast<float>(2.0 * u - 1.0);
        }
}

float round_to_f16(float x) {  // matrix.hpp:67-80
    if (x == 0.0f || !std::isfinite(x)) return x;
    int e = 0;
    std::frexp(std::fabs(x), &e);
    if (e - 1 < -14) {
        const float q = std::ldexp(1.0f, -24);
        return std::nearbyint(x / q) * q;
    }
    if (e - 1 > 15) return x > 0 ? 65504.0f : -65504.0f;
    return std::ldexp(std::nearbyint(std::ldexp(x, 11 - e)), e - 11);
}

float round_to_bf16(float x) {
    if (!std::isfinite(x)) return x;
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

void round_matrix_to_f16(Matrix& m) {
    for (auto& v : m.data) v = round_to_f16(v);
}

void round_matrix(Matrix& m, ElemType e) {
    if (e == ElemType::F16)
        for (auto& v : m.data) v = round_to_f16(v);
    else if (e == ElemType::BF16)
        for (auto& v : m.data) v = round_to_bf16(v);
}

uint64_t digest(const Matrix& m) {  // FNV-1a, matrix.hpp:86-103
    uint64_t h = 1469598103934665603ull;
    for (long r = 0; r < m.rows; ++r)
        for (long c = 0; c < m.cols; ++c) {
            const float v = m.at(r, c);
            uint32_t bits;
            std::memcpy(&bits, &v, 4);
            for (int i = 0; i < 4; ++i) {
                h ^= (bits >> (8 * i)) & 0xffu;
                h *= 1099511628211ull;
            }
        }
    return h;
}

Matrix read_matrix(const std::string& path, Layout layout) {
    std::ifstream in(path);
    if (!in) fail(ErrorKind::IoError, "cannot open '" + path + "'");
    long rows = 0, cols = 0;
    if (!(in >> rows >> cols) || rows < 1 || cols < 1)
        fail(ErrorKind::IoError, "bad matrix header in '" + path + "'");
    Matrix m = Matrix::zeros(rows, cols, layout);
    for (long r = 0; r < rows; ++r)
        for (long c = 0; c < cols; ++c)
            if (!(in >> m.at(r, c))) fail(ErrorKind::IoError, "short matrix data in '" + path + "'");
    return m;
}

void write_matrix(const std::string& path, const Matrix& m) {
    std::ofstream out(path);
    if (!out) fail(ErrorKind::IoError, "cannot open '" + path + "' for writing");
    out << m.rows << " " << m.cols << "\n";
    for (long r = 0; r < m.rows; ++r) {
        for (long c = 0; c < m.cols; ++c) out << (c ? " " : "") << m.at(r, c);
        out << "\n";
    }
}

}  // namespace fireiron
