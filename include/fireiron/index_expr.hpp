// Symbolic integer index algebra (loop variables, unit ids, swizzles).
// API-compatible with proj/include/anvil/index_expr.hpp:16-233; domain is
// nonnegative integers so C and floor division agree.
#pragma once

#include <map>
#include <memory>
#include <string>

#include "fireiron/error.hpp"

namespace fireiron {

enum class ExprOp { Const, Var, Add, Mul, Div, Mod, Shr, Shl, BitAnd, BitOr };

struct ExprNode;
using Expr = std::shared_ptr<const ExprNode>;

struct ExprNode {
    ExprOp op = ExprOp::Const;
    long value = 0;    // Const
    std::string name;  // Var
    Expr lhs, rhs;     // binary
};

Expr iconst(long v);
Expr ivar(std::string name);
Expr ibin(ExprOp op, Expr a, Expr b);
inline Expr iadd(Expr a, Expr b) { return ibin(ExprOp::Add, std::move(a), std::move(b)); }
inline Expr imul(Expr a, Expr b) { return ibin(ExprOp::Mul, std::move(a), std::move(b)); }
inline Expr idiv(Expr a, Expr b) { return ibin(ExprOp::Div, std::move(a), std::move(b)); }
inline Expr imod(Expr a, Expr b) { return ibin(ExprOp::Mod, std::move(a), std::move(b)); }
inline Expr ishr(Expr a, Expr b) { return ibin(ExprOp::Shr, std::move(a), std::move(b)); }
inline Expr ishl(Expr a, Expr b) { return ibin(ExprOp::Shl, std::move(a), std::move(b)); }
inline Expr iand(Expr a, Expr b) { return ibin(ExprOp::BitAnd, std::move(a), std::move(b)); }
inline Expr ior(Expr a, Expr b) { return ibin(ExprOp::BitOr, std::move(a), std::move(b)); }

bool is_const(const Expr& e, long v);

using Env = std::map<std::string, long>;
long eval(const Expr& e, const Env& env);

// Terminating rewrite set: constant folding, 0*x, 1*x, x+0, (x*c1)*c2,
// (x+c1)+c2, x/1, x%1, (x*c1)/c2 and (x*c1)%c2 when c2 | c1, shifts by 0,
// x&0, x|0, 0 op x for the non-commutative ops.
Expr simplify(const Expr& e);

// Fully parenthesised C text, constants in decimal.
std::string emit_c(const Expr& e);

// Swizzle over the single free variable "id".
long apply_swizzle(const Expr& s, long id);
Expr subst_var(const Expr& e, const std::string& name, const Expr& repl);
bool structurally_equal(const Expr& a, const Expr& b);

}  // namespace fireiron
