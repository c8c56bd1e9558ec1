// Strategy scripts: tokenizer, parser and canonical printer
// (reference grammar: proj/include/anvil/script.hpp:38-793).
#include "fireiron/script.hpp"

#include <cctype>
#include <cstring>

namespace fireiron {

namespace {

struct Token {
    std::string text;
    int col = 0;
};
struct Line {
    int number = 0;
    std::vector<Token> tokens;
};

std::string lowercase(std::string s) {
    for (auto& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}

[[noreturn]] void parse_fail(int line, int col, const std::string& msg) {
    fail(ErrorKind::ParseError, "line " + std::to_string(line) + ", col " + std::to_string(col) + ": " + msg);
}

// Whitespace tokens per line; '#' starts a comment. raw keeps every line.
std::vector<Line> tokenize(const std::string& text, std::vector<std::string>& raw) {
    std::vector<Line> lines;
    raw.clear();
    size_t start = 0;
    int number = 0;
    while (start <= text.size()) {
        size_t end = text.find('\n', start);
        if (end == std::string::npos) end = text.size();
        std::string s = text.substr(start, end - start);
        raw.push_back(s);
        ++number;
        if (auto h = s.find('#'); h != std::string::npos) s.resize(h);
        Line ln;
        ln.number = number;
        for (size_t i = 0; i < s.size();) {
            if (std::isspace(static_cast<unsigned char>(s[i]))) {
                ++i;
                continue;
            }
            size_t j = i;
            while (j < s.size() && !std::isspace(static_cast<unsigned char>(s[j]))) ++j;
            ln.tokens.push_back({s.substr(i, j - i), static_cast<int>(i) + 1});
            i = j;
        }
        if (!ln.tokens.empty()) lines.push_back(std::move(ln));
        if (end == text.size()) break;
        start = end + 1;
    }
    return lines;
}

// Recursive-descent parser for one whitespace-free swizzle token. Precedence
// (loosest first): |, &, << >>, +, * / %.
class ExprReader {
public:
    ExprReader(const std::string& s, int line, int col) : s_(s), line_(line), col_(col) {}

    Expr parse() {
        Expr e = bit_or();
        if (p_ != s_.size()) err("trailing characters");
        return e;
    }

private:
    const std::string& s_;
    size_t p_ = 0;
    int line_, col_;

    [[noreturn]] void err(const std::string& m) { parse_fail(line_, col_, m + " in '" + s_ + "'"); }
    bool take(char c) {
        if (p_ < s_.size() && s_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    bool take2(char a, char b) {
        if (p_ + 1 < s_.size() && s_[p_] == a && s_[p_ + 1] == b) {
            p_ += 2;
            return true;
        }
        return false;
    }
    Expr atom() {
        if (take('(')) {
            Expr e = bit_or();
            if (!take(')')) err("expected ')'");
            return e;
        }
        if (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) {
            const size_t b = p_;
            if (s_.compare(p_, 2, "0x") == 0 || s_.compare(p_, 2, "0X") == 0) {
                p_ += 2;
                while (p_ < s_.size() && std::isxdigit(static_cast<unsigned char>(s_[p_]))) ++p_;
                return iconst(std::stol(s_.substr(b + 2, p_ - b - 2), nullptr, 16));
            }
            while (p_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[p_]))) ++p_;
            return iconst(std::stol(s_.substr(b, p_ - b)));
        }
        if (p_ < s_.size() && (std::isalpha(static_cast<unsigned char>(s_[p_])) || s_[p_] == '_')) {
            const size_t b = p_;
            while (p_ < s_.size() &&
                   (std::isalnum(static_cast<unsigned char>(s_[p_])) || s_[p_] == '_' || s_[p_] == '.'))
                ++p_;
            return ivar(s_.substr(b, p_ - b));
        }
        err("expected an operand");
    }
    Expr product() {
        Expr e = atom();
        for (;;) {
            if (take('*')) e = imul(e, atom());
            else if (take('/')) e = idiv(e, atom());
            else if (take('%')) e = imod(e, atom());
            else return e;
        }
    }
    Expr sum() {
        Expr e = product();
        while (take('+')) e = iadd(e, product());
        return e;
    }
    Expr shift() {
        Expr e = sum();
        for (;;) {
            if (take2('>', '>')) e = ishr(e, sum());
            else if (take2('<', '<')) e = ishl(e, sum());
            else return e;
        }
    }
    Expr bit_and() {
        Expr e = shift();
        while (take('&')) e = iand(e, shift());
        return e;
    }
    Expr bit_or() {
        Expr e = bit_and();
        while (take('|')) e = ior(e, bit_and());
        return e;
    }
};

ComputeLevel parse_level(const std::string& tok, int line, int col) {
    const std::string t = lowercase(tok);
    if (t == "kernel") return ComputeLevel::Kernel;
    if (t == "block" || t == "cta") return ComputeLevel::Block;
    if (t == "warp") return ComputeLevel::Warp;
    if (t == "thread" || t == "lane") return ComputeLevel::Thread;
    parse_fail(line, col, "unknown compute level '" + tok + "'");
}

MemLevel parse_mem(const std::string& tok, int line, int col) {
    const std::string t = lowercase(tok);
    if (t == "gl") return MemLevel::gl();
    if (t == "sh") return MemLevel::sh();
    if (t == "rf") return MemLevel::rf();
    if (t == "fr") return MemLevel::fr();
    if (t == "tm") return MemLevel::tm();
    if (t.rfind("fr(", 0) == 0 || t.rfind("fr<", 0) == 0) {
        long dims[3] = {0, 0, 0};
        size_t p = 3;
        for (long& d : dims) {
            size_t q = p;
            while (q < t.size() && std::isdigit(static_cast<unsigned char>(t[q]))) ++q;
            if (q == p) parse_fail(line, col, "bad fragment geometry in '" + tok + "'");
            d = std::stol(t.substr(p, q - p));
            p = q + 1;
        }
        return MemLevel::fr(static_cast<int>(dims[0]), static_cast<int>(dims[1]), static_cast<int>(dims[2]));
    }
    parse_fail(line, col, "unknown memory level '" + tok + "'");
}

Major parse_major(const std::string& tok, int line, int col) {
    const std::string t = lowercase(tok);
    if (t == "rowmajor") return Major::RowMajor;
    if (t == "colmajor") return Major::ColMajor;
    parse_fail(line, col, "unknown layout '" + tok + "' (rowmajor|colmajor)");
}

ElemType parse_elem(const std::string& tok, int line, int col) {
    const std::string t = lowercase(tok);
    if (t == "f32" || t == "float") return ElemType::F32;
    if (t == "f16" || t == "half") return ElemType::F16;
    if (t == "bf16" || t == "bfloat16") return ElemType::BF16;
    parse_fail(line, col, "unknown element type '" + tok + "' (f32|f16|bf16)");
}

Operand parse_operand(const std::string& tok, int line, int col) {
    const std::string t = lowercase(tok);
    if (t == "a") return Operand::A;
    if (t == "b") return Operand::B;
    if (t == "src") return Operand::Src;
    parse_fail(line, col, "unknown operand '" + tok + "' (a|b|src)");
}

struct Cursor {
    const std::vector<Line>& lines;
    size_t i = 0;
    bool done() const { return i >= lines.size(); }
    const Line& peek() const { return lines[i]; }
    const Line& next() { return lines[i++]; }
};

void apply_header_groups(Spec& root, const Line& line, size_t from) {
    size_t i = from;
    const size_t n = root.is_matmul() ? 3 : 2;
    auto need = [&](const char* what) {
        if (i + n + 1 > line.tokens.size())
            parse_fail(line.number, line.tokens.back().col, std::string("missing ") + what);
    };
    while (i < line.tokens.size()) {
        const std::string key = lowercase(line.tokens[i].text);
        if (key == "elems") {
            need("element types");
            std::vector<ElemType> e;
            for (size_t j = 0; j < n; ++j)
                e.push_back(parse_elem(line.tokens[i + 1 + j].text, line.number, line.tokens[i + 1 + j].col));
            if (root.is_matmul()) {
                root.mm().a.elem = e[0];
                root.mm().b.elem = e[1];
                root.mm().c.elem = e[2];
            } else {
                root.mv().src.elem = e[0];
                root.mv().dst.elem = e[1];
                if (e[0] != e[1])
                    parse_fail(line.number, line.tokens[i].col, "move endpoints must share an element type");
            }
        } else if (key == "layouts") {
            need("layouts");
            std::vector<Major> m;
            for (size_t j = 0; j < n; ++j)
                m.push_back(parse_major(line.tokens[i + 1 + j].text, line.number, line.tokens[i + 1 + j].col));
            if (root.is_matmul()) {
                root.mm().a.layout.major = m[0];
                root.mm().b.layout.major = m[1];
                root.mm().c.layout.major = m[2];
            } else {
                root.mv().src.layout.major = m[0];
                root.mv().dst.layout.major = m[1];
            }
        } else {
            parse_fail(line.number, line.tokens[i].col, "unexpected token '" + line.tokens[i].text + "'");
        }
        i += n + 1;
    }
}

NodePtr parse_chain(Cursor& cur, bool expect_close);

long int_token(const Line& ln, size_t i, const char* what) {
    const auto& t = ln.tokens;
    if (i >= t.size()) parse_fail(ln.number, t.back().col, std::string("missing ") + what);
    try {
        size_t used = 0;
        long v = std::stol(t[i].text, &used);
        (void)used;
        return v;
    } catch (...) {
        parse_fail(ln.number, t[i].col, std::string("bad ") + what + " '" + t[i].text + "'");
    }
}

const Token& tok_at(const Line& ln, size_t i, const char* what) {
    if (i >= ln.tokens.size()) parse_fail(ln.number, ln.tokens.back().col, std::string("missing ") + what);
    return ln.tokens[i];
}

// One step; `to` lines merge into the previous tile and return nullptr.
NodePtr parse_step(Cursor& cur, const Line& ln, NodePtr prev) {
    const auto& t = ln.tokens;
    const std::string head = lowercase(t[0].text);
    if (head == "tile") {
        const long r = int_token(ln, 1, "tile rows"), c = int_token(ln, 2, "tile cols");
        TileRefinements ref;
        for (size_t i = 3; i < t.size();) {
            const std::string k = lowercase(t[i].text);
            if (k == ".to") {
                const Token& v = tok_at(ln, i + 1, "level");
                ref.to = parse_level(v.text, ln.number, v.col);
                i += 2;
            } else if (k == ".layout") {
                const Token& v = tok_at(ln, i + 1, "layout");
                ref.layout = parse_major(v.text, ln.number, v.col);
                i += 2;
            } else if (k == ".swizzle") {
                const Token& v = tok_at(ln, i + 1, "swizzle expression");
                ref.swizzle = ExprReader(v.text, ln.number, v.col).parse();
                i += 2;
            } else if (k == ".unroll") {
                ref.unroll = true;
                ++i;
            } else if (k == ".pair") {
                ref.pair = true;
                ++i;
            } else if (k == ".multicast") {
                ref.multicast = true;
                ++i;
            } else {
                parse_fail(ln.number, t[i].col, "unknown tile refinement '" + t[i].text + "'");
            }
        }
        try {
            return n_tile(r, c, std::move(ref), nullptr, ln.number);
        } catch (const Error& e) {
            parse_fail(ln.number, t[0].col, e.what());
        }
    }
    if (head == "to") {
        const Token& v = tok_at(ln, 1, "level");
        if (t.size() > 2) parse_fail(ln.number, t[2].col, "unexpected token after 'to'");
        if (!prev || prev->kind != NodeKind::Tile || prev->tile_ref.to)
            parse_fail(ln.number, t[0].col, "'to' must follow a tile step without one");
        prev->tile_ref.to = parse_level(v.text, ln.number, v.col);
        return nullptr;
    }
    if (head == "split") {
        const long k = int_token(ln, 1, "split size");
        SplitRefinements ref;
        for (size_t i = 2; i < t.size();) {
            const std::string kw = lowercase(t[i].text);
            if (kw == ".unroll") ref.unroll = true;
            else if (kw == ".sync") ref.sync = true;
            else if (kw == ".splitk") ref.splitk = true;
            else if (kw == ".prefetchloads") ref.prefetch = true;
            else if (kw == ".doublebufferloop") ref.double_buffer = true;
            else if (kw == ".stages") {
                ref.stages = static_cast<int>(int_token(ln, i + 1, "stage count"));
                i += 2;
                continue;
            } else parse_fail(ln.number, t[i].col, "unknown split refinement '" + t[i].text + "'");
            ++i;
        }
        try {
            return n_split(k, ref, nullptr, ln.number);
        } catch (const Error& e) {
            parse_fail(ln.number, t[0].col, e.what());
        }
    }
    if (head == "load") {
        const Operand op = parse_operand(tok_at(ln, 1, "operand").text, ln.number, t[1].col);
        const MemLevel target = parse_mem(tok_at(ln, 2, "target level").text, ln.number, t[2].col);
        LoadRefinements ref;
        bool open = false;
        for (size_t i = 3; i < t.size();) {
            const std::string k = lowercase(t[i].text);
            if (k == "{") {
                open = true;
                if (i + 1 != t.size()) parse_fail(ln.number, t[i + 1].col, "'{' ends the line");
                break;
            }
            if (k == ".storagelayout") {
                const Token& v = tok_at(ln, i + 1, "layout");
                ref.storage_layout = parse_major(v.text, ln.number, v.col);
                i += 2;
            } else if (k == ".pad") {
                ref.pad = int_token(ln, i + 1, "pad");
                i += 2;
            } else if (k == ".align") {
                ref.align = int_token(ln, i + 1, "align");
                i += 2;
            } else if (k == ".nosync") {
                ref.no_sync = true;
                ++i;
            } else if (k == ".reusebuffer") {
                ref.reuse_buffer = true;
                ++i;
            } else if (k == ".doublebuffer") {
                ref.double_buffer = true;
                ++i;
            } else if (k == ".postponed") {
                ref.postponed = true;
                ++i;
            } else {
                parse_fail(ln.number, t[i].col, "unknown load refinement '" + t[i].text + "'");
            }
        }
        if (!open) parse_fail(ln.number, t.back().col, "load needs a '{ ... }' move decomposition");
        NodePtr move = parse_chain(cur, true);
        try {
            return n_load(op, target, std::move(move), std::move(ref), nullptr, ElemType::F32, ln.number);
        } catch (const Error& e) {
            parse_fail(ln.number, t[0].col, e.what());
        }
    }
    if (head == "epilog") {
        const MemLevel acc = parse_mem(tok_at(ln, 1, "accumulator level").text, ln.number, t[1].col);
        if (t.size() < 3 || t[2].text != "{")
            parse_fail(ln.number, t.back().col, "epilog needs '{ init { ... } store { ... } }'");
        auto block = [&](const char* name) {
            if (cur.done()) parse_fail(ln.number, 1, std::string("missing ") + name + " block");
            const Line& l = cur.next();
            if (lowercase(l.tokens[0].text) != name || l.tokens.size() != 2 || l.tokens[1].text != "{")
                parse_fail(l.number, l.tokens[0].col, std::string("expected '") + name + " {'");
            return parse_chain(cur, true);
        };
        NodePtr init = block("init");
        NodePtr store = block("store");
        if (cur.done() || cur.peek().tokens[0].text != "}") parse_fail(ln.number, 1, "epilog block not closed");
        cur.next();
        return n_epilog(acc, std::move(init), std::move(store), nullptr, ln.number);
    }
    if (head == "mmatile") {
        if (t.size() > 1) parse_fail(ln.number, t[1].col, "mmaTile takes no arguments");
        return n_mma_tile(nullptr, ln.number);
    }
    if (head == "done") {
        if (t.size() > 2) parse_fail(ln.number, t[2].col, "unexpected token after done");
        return n_done(t.size() > 1 ? t[1].text : "", ln.number);
    }
    parse_fail(ln.number, t[0].col, "unknown step '" + t[0].text + "'");
}

NodePtr parse_chain(Cursor& cur, bool expect_close) {
    std::vector<NodePtr> steps;
    bool closed = false;
    while (!cur.done()) {
        const Line& ln = cur.peek();
        if (ln.tokens[0].text == "}") {
            cur.next();
            closed = true;
            break;
        }
        cur.next();
        NodePtr n = parse_step(cur, ln, steps.empty() ? nullptr : steps.back());
        if (n) steps.push_back(std::move(n));
    }
    if (expect_close && !closed)
        parse_fail(cur.lines.empty() ? 1 : cur.lines.back().number, 1, "unterminated block ('}' missing)");
    NodePtr chain;
    for (auto it = steps.rbegin(); it != steps.rend(); ++it) {
        (*it)->child = std::move(chain);
        chain = *it;
    }
    return chain;
}

MicroKernel build_micro_kernel(const MicroKernelSection& sec, const Spec& root) {
    MicroKernel mk;
    mk.name = sec.name;
    mk.pattern = parse_spec_short_form(sec.pattern_line, &root, sec.line);
    mk.body = sec.body;
    mk.declared_vars = sec.vars;
    return mk;
}

}  // namespace

// script.hpp:259-334
Spec parse_spec_short_form(const std::string& text, const Spec* basis, int line) {
    size_t pos = 0;
    auto err = [&](const std::string& m) { parse_fail(line, static_cast<int>(pos) + 1, m); };
    auto expect = [&](char c) {
        if (pos >= text.size() || text[pos] != c) err(std::string("expected '") + c + "'");
        ++pos;
    };
    auto until = [&](const char* stops) {
        const size_t b = pos;
        while (pos < text.size() && !std::strchr(stops, text[pos])) ++pos;
        return text.substr(b, pos - b);
    };
    auto dim = [&](const std::string& tok) -> long {
        if (basis) {
            const std::string t = lowercase(tok);
            if (t == "m") return basis->m();
            if (t == "n") return basis->n();
            if (t == "k") return basis->k();
        }
        try {
            return std::stol(tok);
        } catch (...) {
            parse_fail(line, static_cast<int>(pos) + 1, "bad dimension '" + tok + "'");
        }
    };
    const std::string head = lowercase(until("("));
    if (head == "matmul") {
        expect('(');
        const long m = dim(until(","));
        expect(',');
        const long n = dim(until(","));
        expect(',');
        const long k = dim(until(")"));
        expect(')');
        expect('(');
        const MemLevel ma = parse_mem(until(","), line, static_cast<int>(pos));
        expect(',');
        const MemLevel mb = parse_mem(until(","), line, static_cast<int>(pos));
        expect(',');
        const MemLevel mc = parse_mem(until(")"), line, static_cast<int>(pos));
        expect(')');
        expect('(');
        const ComputeLevel lv = parse_level(until(")"), line, static_cast<int>(pos));
        expect(')');
        if (pos != text.size()) err("trailing characters after short form");
        return make_matmul_spec(m, n, k, {}, {ma, mb, mc},
                                {Layout::col_major(), Layout::col_major(), Layout::col_major()}, lv);
    }
    if (head == "move") {
        expect('(');
        const long r = dim(until("x"));
        expect('x');
        const long c = dim(until(")"));
        expect(')');
        expect('(');
        const MemLevel ms = parse_mem(until("-"), line, static_cast<int>(pos));
        expect('-');
        expect('>');
        const MemLevel md = parse_mem(until(")"), line, static_cast<int>(pos));
        expect(')');
        expect('(');
        const ComputeLevel lv = parse_level(until(")"), line, static_cast<int>(pos));
        expect(')');
        if (pos != text.size()) err("trailing characters after short form");
        return make_move_spec(make_matrix("SRC", r, c, ElemType::F32, ms, Layout::col_major()),
                              make_matrix("DST", r, c, ElemType::F32, md, Layout::col_major()), lv);
    }
    parse_fail(line, 1, "expected MatMul(...) or Move(...)");
}

// script.hpp:607-668
ParsedScript parse_script(const std::string& text) {
    std::vector<std::string> raw;
    const std::vector<Line> lines = tokenize(text, raw);
    if (lines.empty()) fail(ErrorKind::ParseError, "line 1, col 1: empty script");
    Cursor cur{lines};
    const Line& header = cur.next();
    if (lowercase(header.tokens[0].text) != "spec" || header.tokens.size() < 2)
        parse_fail(header.number, header.tokens[0].col, "script must start with 'spec <short-form>'");
    ParsedScript out;
    out.root = parse_spec_short_form(header.tokens[1].text, nullptr, header.number);
    apply_header_groups(out.root, header, 2);

    while (!cur.done() && lowercase(cur.peek().tokens[0].text) == "microkernel") {
        const Line& head = cur.next();
        if (head.tokens.size() != 2) parse_fail(head.number, head.tokens[0].col, "microkernel <name>");
        MicroKernelSection sec;
        sec.name = head.tokens[1].text;
        sec.line = head.number;
        if (cur.done() || lowercase(cur.peek().tokens[0].text) != "pattern")
            parse_fail(head.number, 1, "microkernel needs a 'pattern <short-form>' line");
        const Line& pat = cur.next();
        if (pat.tokens.size() != 2) parse_fail(pat.number, pat.tokens[0].col, "pattern <short-form>");
        sec.pattern_line = pat.tokens[1].text;
        if (!cur.done() && lowercase(cur.peek().tokens[0].text) == "vars") {
            const Line& vars = cur.next();
            for (size_t i = 1; i < vars.tokens.size(); ++i) sec.vars.push_back(vars.tokens[i].text);
        }
        if (cur.done() || cur.peek().tokens[0].text != "---")
            parse_fail(sec.line, 1, "microkernel body must be fenced with --- lines");
        const int fence = cur.peek().number;
        cur.next();
        // verbatim body: raw lines up to the closing fence (raw is 0-based)
        int close = -1;
        for (size_t r = static_cast<size_t>(fence); r < raw.size(); ++r)
            if (raw[r] == "---") {
                close = static_cast<int>(r);
                break;
            }
        if (close < 0) parse_fail(fence, 1, "unterminated microkernel body");
        for (int r = fence; r < close; ++r) sec.body += raw[static_cast<size_t>(r)] + "\n";
        while (!cur.done() && cur.peek().number <= close + 1) cur.next();
        out.micro_kernels.register_kernel(build_micro_kernel(sec, out.root));
        out.micro_kernel_sections.push_back(std::move(sec));
    }
    out.tree = parse_chain(cur, false);
    if (!out.tree) fail(ErrorKind::ParseError, "line 1, col 1: script has no decomposition steps");
    return out;
}

std::string expr_token(const Expr& e) {
    if (e->op == ExprOp::Const) return std::to_string(e->value);
    if (e->op == ExprOp::Var) return e->name;
    const char* op = "?";
    switch (e->op) {
        case ExprOp::Add: op = "+"; break;
        case ExprOp::Mul: op = "*"; break;
        case ExprOp::Div: op = "/"; break;
        case ExprOp::Mod: op = "%"; break;
        case ExprOp::Shr: op = ">>"; break;
        case ExprOp::Shl: op = "<<"; break;
        case ExprOp::BitAnd: op = "&"; break;
        case ExprOp::BitOr: op = "|"; break;
        default: break;
    }
    return "(" + expr_token(e->lhs) + op + expr_token(e->rhs) + ")";
}

namespace {

std::string major_tok(Major m) { return m == Major::RowMajor ? "rowmajor" : "colmajor"; }

void print_chain(const NodePtr& node, std::string& out, int indent) {
    const std::string pad(static_cast<size_t>(indent) * 2, ' ');
    for (const DecompNode* n = node.get(); n; n = n->child.get()) {
        switch (n->kind) {
            case NodeKind::Tile: {
                std::string l = pad + "tile " + std::to_string(n->tile_r) + " " + std::to_string(n->tile_c);
                if (n->tile_ref.to) l += " .to " + lowercase(level_name(*n->tile_ref.to));
                if (n->tile_ref.layout) l += " .layout " + major_tok(*n->tile_ref.layout);
                if (n->tile_ref.swizzle) l += " .swizzle " + expr_token(n->tile_ref.swizzle);
                if (n->tile_ref.pair) l += " .pair";
                if (n->tile_ref.multicast) l += " .multicast";
                if (n->tile_ref.unroll) l += " .unroll";
                out += l + "\n";
                break;
            }
            case NodeKind::Split: {
                std::string l = pad + "split " + std::to_string(n->split_k);
                if (n->split_ref.unroll) l += " .unroll";
                if (n->split_ref.sync) l += " .sync";
                if (n->split_ref.double_buffer) l += " .doubleBufferLoop";
                else if (n->split_ref.stages > 0) l += " .stages " + std::to_string(n->split_ref.stages);
                if (n->split_ref.prefetch) l += " .prefetchLoads";
                if (n->split_ref.splitk) l += " .splitk";
                out += l + "\n";
                break;
            }
            case NodeKind::Load: {
                std::string l = pad + "load " + lowercase(operand_name(n->operand)) + " " +
                                lowercase(mem_name(n->target));
                if (n->load_ref.storage_layout) l += " .storagelayout " + major_tok(*n->load_ref.storage_layout);
                if (n->load_ref.pad > 0) l += " .pad " + std::to_string(n->load_ref.pad);
                if (n->load_ref.align) l += " .align " + std::to_string(*n->load_ref.align);
                if (n->load_ref.no_sync) l += " .nosync";
                if (n->load_ref.reuse_buffer) l += " .reusebuffer";
                if (n->load_ref.double_buffer) l += " .doubleBuffer";
                if (n->load_ref.postponed) l += " .postponed";
                out += l + " {\n";
                print_chain(n->move_decomp, out, indent + 1);
                out += pad + "}\n";
                break;
            }
            case NodeKind::Epilog:
                out += pad + "epilog " + lowercase(mem_name(n->acc_level)) + " {\n";
                out += pad + "  init {\n";
                print_chain(n->init_decomp, out, indent + 2);
                out += pad + "  }\n";
                out += pad + "  store {\n";
                print_chain(n->store_decomp, out, indent + 2);
                out += pad + "  }\n";
                out += pad + "}\n";
                break;
            case NodeKind::MmaTile: out += pad + "mmatile\n"; break;
            case NodeKind::Done:
                out += pad + "done" + (n->micro_kernel.empty() ? "" : " " + n->micro_kernel) + "\n";
                break;
        }
    }
}

}  // namespace

std::string print_script(const ParsedScript& script) {
    const Spec& root = script.root;
    std::string out = "spec " + spec_short_form(root);
    const bool mm = root.is_matmul();
    const bool default_elems = mm ? (root.mm().a.elem == ElemType::F32 && root.mm().b.elem == ElemType::F32 &&
                                     root.mm().c.elem == ElemType::F32)
                                  : root.mv().src.elem == ElemType::F32;
    const bool default_layouts =
        mm ? (root.mm().a.layout.major == Major::ColMajor && root.mm().b.layout.major == Major::ColMajor &&
              root.mm().c.layout.major == Major::ColMajor)
           : (root.mv().src.layout.major == Major::ColMajor && root.mv().dst.layout.major == Major::ColMajor);
    if (!default_elems) {
        out += " elems";
        if (mm)
            out += std::string(" ") + elem_name(root.mm().a.elem) + " " + elem_name(root.mm().b.elem) + " " +
                   elem_name(root.mm().c.elem);
        else
            out += std::string(" ") + elem_name(root.mv().src.elem) + " " + elem_name(root.mv().dst.elem);
    }
    if (!default_layouts) {
        out += " layouts";
        if (mm)
            out += " " + major_tok(root.mm().a.layout.major) + " " + major_tok(root.mm().b.layout.major) + " " +
                   major_tok(root.mm().c.layout.major);
        else
            out += " " + major_tok(root.mv().src.layout.major) + " " + major_tok(root.mv().dst.layout.major);
    }
    out += "\n";
    for (const auto& sec : script.micro_kernel_sections) {
        out += "\nmicrokernel " + sec.name + "\n";
        out += "pattern " + sec.pattern_line + "\n";
        if (!sec.vars.empty()) {
            out += "vars";
            for (const auto& v : sec.vars) out += " " + v;
            out += "\n";
        }
        out += "---\n" + sec.body + "---\n";
    }
    out += "\n";
    print_chain(script.tree, out, 0);
    return out;
}

void apply_size_overrides(ParsedScript& s, long m, long n, long k) {
    if (m <= 0 && n <= 0 && k <= 0) return;
    if (s.root.is_matmul()) {
        auto& o = s.root.mm();
        const long M = m > 0 ? m : s.root.m(), N = n > 0 ? n : s.root.n(), K = k > 0 ? k : s.root.k();
        o.a.rows = M;
        o.a.cols = K;
        o.b.rows = K;
        o.b.cols = N;
        o.c.rows = M;
        o.c.cols = N;
    } else {
        auto& o = s.root.mv();
        const long R = m > 0 ? m : o.src.rows, C = n > 0 ? n : o.src.cols;
        o.src.rows = o.dst.rows = R;
        o.src.cols = o.dst.cols = C;
    }
    MicroKernelSet rebuilt;
    for (const auto& sec : s.micro_kernel_sections) rebuilt.register_kernel(build_micro_kernel(sec, s.root));
    s.micro_kernels = std::move(rebuilt);
}

}  // namespace fireiron
