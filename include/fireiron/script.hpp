// Strategy script front-end (.fi text <-> Spec + tree + micro-kernels).
// Grammar and canonical printing follow proj/include/anvil/script.hpp:38-793;
// additions for sm_100a: elem "bf16", mem "tm", tile ".pair", split
// ".stages N" and ".splitk". parse(print(s)) == s for canonical scripts.
#pragma once

#include <string>
#include <vector>

#include "fireiron/decomp.hpp"

namespace fireiron {

Spec parse_spec_short_form(const std::string& text, const Spec* basis = nullptr, int line = 0);

struct MicroKernelSection {
    std::string name;
    std::string pattern_line;
    std::vector<std::string> vars;
    std::string body;
    int line = 0;
};

struct ParsedScript {
    Spec root;
    NodePtr tree;
    MicroKernelSet micro_kernels;
    std::vector<MicroKernelSection> micro_kernel_sections;
};

ParsedScript parse_script(const std::string& text);
std::string print_script(const ParsedScript& script);

// The anvil CLI --m/--n/--k override (tools/anvil.cpp:29-60): re-derives the
// root dims and rebuilds micro-kernel patterns that reference M/N/K.
void apply_size_overrides(ParsedScript& script, long m, long n, long k);

// Swizzle token rendering (space free; reparses to the same tree).
std::string expr_token(const Expr& e);

}  // namespace fireiron
