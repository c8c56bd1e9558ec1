// Host matrices, reproducible generators, grid rounding and digests.
// Bit-compatible with proj/include/anvil/matrix.hpp:15-133 (splitmix64 stream
// in logical row-major draw order, FNV-1a digest over fp32 bits).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "fireiron/types.hpp"

namespace fireiron {

struct Matrix {
    long rows = 0, cols = 0;
    Layout layout;
    std::vector<float> data;

    static Matrix zeros(long r, long c, Layout l = Layout::col_major());
    long linear(long r, long c) const {
        return r * layout.row_stride(rows, cols) + c * layout.col_stride(rows, cols);
    }
    float at(long r, long c) const { return data[static_cast<size_t>(linear(r, c))]; }
    float& at(long r, long c) { return data[static_cast<size_t>(linear(r, c))]; }
};

struct Rng {
    uint64_t state;
    explicit Rng(uint64_t seed) : state(seed) {}
    uint64_t next();
};

void fill_integers(Matrix& m, uint64_t seed, long lo = -3, long hi = 3);
void fill_uniform(Matrix& m, uint64_t seed);

float round_to_f16(float x);   // reference semantics (saturating above 65504)
float round_to_bf16(float x);  // IEEE round-to-nearest-even
void round_matrix_to_f16(Matrix& m);
void round_matrix(Matrix& m, ElemType e);

uint64_t digest(const Matrix& m);
Matrix read_matrix(const std::string& path, Layout layout = Layout::col_major());
void write_matrix(const std::string& path, const Matrix& m);

}  // namespace fireiron
