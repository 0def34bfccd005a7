// Host-side GF(2) prep for the isometry route: packed matrices, the BASELINE code
// generator, validation, isometry_transform and information_sets. Word-level
// (64 columns per XOR) restatements of the reference's per-bit routines; the pivot
// rules are kept identical so the Gamma_j — and therefore the bound trace — match
// bit for bit.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sdb {

struct BitMat {
    int rows = 0, cols = 0, stride = 0;  // stride: u64 words per row
    std::vector<uint64_t> w;

    BitMat() = default;
    BitMat(int r, int c) : rows(r), cols(c), stride((c + 63) / 64), w(size_t(r) * size_t((c + 63) / 64), 0) {}

    uint64_t *row(int r) { return w.data() + size_t(r) * stride; }
    const uint64_t *row(int r) const { return w.data() + size_t(r) * stride; }
    bool get(int r, int c) const { return (row(r)[c >> 6] >> (c & 63)) & 1u; }
    void set(int r, int c, bool v) {
        uint64_t m = uint64_t(1) << (c & 63);
        if (v) row(r)[c >> 6] |= m; else row(r)[c >> 6] &= ~m;
    }
    void xor_into(int dst, int src) {
        uint64_t *d = row(dst);
        const uint64_t *s = row(src);
        for (int i = 0; i < stride; i++) d[i] ^= s[i];
    }
    void swap_rows(int a, int b) {
        if (a == b) return;
        uint64_t *x = row(a), *y = row(b);
        for (int i = 0; i < stride; i++) std::swap(x[i], y[i]);
    }
    bool row_is_zero(int r) const {
        const uint64_t *x = row(r);
        for (int i = 0; i < stride; i++)
            if (x[i]) return false;
        return true;
    }
    // from caller words (row_words stride); padding beyond cols is masked off
    static BitMat from_words(const uint64_t *src, int rows, int cols, int row_words);
    void to_words(uint64_t *dst, int row_words) const;
    std::string row_string(int r) const;
};

// Gaussian elimination to reduced row echelon form in place, pivots ascending
// (bitvec.cpp:213-233 echelonize); returns pivot columns.
std::vector<int> echelonize(BitMat &m);
int rank(const BitMat &m);
// Basis of the Euclidean kernel in the reference's construction order (bitvec.cpp:242-259).
BitMat null_space(const BitMat &m);

struct Validation {
    bool ok = true;
    std::string message;
};
// validate_normalizer (distance.cpp:71-93), same checks and messages.
Validation validate_normalizer(const BitMat &a);

// isometry_transform (prep.cpp:299-315): row (a|b) -> (a|b|a^b).
BitMat isometry_transform(const BitMat &a);

struct InfoSet {
    BitMat matrix;
    int rank_deficit = 0;
    std::vector<int> pivots;  // per row, -1 past the pivots found
};
// information_sets (prep.cpp:317-364); throws ValidationError-equivalent on rank loss.
std::vector<InfoSet> information_sets(const BitMat &b);

// BASELINE.md §2 generator (xorshift64* transvections on the canonical generators).
BitMat generate_code(int n, int k, uint64_t seed, int transvections);

// random_stabilizer (distance.cpp:242-294): mt19937_64(seed) grows a self-orthogonal C, the
// normalizer is a basis of its symplectic dual. Same draws, same null-space order.
BitMat random_stabilizer(int n, int k, uint64_t seed);

// Matrix text format (matrix_io.cpp:26-106): "K N" header, K rows of N characters '0'/'1';
// whitespace inside rows and blank lines ignored. Throws ParseFailure with the reference's
// "origin:line: what" diagnostics.
BitMat parse_matrix_text(const std::string &text, const std::string &origin);
std::string format_matrix(const BitMat &m);

// <u,v>_s over the first 2n columns of both (n = pair count).
int symplectic_ip(const uint64_t *u, const uint64_t *v, int n);

}  // namespace sdb
