// Host prep of the package routes: Saved_1_Gamma's constrained
// F2 diagonalization and Saved_2_Gamma's two F4 diagonalizations, with the reference's pivot
// rules so the packages — and therefore the bound traces — are the reference's bit for bit.
#pragma once

#include <utility>
#include <vector>

#include "gf2.hpp"

namespace sdb {

// One generator matrix with its package partition (reference PackagedGamma,
// prep.hpp:25-35): packages[i] lists the member rows of package i (1 or 3 rows),
// pivots[i] its pivot column (-1 for none).
struct Packaged {
    BitMat matrix;
    std::vector<std::vector<int>> packages;
    std::vector<int> pivots;
    int pair_count = 0;
    int n_pp = 0;
    int rank_deficit = 0;
};

// Additive code over F4 as two bit planes: symbol (r, c) = plane_a(r, c) + alpha plane_b(r, c)
// (reference gf4.hpp:17-56; an F2 row (a | b) is the F4 row a + alpha b).
struct F4Mat {
    BitMat a, b;  // rows x n each
    int rows() const { return a.rows; }
    int cols() const { return a.cols; }
    unsigned get(int r, int c) const { return unsigned(a.get(r, c)) | (unsigned(b.get(r, c)) << 1); }
    void add_row_into(int src, int dst) {
        a.xor_into(dst, src);
        b.xor_into(dst, src);
    }
    bool row_is_zero(int r) const { return a.row_is_zero(r) && b.row_is_zero(r); }
};

F4Mat to_gf4(const BitMat &m);     // (a | b) -> a + alpha b       (gf4.cpp:37-51)
BitMat to_gf2(const F4Mat &m);     // exact inverse                 (gf4.cpp:53-63)

// diagonalize_f2 (prep.cpp:155-254): (I_n | M1 over 0 | M2), k appended rows completing the
// 3-packages, one package per coordinate pair.
Packaged diagonalize_f2(const BitMat &a);

// diagonalize_f4 (prep.cpp:256-276): F4 diagonalization in column order; also returns the
// principal (unpivoted) columns.
std::pair<Packaged, std::vector<int>> diagonalize_f4(const F4Mat &a4);

// second_gamma (prep.cpp:278-297): principal columns first; n_pp = packages pivoted on them.
Packaged second_gamma(const F4Mat &b4, const std::vector<int> &principal);

}  // namespace sdb
