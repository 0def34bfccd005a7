#include "packages.hpp"

#include <algorithm>
#include <string>

#include "errors.hpp"

namespace sdb {

F4Mat to_gf4(const BitMat &m) {
    if (m.cols % 2 != 0) throw InvalidArgument("to_gf4: column count must be even");
    const int n = m.cols / 2;
    F4Mat out{BitMat(m.rows, n), BitMat(m.rows, n)};
    for (int r = 0; r < m.rows; r++)
        for (int c = 0; c < n; c++) {
            if (m.get(r, c)) out.a.set(r, c, true);
            if (m.get(r, n + c)) out.b.set(r, c, true);
        }
    return out;
}

BitMat to_gf2(const F4Mat &m) {
    const int n = m.cols();
    BitMat out(m.rows(), 2 * n);
    for (int r = 0; r < m.rows(); r++)
        for (int c = 0; c < n; c++) {
            if (m.a.get(r, c)) out.set(r, c, true);
            if (m.b.get(r, c)) out.set(r, n + c, true);
        }
    return out;
}

namespace {

void swap_cols(BitMat &m, int c1, int c2) {
    if (c1 == c2) return;
    for (int r = 0; r < m.rows; r++) {
        const bool x = m.get(r, c1), y = m.get(r, c2);
        if (x != y) {
            m.set(r, c1, y);
            m.set(r, c2, x);
        }
    }
}

void append_row(BitMat &m, const uint64_t *src) {
    m.w.insert(m.w.end(), src, src + m.stride);
    m.rows++;
}

// One F4 pivot: a column and its one or two pivot rows (reference F4Pivot, prep.cpp:20-24).
struct F4Pivot {
    int col, r1, r2;
};

// Shared core of both F4 diagonalizations (reference f4_diagonalize_core,
// prep.cpp:31-106): columns in the given order; two distinct nonzero symbols among
// unprocessed rows pivot both rows and clear the column everywhere else, a single symbol x
// pivots one row and reduces the rest of the column to {0, y}.
struct F4Core {
    F4Mat m;
    std::vector<F4Pivot> pivots;
    std::vector<char> processed;
};

F4Core f4_core(F4Mat m, const std::vector<int> &order) {
    const int rows = m.rows();
    F4Core out;
    out.processed.assign(size_t(rows), 0);
    int done = 0;
    for (int c : order) {
        if (done == rows) break;
        int i1 = -1, i2 = -1;
        for (int i = 0; i < rows; i++) {
            if (out.processed[size_t(i)]) continue;
            const unsigned s = m.get(i, c);
            if (!s) continue;
            if (i1 < 0) {
                i1 = i;
            } else if (s != m.get(i1, c)) {
                i2 = i;
                break;
            }
        }
        if (i1 < 0) continue;  // principal candidate
        if (i2 >= 0) {
            const unsigned s1 = m.get(i1, c), s2 = m.get(i2, c);
            for (int q = 0; q < rows; q++) {
                if (q == i1 || q == i2) continue;
                const unsigned e = m.get(q, c);
                if (!e) continue;
                if (e == s1) {
                    m.add_row_into(i1, q);
                } else if (e == s2) {
                    m.add_row_into(i2, q);
                } else {
                    m.add_row_into(i1, q);
                    m.add_row_into(i2, q);
                }
            }
            out.processed[size_t(i1)] = out.processed[size_t(i2)] = 1;
            done += 2;
            out.pivots.push_back({c, i1, i2});
        } else {
            const unsigned x = m.get(i1, c);
            unsigned y = 0;
            for (int q = 0; q < rows; q++) {
                if (q == i1) continue;
                const unsigned e = m.get(q, c);
                if (e && e != x) {
                    y = e;
                    break;
                }
            }
            for (int q = 0; q < rows; q++) {
                if (q == i1) continue;
                const unsigned e = m.get(q, c);
                if (!e || e == y) continue;
                m.add_row_into(i1, q);
            }
            out.processed[size_t(i1)] = 1;
            done += 1;
            out.pivots.push_back({c, i1, -1});
        }
    }
    out.m = std::move(m);
    return out;
}

// Drop zero rows, append each 3-package's sum row, build the packages over F2
// (reference assemble_f4_gamma, prep.cpp:108-151).
Packaged assemble(F4Core core) {
    const int rows = core.m.rows(), n = core.m.cols();
    for (int r = 0; r < rows; r++)
        if (!core.processed[size_t(r)] && !core.m.row_is_zero(r))
            throw InternalFailure("f4 diagonalization left a nonzero unprocessed row");
    std::vector<int> remap(size_t(rows), -1);
    F4Mat kept{BitMat(0, n), BitMat(0, n)};
    for (int r = 0; r < rows; r++) {
        if (core.m.row_is_zero(r)) continue;
        append_row(kept.a, core.m.a.row(r));
        append_row(kept.b, core.m.b.row(r));
        remap[size_t(r)] = kept.rows() - 1;
    }
    Packaged g;
    for (const F4Pivot &p : core.pivots) {
        if (p.r2 < 0) {
            g.packages.push_back({remap[size_t(p.r1)]});
        } else {
            const int m1 = remap[size_t(p.r1)], m2 = remap[size_t(p.r2)];
            std::vector<uint64_t> sa(kept.a.row(m1), kept.a.row(m1) + kept.a.stride),
                sb(kept.b.row(m1), kept.b.row(m1) + kept.b.stride);
            for (int w = 0; w < kept.a.stride; w++) {
                sa[size_t(w)] ^= kept.a.row(m2)[w];
                sb[size_t(w)] ^= kept.b.row(m2)[w];
            }
            append_row(kept.a, sa.data());
            append_row(kept.b, sb.data());
            g.packages.push_back({m1, m2, kept.rows() - 1});
        }
        g.pivots.push_back(p.col);
    }
    g.pair_count = n;
    g.matrix = to_gf2(kept);
    g.n_pp = int(g.packages.size());
    return g;
}

}  // namespace

Packaged diagonalize_f2(const BitMat &a) {
    if (a.cols % 2 != 0) throw InvalidArgument("diagonalize_f2: column count must be even");
    const int n = a.cols / 2, rows = a.rows;
    if (rows < n || rows > 2 * n) throw ValidationFailure("diagonalize_f2: row count must lie between n and 2n");
    BitMat b = a;
    // identity on the first half, with paired column permutations and half swaps only
    for (int p = 0; p < n; p++) {
        int pj = n, ph = 0, pi = rows;
        for (int j = p; j < n && pj == n; j++)
            for (int h = 0; h < 2 && pj == n; h++) {
                const int col = h == 0 ? j : n + j;
                for (int i = p; i < rows; i++)
                    if (b.get(i, col)) {
                        pj = j;
                        ph = h;
                        pi = i;
                        break;
                    }
            }
        if (pj == n)
            throw ValidationFailure(
                "diagonalize_f2: systematic form unreachable; matrix is rank-deficient or not a valid normalizer");
        if (pj != p) {
            swap_cols(b, p, pj);
            swap_cols(b, n + p, n + pj);
        }
        if (ph == 1) swap_cols(b, p, n + p);
        if (pi != p) b.swap_rows(p, pi);
        for (int i = 0; i < rows; i++)
            if (i != p && b.get(i, p)) b.xor_into(i, p);
    }
    // bottom rows: echelon on the second half, each pivot column cleared everywhere else
    const int k = rows - n;
    std::vector<int> m2;
    int r = n;
    for (int c = 0; c < n && r < rows; c++) {
        int sel = rows;
        for (int i = r; i < rows; i++)
            if (b.get(i, n + c)) {
                sel = i;
                break;
            }
        if (sel == rows) continue;
        b.swap_rows(r, sel);
        for (int i = 0; i < rows; i++)
            if (i != r && b.get(i, n + c)) b.xor_into(i, r);
        m2.push_back(c);
        r++;
    }
    if (int(m2.size()) != k) throw ValidationFailure("diagonalize_f2: rows are linearly dependent");
    Packaged g;
    g.packages.assign(size_t(n), {});
    g.pivots.resize(size_t(n));
    for (int i = 0; i < k; i++) {
        const int j = m2[size_t(i)];
        std::vector<uint64_t> sum(b.row(j), b.row(j) + b.stride);
        for (int w = 0; w < b.stride; w++) sum[size_t(w)] ^= b.row(n + i)[w];
        append_row(b, sum.data());
        g.packages[size_t(j)] = {j, n + i, rows + i};
    }
    for (int j = 0; j < n; j++) {
        if (g.packages[size_t(j)].empty()) g.packages[size_t(j)] = {j};
        g.pivots[size_t(j)] = j;
    }
    g.matrix = std::move(b);
    g.pair_count = n;
    g.n_pp = n;
    return g;
}

std::pair<Packaged, std::vector<int>> diagonalize_f4(const F4Mat &a4) {
    const int n = a4.cols();
    std::vector<int> order;
    for (int c = 0; c < n; c++) order.push_back(c);
    F4Core core = f4_core(a4, order);
    std::vector<char> pivoted(size_t(n), 0);
    for (const F4Pivot &p : core.pivots) pivoted[size_t(p.col)] = 1;
    std::vector<int> principal;
    for (int c = 0; c < n; c++)
        if (!pivoted[size_t(c)]) principal.push_back(c);
    Packaged g = assemble(std::move(core));
    if (rank(g.matrix) != a4.rows()) throw ValidationFailure("diagonalize_f4: rows are linearly dependent");
    return {std::move(g), std::move(principal)};
}

Packaged second_gamma(const F4Mat &b4, const std::vector<int> &principal) {
    const int n = b4.cols();
    std::vector<char> is_principal(size_t(n), 0);
    for (int c : principal) is_principal[size_t(c)] = 1;
    std::vector<int> order(principal);
    for (int c = 0; c < n; c++)
        if (!is_principal[size_t(c)]) order.push_back(c);
    Packaged g = assemble(f4_core(b4, order));
    g.n_pp = 0;
    for (int p : g.pivots)
        if (p >= 0 && is_principal[size_t(p)]) g.n_pp++;
    return g;
}

}  // namespace sdb
