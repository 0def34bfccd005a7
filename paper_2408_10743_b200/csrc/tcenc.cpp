// Coordinate encoding of the tensor-core tile kernel (device.hpp: TcPlan).
//
// A candidate is a set S of rows of one Gamma, split into a head S_h and a tail S_t. Its
// symplectic weight popc(x|z) counts the symbols s with (x_s, z_s) != 0. Per symbol, look at
// the three columns a_s, b_s, (a^b)_s of the matrix:
//   * unit column (exactly one row p has a 1 there): the column of a combination is [p in S],
//     so the symbol is nonzero iff p in S or its other independent component c_s (b for a
//     pivot on a, a otherwise) is odd:   [nz] = [p in S] + [p not in S] (1 - s_h s_t) / 2
//     with s = +-1 the sign of c_s over S_h / S_t. Since p lies in at most one of S_h, S_t,
//     [p not in S] s_h s_t = (masked s_h)(masked s_t), a side's value zeroed when that side
//     holds p. One coordinate, coefficient S/2, plus alpha [p in S] split into c_h + c_t.
//   * no unit column: [nz] = (3 - s_a - s_b - s_ab) / 4, three coordinates, coefficient 1
//     (needs S = 4).
//   * all three columns zero: never nonzero, no coordinate.
// Each row masks at most one coordinate (a row already used as a mask leaves the symbol to
// another unit column or to the three-coordinate form), so c = alpha * |S ∩ mask rows|.
// The head carries -s (bytes +-1), the tail v * s (v = S/2 on unit-column coordinates, 1
// elsewhere); a tail's coordinate kc carries -c_t against the head's constant -1; padding
// coordinates contribute -v each, returned in C0:
//     S * popc(x|z) = C0 + c_h + sum_k head_k tail_k.
// On the isometry route every symbol of Gamma_1 / Gamma_2 has a pivot (information_sets puts
// n + k pivots on n symbols), so K = n + 1 rounded up to 32: config 4 needs 64 coordinates for
// Gamma_1, Gamma_2 and 96 for Gamma_3, config 5 96 and 128.
#include "tcenc.hpp"

#include <algorithm>
#include <random>

namespace sdb {

namespace {

// coordinate k of a 32-coordinate word lives at bit 8 i + j with k % 32 = 4 j + i, so that
// (word >> j) & 0x01010101 gives the bytes of coordinates 4j..4j+3
inline int coord_bit(int k) {
    const int q = k & 31;
    return 8 * (q & 3) + (q >> 2);
}

struct ColumnSet {
    int N = 0, words = 0;
    std::vector<uint64_t> bits;  // [3 * n][words]: a_s, b_s, (a^b)_s over the rows
};

ColumnSet columns_of(const BitMat &m, int N, int n, bool image) {
    ColumnSet c;
    c.N = N;
    c.words = (N + 63) / 64;
    c.bits.assign(size_t(3) * n * c.words, 0);
    // transpose by visiting set bits only: column (type, s) of the a, b and a^b blocks
    for (int r = 0; r < m.rows && r < N; r++) {
        const uint64_t *row = m.row(r);
        const uint64_t bit = uint64_t(1) << (r & 63);
        const int ncols = image ? 3 * n : 2 * n;
        for (int w = 0; w * 64 < ncols; w++) {
            uint64_t x = row[w];
            if (64 * w + 64 > ncols) x &= (uint64_t(1) << (ncols - 64 * w)) - 1;
            while (x) {
                const int col = 64 * w + __builtin_ctzll(x);
                x &= x - 1;
                c.bits[size_t(col) * c.words + (r >> 6)] |= bit;  // col = type * n + s
            }
        }
    }
    if (!image)  // the a^b column from a and b
        for (int s = 0; s < n; s++)
            for (int i = 0; i < c.words; i++)
                c.bits[(size_t(2) * n + s) * c.words + i] =
                    c.bits[size_t(s) * c.words + i] ^ c.bits[(size_t(n) + s) * c.words + i];
    return c;
}

}  // namespace

TcEncoding tc_encode(const std::vector<const BitMat *> &mats, int N, int n, bool image) {
    TcEncoding enc;
    const int G = int(mats.size());
    struct Coord {
        int type;   // 0: a, 1: b, 2: a^b (the column whose bits are the sign)
        int sym;
        int mask_row;  // -1: none
    };
    std::vector<std::vector<Coord>> c1(static_cast<size_t>(G)), c3(static_cast<size_t>(G));
    enc.kmax = 32;
    std::vector<ColumnSet> cols(static_cast<size_t>(G));
    for (int j = 0; j < G; j++) cols[size_t(j)] = columns_of(*mats[size_t(j)], N, n, image);
    for (int j = 0; j < G; j++) {
        const ColumnSet &cs = cols[size_t(j)];
        auto col = [&](int type, int s) { return cs.bits.data() + (size_t(type) * n + s) * cs.words; };
        auto weight = [&](int type, int s) {
            int w = 0;
            for (int i = 0; i < cs.words; i++) w += __builtin_popcountll(col(type, s)[i]);
            return w;
        };
        auto first_row = [&](int type, int s) {
            for (int i = 0; i < cs.words; i++)
                if (col(type, s)[i]) return 64 * i + __builtin_ctzll(col(type, s)[i]);
            return -1;
        };
        std::vector<char> used(size_t(N), 0);
        for (int s = 0; s < n; s++) {
            int unit_type = -1, p = -1;
            for (int type = 0; type < 3 && unit_type < 0; type++)
                if (weight(type, s) == 1) {
                    const int r = first_row(type, s);
                    if (!used[size_t(r)]) {
                        unit_type = type;
                        p = r;
                    }
                }
            if (unit_type >= 0) {
                used[size_t(p)] = 1;
                c1[size_t(j)].push_back(Coord{unit_type == 0 ? 1 : 0, s, p});
            } else if (weight(0, s) || weight(1, s)) {
                c3[size_t(j)].push_back(Coord{0, s, -1});
            }
        }
    }
    // layout per Gamma
    std::vector<std::vector<Coord>> layout(static_cast<size_t>(G));  // type -1: padding / constant
    enc.gam.assign(size_t(G), TcGammaDev{});
    for (int j = 0; j < G; j++) {
        TcGammaDev &gm = enc.gam[size_t(j)];
        const int n1 = int(c1[size_t(j)].size()), n0 = int(c3[size_t(j)].size());
        gm.S = n0 > 0 ? 4 : 2;
        gm.alpha = gm.S / 2;
        std::vector<Coord> &L = layout[size_t(j)];
        int pad_v = 0;  // sum of the padding coordinates' tail coefficients
        for (const Coord &c : c1[size_t(j)]) L.push_back(c);
        if (gm.S == 4) {
            while (L.size() % 4) {
                L.push_back(Coord{-1, -1, -1});
                pad_v += 2;
            }
            gm.W1 = int(L.size()) / 4;
            for (const Coord &c : c3[size_t(j)])
                for (int type = 0; type < 3; type++) L.push_back(Coord{type, c.sym, -1});
        } else {
            gm.W1 = 0;  // every tail coefficient is 1
        }
        gm.kc = int(L.size());
        L.push_back(Coord{-1, -1, -1});
        gm.kt = int(L.size());  // two threshold coordinates (not padding: they carry -(T + 1))
        L.push_back(Coord{-1, -1, -1});
        L.push_back(Coord{-1, -1, -1});
        while (L.size() % 32) {
            L.push_back(Coord{-1, -1, -1});
            pad_v += 1;
        }
        gm.K = int(L.size());
        gm.C0 = n1 * gm.alpha + 3 * n0 + pad_v;
        enc.kmax = std::max(enc.kmax, gm.K);
    }
    enc.ok = enc.kmax <= kTcMaxK;
    if (!enc.ok) return enc;
    enc.kw = enc.kmax / 32;
    enc.sign.assign(size_t(G) * N * enc.kw, 0);
    enc.mask.assign(size_t(G) * N, -1);
    for (int j = 0; j < G; j++) {
        const ColumnSet &cs = cols[size_t(j)];
        const std::vector<Coord> &L = layout[size_t(j)];
        for (int k = 0; k < int(L.size()); k++) {
            const Coord &c = L[size_t(k)];
            if (c.type < 0) continue;
            const uint64_t *colw = cs.bits.data() + (size_t(c.type) * n + c.sym) * cs.words;
            for (int i = 0; i < cs.words; i++)
                for (uint64_t x = colw[i]; x; x &= x - 1) {
                    const int r = 64 * i + __builtin_ctzll(x);
                    if (r < N) enc.sign[(size_t(j) * N + r) * enc.kw + k / 32] |= uint32_t(1) << coord_bit(k);
                }
            if (c.mask_row >= 0) enc.mask[size_t(j) * N + c.mask_row] = short(k);
        }
    }
    return enc;
}

int tc_selfcheck(const TcEncoding &enc, const std::vector<const BitMat *> &mats, int N, int n, bool image,
                 uint64_t seed, int trials) {
    if (!enc.ok) return -1;
    std::mt19937_64 rng(seed);
    int bad = 0;
    const int G = int(mats.size());
    for (int j = 0; j < G; j++) {
        const TcGammaDev &gm = enc.gam[size_t(j)];
        const BitMat &m = *mats[size_t(j)];
        for (int tr = 0; tr < trials; tr++) {
            // a random subset, split at random into head and tail (any split satisfies the identity)
            std::vector<int> head, tail;
            const int density = 1 + int(rng() % 8);
            for (int r = 0; r < N; r++)
                if (rng() % 16 < unsigned(density)) (rng() & 1 ? head : tail).push_back(r);
            // true weight
            int w = 0;
            for (int s = 0; s < n; s++) {
                bool a = false, b = false;
                for (int r : head) a ^= r < m.rows && m.get(r, s), b ^= r < m.rows && m.get(r, n + s);
                for (int r : tail) a ^= r < m.rows && m.get(r, s), b ^= r < m.rows && m.get(r, n + s);
                w += a || b;
            }
            // operand bytes as the kernel builds them
            auto bytes = [&](const std::vector<int> &rows, bool is_head, int &cnt) {
                std::vector<int8_t> v(size_t(gm.K));
                std::vector<uint32_t> sw(size_t(enc.kw), 0);
                cnt = 0;
                for (int r : rows) {
                    for (int w2 = 0; w2 < enc.kw; w2++) sw[size_t(w2)] ^= enc.sign[(size_t(j) * N + r) * enc.kw + w2];
                    cnt += enc.mask[size_t(j) * N + r] >= 0;
                }
                for (int k = 0; k < gm.K; k++) {
                    const bool bit = (sw[size_t(k / 32)] >> coord_bit(k)) & 1;
                    const int v1 = gm.S == 4 && k / 4 < gm.W1 ? 2 : 1;
                    v[size_t(k)] = int8_t(is_head ? (bit ? 1 : -1) : (bit ? -v1 : v1));
                }
                for (int r : rows) {
                    const int c = enc.mask[size_t(j) * N + r];
                    if (c >= 0) v[size_t(c)] = 0;
                }
                if (!is_head) v[size_t(gm.kc)] = int8_t(-(gm.alpha * cnt));
                v[size_t(gm.kt)] = v[size_t(gm.kt + 1)] = 0;
                return v;
            };
            int ch = 0, ct = 0;
            std::vector<int8_t> hv = bytes(head, true, ch), tv = bytes(tail, false, ct);
            int acc = 0;
            for (int k = 0; k < gm.K; k++) acc += int(hv[size_t(k)]) * int(tv[size_t(k)]);
            if (gm.S * w != gm.C0 + gm.alpha * ch + acc) bad++;
            // the threshold fold: with T = S thr - C0 - ch in the head's kt bytes and 1, 16 in
            // the tail's, the accumulator is negative iff w <= thr
            const int thr = w + int(rng() % 5) - 2;
            int r = 0, q = 0;
            tc_threshold_bytes(gm.S * thr - gm.C0 - gm.alpha * ch, r, q);
            hv[size_t(gm.kt)] = int8_t(r);
            hv[size_t(gm.kt + 1)] = int8_t(q);
            tv[size_t(gm.kt)] = 1;
            tv[size_t(gm.kt + 1)] = 16;
            int acc2 = 0;
            for (int k = 0; k < gm.K; k++) acc2 += int(hv[size_t(k)]) * int(tv[size_t(k)]);
            if ((acc2 < 0) != (w <= thr) || int(int16_t(acc2)) != acc2) bad++;
        }
    }
    (void)image;
    return bad;
}

}  // namespace sdb
