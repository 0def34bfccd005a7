#include "gf2.hpp"

#include <algorithm>
#include <cctype>
#include <random>
#include <sstream>
#include <stdexcept>

#include "errors.hpp"

namespace sdb {

BitMat BitMat::from_words(const uint64_t *src, int rows, int cols, int row_words) {
    BitMat m(rows, cols);
    const int copy = std::min(row_words, m.stride);
    for (int r = 0; r < rows; r++) {
        for (int i = 0; i < copy; i++) m.row(r)[i] = src[size_t(r) * row_words + i];
        if (cols & 63) m.row(r)[m.stride - 1] &= (~uint64_t(0)) >> (64 - (cols & 63));
    }
    return m;
}

void BitMat::to_words(uint64_t *dst, int row_words) const {
    for (int r = 0; r < rows; r++)
        for (int i = 0; i < row_words; i++) dst[size_t(r) * row_words + i] = i < stride ? row(r)[i] : 0;
}

std::string BitMat::row_string(int r) const {
    std::string s(size_t(cols), '0');
    for (int c = 0; c < cols; c++)
        if (get(r, c)) s[size_t(c)] = '1';
    return s;
}

std::vector<int> echelonize(BitMat &m) {
    std::vector<int> pivots;
    int r = 0;
    for (int c = 0; c < m.cols && r < m.rows; c++) {
        const int wi = c >> 6;
        const uint64_t bit = uint64_t(1) << (c & 63);
        int sel = -1;
        for (int i = r; i < m.rows; i++)
            if (m.row(i)[wi] & bit) { sel = i; break; }
        if (sel < 0) continue;
        m.swap_rows(r, sel);
        for (int i = 0; i < m.rows; i++)
            if (i != r && (m.row(i)[wi] & bit)) m.xor_into(i, r);
        pivots.push_back(c);
        r++;
    }
    return pivots;
}

int rank(const BitMat &m) {
    BitMat c = m;
    return int(echelonize(c).size());
}

BitMat null_space(const BitMat &m) {
    BitMat ech = m;
    const std::vector<int> pivots = echelonize(ech);
    std::vector<char> is_pivot(size_t(m.cols), 0);
    for (int c : pivots) is_pivot[size_t(c)] = 1;
    BitMat basis(m.cols - int(pivots.size()), m.cols);
    int out = 0;
    for (int f = 0; f < m.cols; f++) {
        if (is_pivot[size_t(f)]) continue;
        basis.set(out, f, true);
        for (size_t r = 0; r < pivots.size(); r++)
            if (ech.get(int(r), f)) basis.set(out, pivots[r], true);
        out++;
    }
    return basis;
}

// 64 bits of row r from column `from` on (zero past the row)
static inline uint64_t bits64(const BitMat &m, int r, int from) {
    const uint64_t *w = m.row(r);
    const int wi = from >> 6, sh = from & 63;
    const uint64_t lo = wi < m.stride ? w[wi] : 0, hi = (sh && wi + 1 < m.stride) ? w[wi + 1] : 0;
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

// OR `len` bits of v (low bits first) into row r at column `at`
static inline void or_bits(BitMat &m, int r, int at, uint64_t v, int len) {
    if (len < 64) v &= (uint64_t(1) << len) - 1;
    uint64_t *w = m.row(r);
    const int wi = at >> 6, sh = at & 63;
    w[wi] |= v << sh;
    if (sh && wi + 1 < m.stride) w[wi + 1] |= v >> (64 - sh);
}

static BitMat swap_halves(const BitMat &a) {
    const int n = a.cols / 2;
    BitMat s(a.rows, a.cols);
    for (int r = 0; r < a.rows; r++)
        for (int i = 0; i < n; i += 64) {
            const int len = std::min(64, n - i);
            or_bits(s, r, i, bits64(a, r, n + i), len);
            or_bits(s, r, n + i, bits64(a, r, i), len);
        }
    return s;
}

Validation validate_normalizer(const BitMat &a) {
    const int rows = a.rows;
    const int n = a.cols / 2;
    const int k = rows - n;
    if (rows == 0) return {false, "matrix has no rows"};
    if (k < 0) return {false, "matrix has fewer rows than n; a normalizer needs n+k >= n rows"};
    if (rows > 2 * n) return {false, "matrix has more rows than columns; rows cannot be independent"};
    if (rank(a) != rows) return {false, "rows are linearly dependent (rank below n+k)"};
    const BitMat dual = null_space(swap_halves(a));
    BitMat ech = a;
    const std::vector<int> pivots = echelonize(ech);
    std::vector<uint64_t> res(size_t(a.stride));
    for (int r = 0; r < dual.rows; r++) {
        std::copy(dual.row(r), dual.row(r) + dual.stride, res.begin());
        for (size_t p = 0; p < pivots.size(); p++)
            if ((res[size_t(pivots[p] >> 6)] >> (pivots[p] & 63)) & 1u)
                for (int i = 0; i < a.stride; i++) res[size_t(i)] ^= ech.row(int(p))[i];
        bool zero = true;
        for (uint64_t x : res) zero = zero && x == 0;
        if (!zero)
            return {false, "not a stabilizer normalizer: dual vector " + dual.row_string(r) +
                               " lies outside the rowspace"};
    }
    return {true, ""};
}

BitMat isometry_transform(const BitMat &a) {
    if (a.cols % 2 != 0) throw InvalidArgument("isometry_transform: column count must be even");
    const int n = a.cols / 2;
    BitMat out(a.rows, 3 * n);
    for (int r = 0; r < a.rows; r++)
        for (int i = 0; i < n; i += 64) {
            const int len = std::min(64, n - i);
            const uint64_t x = bits64(a, r, i), z = bits64(a, r, n + i);
            or_bits(out, r, i, x, len);
            or_bits(out, r, n + i, z, len);
            or_bits(out, r, 2 * n + i, x ^ z, len);
        }
    return out;
}

std::vector<InfoSet> information_sets(const BitMat &b) {
    const int n_rows = b.rows, n_cols = b.cols;
    if (rank(b) != n_rows) throw ValidationFailure("information_sets: rows are linearly dependent");
    std::vector<char> used(size_t(n_cols), 0);
    std::vector<InfoSet> out;
    BitMat cur = b;
    for (;;) {
        std::vector<int> pivot_cols;
        int r = 0;
        for (int c = 0; c < n_cols && r < n_rows; c++) {
            if (used[size_t(c)]) continue;
            const int wi = c >> 6;
            const uint64_t bit = uint64_t(1) << (c & 63);
            int sel = -1;
            for (int i = r; i < n_rows; i++)
                if (cur.row(i)[wi] & bit) { sel = i; break; }
            if (sel < 0) continue;
            cur.swap_rows(r, sel);
            for (int i = 0; i < n_rows; i++)
                if (i != r && (cur.row(i)[wi] & bit)) cur.xor_into(i, r);
            pivot_cols.push_back(c);
            r++;
        }
        if (pivot_cols.empty()) break;
        InfoSet is;
        is.matrix = cur;
        is.rank_deficit = n_rows - int(pivot_cols.size());
        is.pivots.assign(size_t(n_rows), -1);
        for (size_t i = 0; i < pivot_cols.size(); i++) is.pivots[i] = pivot_cols[i];
        for (int c : pivot_cols) used[size_t(c)] = 1;
        out.push_back(std::move(is));
    }
    return out;
}

static uint64_t xorshift64star(uint64_t &s) {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    return s * 0x2545F4914F6CDD1DULL;
}

// bits [from, from + 64) of a packed row (zero beyond the row's words is the caller's padding)
static inline uint64_t word_at(const uint64_t *r, int from) {
    const int wi = from >> 6, sh = from & 63;
    return sh ? (r[wi] >> sh) | (r[wi + 1] << (64 - sh)) : r[wi];
}

int symplectic_ip(const uint64_t *u, const uint64_t *v, int n) {
    // bits [0, n) are x, [n, 2n) are z: parity of popc(u_x & v_z) + popc(u_z & v_x), 64 at a time
    int par = 0;
    for (int i = 0; i < n; i += 64) {
        const int len = std::min(64, n - i);
        const uint64_t mask = len == 64 ? ~uint64_t(0) : ((uint64_t(1) << len) - 1);
        // word_at may read one word past the x block; row strides cover 2n bits, and the
        // z block lies right after, so reads stay inside the row
        const uint64_t ux = word_at(u, i) & mask, uz = (((n + i) & 63) + len > 64 || len == 64 ? word_at(u, n + i)
                                                                                                : u[(n + i) >> 6] >> ((n + i) & 63)) & mask;
        const uint64_t vx = word_at(v, i) & mask, vz = (((n + i) & 63) + len > 64 || len == 64 ? word_at(v, n + i)
                                                                                                : v[(n + i) >> 6] >> ((n + i) & 63)) & mask;
        par ^= (__builtin_popcountll(ux & vz) ^ __builtin_popcountll(uz & vx)) & 1;
    }
    return par;
}

BitMat generate_code(int n, int k, uint64_t seed, int transvections) {
    if (n <= 0 || k < 0 || k > n) throw InvalidArgument("generate_code: need 0 <= k <= n, n >= 1");
    if (seed == 0) throw InvalidArgument("generate_code: xorshift64* needs a nonzero seed");
    if (transvections <= 0) transvections = 4 * n;
    const int rows = n + k, cols = 2 * n;
    BitMat a(rows, cols);
    int r = 0;
    for (int i = 0; i < n - k; i++) a.set(r++, n + i, true);
    for (int i = n - k; i < n; i++) a.set(r++, i, true);
    for (int i = n - k; i < n; i++) a.set(r++, n + i, true);
    BitMat v(1, cols);
    uint64_t s = seed;
    const int words = (cols + 63) / 64;
    for (int t = 0; t < transvections; t++) {
        for (;;) {
            for (int w = 0; w < words; w++) v.row(0)[w] = xorshift64star(s);
            if (cols & 63) v.row(0)[words - 1] &= (~uint64_t(0)) >> (64 - (cols & 63));
            if (!v.row_is_zero(0)) break;
        }
        for (int i = 0; i < rows; i++)
            if (symplectic_ip(a.row(i), v.row(0), n)) {
                uint64_t *u = a.row(i);
                for (int w = 0; w < a.stride; w++) u[w] ^= v.row(0)[w];
            }
    }
    return a;
}

BitMat random_stabilizer(int n, int k, uint64_t seed) {
    if (n <= 0 || k < 0 || k > n) throw InvalidArgument("random_stabilizer: need 0 <= k <= n, n >= 1");
    std::mt19937_64 rng(seed);
    const int cols = 2 * n, dim_c = n - k;
    BitMat c(0, cols), ech(0, cols);
    std::vector<int> pivots;
    auto append = [](BitMat &m, const uint64_t *row) {
        m.w.insert(m.w.end(), row, row + m.stride);
        m.rows++;
    };
    while (c.rows < dim_c) {
        // uniform draw from the symplectic complement of the rows so far
        const BitMat basis = null_space(swap_halves(c));
        for (;;) {
            std::vector<uint64_t> v(size_t(c.stride), 0);
            const int dim = basis.rows;
            std::vector<uint64_t> draw(size_t((dim + 63) / 64));
            for (uint64_t &x : draw) x = rng();
            for (int i = 0; i < dim; i++)
                if ((draw[size_t(i / 64)] >> (i % 64)) & 1u)
                    for (int w = 0; w < c.stride; w++) v[size_t(w)] ^= basis.row(i)[w];
            std::vector<uint64_t> res(v);
            for (int r = 0; r < ech.rows; r++)
                if ((res[size_t(pivots[size_t(r)] >> 6)] >> (pivots[size_t(r)] & 63)) & 1u)
                    for (int w = 0; w < c.stride; w++) res[size_t(w)] ^= ech.row(r)[w];
            int pivot = -1;
            for (int b = 0; b < cols && pivot < 0; b++)
                if ((res[size_t(b >> 6)] >> (b & 63)) & 1u) pivot = b;
            if (pivot < 0) continue;  // dependent draw
            append(c, v.data());
            append(ech, res.data());
            pivots.push_back(pivot);
            break;
        }
    }
    return null_space(swap_halves(c));
}

namespace {
[[noreturn]] void parse_fail(const std::string &origin, size_t line, const std::string &what) {
    throw ParseFailure(origin + ":" + std::to_string(line) + ": " + what);
}
bool blank_line(const std::string &s) {
    for (char ch : s)
        if (!std::isspace(static_cast<unsigned char>(ch))) return false;
    return true;
}
}  // namespace

BitMat parse_matrix_text(const std::string &text, const std::string &origin) {
    std::istringstream in(text);
    std::string line;
    size_t line_no = 0;
    long k_rows = -1, n_cols = -1;
    while (std::getline(in, line)) {
        ++line_no;
        if (blank_line(line)) continue;
        std::istringstream header(line);
        std::string extra;
        if (!(header >> k_rows >> n_cols) || (header >> extra))
            parse_fail(origin, line_no, "bad header; expected two integers \"K N\"");
        break;
    }
    if (k_rows < 0) parse_fail(origin, line_no, "empty input; expected a \"K N\" header");
    if (k_rows == 0 || n_cols <= 0) parse_fail(origin, line_no, "bad header; K and N must be positive");
    if (n_cols % 2 != 0) parse_fail(origin, line_no, "N must be even (columns come in symplectic pairs)");
    if (k_rows > n_cols) parse_fail(origin, line_no, "K exceeds N; rows cannot be independent");
    BitMat m(0, int(n_cols));
    std::vector<uint64_t> row(size_t(m.stride));
    long rows_read = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (blank_line(line)) continue;
        if (rows_read == k_rows) parse_fail(origin, line_no, "expected " + std::to_string(k_rows) + " rows, found more");
        std::fill(row.begin(), row.end(), 0);
        long bits = 0;
        for (size_t col = 0; col < line.size(); ++col) {
            const char ch = line[col];
            if (std::isspace(static_cast<unsigned char>(ch))) continue;
            if (ch != '0' && ch != '1')
                parse_fail(origin, line_no,
                           "row " + std::to_string(rows_read + 1) + ", column " + std::to_string(col + 1) +
                               ": expected '0' or '1', found '" + std::string(1, ch) + "'");
            if (bits == n_cols)
                parse_fail(origin, line_no,
                           "row " + std::to_string(rows_read + 1) + " has more than " + std::to_string(n_cols) +
                               " bits");
            if (ch == '1') row[size_t(bits >> 6)] |= uint64_t(1) << (bits & 63);
            ++bits;
        }
        if (bits != n_cols)
            parse_fail(origin, line_no,
                       "row " + std::to_string(rows_read + 1) + " has " + std::to_string(bits) + " bits, expected " +
                           std::to_string(n_cols));
        m.w.insert(m.w.end(), row.begin(), row.end());
        m.rows++;
        ++rows_read;
    }
    if (rows_read != k_rows)
        parse_fail(origin, line_no,
                   "expected " + std::to_string(k_rows) + " rows, found " + std::to_string(rows_read));
    return m;
}

std::string format_matrix(const BitMat &m) {
    std::string out = std::to_string(m.rows) + " " + std::to_string(m.cols) + "\n";
    for (int r = 0; r < m.rows; r++) out += m.row_string(r) + "\n";
    return out;
}

}  // namespace sdb
