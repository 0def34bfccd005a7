#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <thread>

#include "comm.hpp"
#include "errors.hpp"

namespace sdb {

size_t problem_smem_bytes(int G, int N, int W, int SW, int BK);

void check_cuda(cudaError_t e, const char *what) {
    if (e != cudaSuccess) throw DeviceFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

std::vector<unsigned long long> binom_table(int N, int BK) {
    const unsigned long long cap = 1ull << 62;
    std::vector<unsigned long long> t(size_t(N + 1) * BK, 0);
    for (int a = 0; a <= N; a++)
        for (int b = 0; b < BK && b <= a; b++) {
            if (b == 0 || b == a) {
                t[size_t(a) * BK + b] = 1;
            } else {
                const unsigned long long x = t[size_t(a - 1) * BK + b - 1], y = t[size_t(a - 1) * BK + b];
                t[size_t(a) * BK + b] = (x >= cap || y >= cap || x + y >= cap) ? cap : x + y;
            }
        }
    return t;
}

static unsigned long long binom_u64(int a, int b) {
    if (b < 0 || a < 0 || b > a) return 0;
    if (b > a - b) b = a - b;
    unsigned __int128 r = 1;
    for (int i = 1; i <= b; i++) {
        r = r * unsigned(a - b + i) / unsigned(i);
        if (r >> 62) return 1ull << 62;
    }
    return (unsigned long long)r;
}

// bits of row r at columns [from, from+len) packed into u32 words
// 64 bits of a row starting at column `from` (zero past the row's last word)
static inline uint64_t row_bits64(const BitMat &m, int r, int from) {
    const uint64_t *w = m.row(r);
    const int wi = from >> 6, sh = from & 63;
    const uint64_t lo = wi < m.stride ? w[wi] : 0, hi = (sh && wi + 1 < m.stride) ? w[wi + 1] : 0;
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

// bits of row r at columns [from, from+len) packed into u32 words
static void extract_bits(const BitMat &m, int r, int from, int len, uint32_t *dst, int words) {
    for (int i = 0; i < words; i++) dst[i] = 0;
    for (int c = 0; c < len; c += 64) {
        uint64_t v = row_bits64(m, r, from + c);
        if (len - c < 64) v &= (uint64_t(1) << (len - c)) - 1;
        if ((c >> 5) < words) dst[c >> 5] = uint32_t(v);
        if ((c >> 5) + 1 < words) dst[(c >> 5) + 1] = uint32_t(v >> 32);
    }
}

ProbeChoice orient_probe_words(std::vector<uint32_t> &rows, int G, int N, int W, int bits) {
    // popc(x|z) is symmetric in x and z position by position, so swapping the x-word and
    // the z-word of one 32-symbol block (in every row of a Gamma) leaves every candidate
    // weight unchanged. The tile kernels' fast path folds the first (probe) word of each
    // block, so put the component that is denser in sums of rows there: systematic Gamma_j
    // carry an identity block in one component (the x columns of Gamma_1 on the isometry
    // route), which makes that component sparse in every combination. When even the
    // oriented probe words fold sparse (pivot-heavy blocks, e.g. the F4-diagonalized package
    // routes), one partner word joins the probe: the block that adds the most set bits.
    uint64_t s = 0x9E3779B97F4A7C15ull;
    auto next = [&s]() {
        s ^= s >> 12;
        s ^= s << 25;
        s ^= s >> 27;
        return s * 0x2545F4914F6CDD1Dull;
    };
    const int g0 = std::min(N, 6), samples = 256;
    std::vector<uint32_t> acc(size_t(2 * W));
    std::vector<uint32_t> sums(size_t(samples) * 2 * W);  // [sample][2W]
    ProbeChoice pc;
    pc.extra.assign(size_t(G), -1);
    pc.fill.assign(size_t(G), -1);
    // the last block's unused bit positions: the fold may carry another block's partner
    // component there (bit b then still tests only symbols at bit b of some block)
    const int last = bits - 32 * (W - 1);
    pc.free_mask = (W > 1 && last > 0 && last < 32) ? ~((1u << last) - 1u) : 0u;
    double base_mean = 0, gain_mean = 0;
    for (int j = 0; j < G; j++) {
        uint32_t *base = rows.data() + size_t(j) * N * 2 * W;
        std::vector<long> dx(size_t(W), 0), dz(size_t(W), 0);
        for (int smp = 0; smp < samples; smp++) {
            std::fill(acc.begin(), acc.end(), 0u);
            for (int i = 0; i < g0; i++) {
                const int r = int(next() % uint64_t(N));
                for (int w = 0; w < 2 * W; w++) acc[size_t(w)] ^= base[size_t(r) * 2 * W + w];
            }
            std::copy(acc.begin(), acc.end(), sums.begin() + long(smp) * 2 * W);
            for (int w = 0; w < W; w++) {
                dx[size_t(w)] += __builtin_popcount(acc[size_t(w)]);
                dz[size_t(w)] += __builtin_popcount(acc[size_t(W + w)]);
            }
        }
        for (int w = 0; w < W; w++)
            if (dz[size_t(w)] > dx[size_t(w)]) {
                for (int r = 0; r < N; r++) std::swap(base[size_t(r) * 2 * W + w], base[size_t(r) * 2 * W + W + w]);
                for (int smp = 0; smp < samples; smp++)
                    std::swap(sums[size_t(smp) * 2 * W + w], sums[size_t(smp) * 2 * W + W + w]);
            }
        if (W == 1) continue;  // the fast path is exact already
        // mean fold weight with the probe words, and with each partner word added
        double fold = 0;
        std::vector<double> with(size_t(W), 0);
        for (int smp = 0; smp < samples; smp++) {
            const uint32_t *v = sums.data() + size_t(smp) * 2 * W;
            uint32_t u = 0;
            for (int w = 0; w < W; w++) u |= v[size_t(w)];
            fold += __builtin_popcount(u);
            for (int e = 0; e < W; e++) with[size_t(e)] += __builtin_popcount(u | v[size_t(W + e)]);
        }
        int best = 0;
        for (int e = 1; e < W; e++)
            if (with[size_t(e)] > with[size_t(best)]) best = e;
        pc.extra[size_t(j)] = best;
        if (pc.free_mask) {
            // which block's partner fills the free bits best
            std::vector<double> fill(size_t(W - 1), 0);
            for (int smp = 0; smp < samples; smp++) {
                const uint32_t *v = sums.data() + size_t(smp) * 2 * W;
                uint32_t u = 0;
                for (int w = 0; w < W; w++) u |= v[size_t(w)];
                for (int e = 0; e < W - 1; e++)
                    fill[size_t(e)] += __builtin_popcount((u | (v[size_t(W + e)] & pc.free_mask)) & pc.free_mask);
            }
            int fb = 0;
            for (int e = 1; e < W - 1; e++)
                if (fill[size_t(e)] > fill[size_t(fb)]) fb = e;
            pc.fill[size_t(j)] = fb;
        }
        base_mean += fold / samples / G;
        gain_mean += (with[size_t(best)] - fold) / samples / G;
    }
    // one more LOP3 per candidate pays only when the plain fold leaves the false-positive rate
    // high: its mean sits well below the 32 bits a word can show
    pc.use_extra = W > 1 && base_mean < 22.0 && gain_mean >= 2.0;
    if (const char *force = std::getenv("SDB_EXTRA_PROBE"))  // experiments: 0 off, 1 on
        pc.use_extra = W > 1 && force[0] == '1';
    return pc;
}

int build_syndromes(const std::vector<GammaIn> &gammas, int n, const Filter &f, std::vector<uint64_t> &out) {
    out.clear();
    if (!f.enabled) return 0;
    const int G = int(gammas.size()), F = f.rows.rows;
    int N = 0;
    for (const GammaIn &gm : gammas) N = std::max(N, gm.matrix.rows);
    // S: (G*N) x F, bit (i, r) = <first 2n columns of Gamma row i, filter row r>_s (the
    // reference's projection, engine.cpp:168-173), from word-aligned copies of both halves:
    // <(x|z), (a|b)>_s = parity(popc(x & b) + popc(z & a))
    BitMat S(G * N, F);
    const int hw = (n + 63) / 64;
    auto halves = [&](const BitMat &m, int r, uint64_t *x, uint64_t *z) {
        for (int w = 0; w < hw; w++) {
            const int len = std::min(64, n - 64 * w);
            const uint64_t mask = len == 64 ? ~uint64_t(0) : ((uint64_t(1) << len) - 1);
            x[w] = row_bits64(m, r, 64 * w) & mask;
            z[w] = row_bits64(m, r, n + 64 * w) & mask;
        }
    };
    std::vector<uint64_t> fa(size_t(F) * size_t(hw)), fb(size_t(F) * size_t(hw)), x(static_cast<size_t>(hw)),
        z(static_cast<size_t>(hw));
    for (int r = 0; r < F; r++) halves(f.rows, r, &fa[size_t(r) * hw], &fb[size_t(r) * hw]);
    for (int j = 0; j < G; j++)
        for (int i = 0; i < gammas[size_t(j)].matrix.rows; i++) {
            halves(gammas[size_t(j)].matrix, i, x.data(), z.data());
            uint64_t *dst = S.row(j * N + i);
            for (int r = 0; r < F; r++) {
                int p = 0;
                for (int w = 0; w < hw; w++)
                    p += __builtin_popcountll(x[size_t(w)] & fb[size_t(r) * hw + w]) +
                         __builtin_popcountll(z[size_t(w)] & fa[size_t(r) * hw + w]);
                if (p & 1) dst[r >> 6] |= uint64_t(1) << (r & 63);
            }
        }
    // every candidate syndrome lies in rowspace(S); it is zero iff it vanishes on the
    // pivot columns of S's echelon form, so keep only those columns
    BitMat E = S;
    const std::vector<int> piv = echelonize(E);
    const int rk = int(piv.size());
    const int SW = std::max(1, (rk + 63) / 64);
    if (SW > kMaxSW) throw InvalidArgument("admissibility syndrome wider than 256 bits (k > 128)");
    out.assign(size_t(G) * N * SW, 0);
    for (int i = 0; i < G * N; i++)
        for (int b = 0; b < rk; b++)
            if (S.get(i, piv[size_t(b)])) out[size_t(i) * SW + (b >> 6)] |= uint64_t(1) << (b & 63);
    return SW;
}

Plan::Plan(std::vector<GammaIn> gammas, Mode mode, int pair_count, const Filter &filter, const sdb_run_options &opts)
    : gammas_(std::move(gammas)), mode_(mode), pair_count_(pair_count), opts_(opts) {
    if (gammas_.empty()) throw InvalidArgument("run_bz: need at least one generator matrix");
    G_ = int(gammas_.size());
    if (G_ > kMaxG) throw InvalidArgument("run_bz: too many generator matrices");
    N_ = gammas_[0].matrix.rows;
    const int cols = gammas_[0].matrix.cols;
    for (const GammaIn &g : gammas_) {
        if (!g.packages.empty()) packaged_ = true;
        if (g.matrix.cols != cols) throw InvalidArgument("run_bz: generator matrices must share one codeword frame");
        if (g.packages.empty() && g.matrix.rows == 0) throw InvalidArgument("run_bz: matrix with no packages");
        N_ = std::max(N_, g.matrix.rows);
    }
    if (!packaged_)
        for (const GammaIn &g : gammas_)
            if (g.matrix.rows != N_) packaged_ = true;  // unequal package counts: packaged kernel
    if (packaged_) {
        if (G_ > kMaxPkgG) throw InvalidArgument("run_bz: package routes take at most 4 generator matrices");
        for (GammaIn &g : gammas_) {
            if (g.packages.empty())
                for (int r = 0; r < g.matrix.rows; r++) g.packages.push_back({r});
            if (g.packages.empty()) throw InvalidArgument("run_bz: matrix with no packages");
            for (const std::vector<int> &pk : g.packages) {
                if (pk.empty() || pk.size() > 3) throw InvalidArgument("run_bz: packages hold one to three rows");
                for (int r : pk)
                    if (r < 0 || r >= g.matrix.rows) throw InvalidArgument("run_bz: package row out of range");
            }
            np_.push_back(int(g.packages.size()));
            P_ = std::max(P_, int(g.packages.size()));
        }
    }
    if (N_ == 0) throw InvalidArgument("run_bz: matrix with no packages");
    const int n = pair_count_;
    if (filter.enabled && filter.rows.cols != 2 * n)
        throw InvalidArgument("enumerate_generation: filter frame mismatch");

    // weight layout
    std::vector<uint32_t> xw, zw;
    if (mode_ == Mode::symplectic) {
        if (cols != 2 * n) throw InvalidArgument("symplectic mode needs 2n columns");
        W_ = (n + 31) / 32;
        scale_ = 1;
        max_weight_ = n;
        sentinel_ = n + 1;
        image_layout_ = true;
    } else {
        sentinel_ = cols + 1;
        max_weight_ = cols;
        bool image = n > 0 && cols == 3 * n;
        for (int j = 0; image && j < G_; j++) {
            const BitMat &m = gammas_[size_t(j)].matrix;
            for (int r = 0; image && r < m.rows; r++)
                for (int i = 0; i < n && image; i += 64) {
                    const uint64_t mask = n - i >= 64 ? ~uint64_t(0) : ((uint64_t(1) << (n - i)) - 1);
                    image = ((row_bits64(m, r, i) ^ row_bits64(m, r, n + i) ^ row_bits64(m, r, 2 * n + i)) & mask) == 0;
                }
        }
        image_layout_ = image;
        if (image) {
            W_ = (n + 31) / 32;
            scale_ = 2;
        } else {
            W_ = (cols + 31) / 32;
            scale_ = 1;
        }
    }
    if (W_ < 1) W_ = 1;
    if (W_ > kMaxW) throw InvalidArgument("rows too wide for the enumeration kernels (n > 256)");
    const bool trace_host = std::getenv("SDB_TRACE_HOST") != nullptr;
    auto tick = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (!trace_host) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[sdb]   plan %s %.3f ms\n", what, 1e3 * std::chrono::duration<double>(now - tick).count());
        tick = now;
    };
    h_rows_.assign(size_t(G_) * N_ * 2 * W_, 0);
    for (int j = 0; j < G_; j++)
        for (int r = 0; r < gammas_[size_t(j)].matrix.rows; r++) {
            uint32_t *dst = h_rows_.data() + (size_t(j) * N_ + r) * 2 * W_;
            const BitMat &m = gammas_[size_t(j)].matrix;
            if (image_layout_) {
                extract_bits(m, r, 0, n, dst, W_);
                extract_bits(m, r, n, n, dst + W_, W_);
            } else {
                extract_bits(m, r, 0, cols, dst, W_);
            }
        }
    lap("rows");
    const ProbeChoice probe = orient_probe_words(h_rows_, G_, N_, W_, image_layout_ ? n : 32 * W_);
    K_ = W_ == 1 ? 2 : W_ + (probe.use_extra ? 1 : 0);
    h_prows_.assign(size_t(G_) * N_ * K_, 0);
    for (int j = 0; j < G_; j++)
        for (int r = 0; r < N_; r++) {
            const uint32_t *src = h_rows_.data() + (size_t(j) * N_ + r) * 2 * W_;
            uint32_t *dst = h_prows_.data() + (size_t(j) * N_ + r) * K_;
            for (int w = 0; w < std::min(K_, W_ == 1 ? 2 : W_); w++) dst[w] = src[w];
            if (K_ > W_ && W_ > 1) dst[W_] = src[W_ + probe.extra[size_t(j)]];
            if (probe.fill[size_t(j)] >= 0) dst[W_ - 1] |= src[W_ + probe.fill[size_t(j)]] & probe.free_mask;
        }
    lap("orient");
    SW_ = build_syndromes(gammas_, n, filter, h_syn_);
    lap("syndromes");
    if (!packaged_ && (mode_ == Mode::symplectic || image_layout_) && W_ <= 4 && n > 0 &&
        std::getenv("SDB_NO_TC") == nullptr) {
        std::vector<const BitMat *> mats;
        for (const GammaIn &g : gammas_) mats.push_back(&g.matrix);
        tc_enc_ = tc_encode(mats, N_, n, mode_ == Mode::hamming);
        tc_ok_ = tc_enc_.ok;
        lap("tc encoding");
    }
    BK_ = std::min(N_, kMaxLevel) + 2;
    h_binom_ = binom_table(N_, BK_);
    lap("binom");
    if (packaged_) {
        // package tables and weighted suffix counts wsuf(q, m) = wsuf(q+1, m) + s_q wsuf(q+1, m-1)
        const unsigned long long cap = 1ull << 62;
        h_pk_rows_.assign(size_t(G_) * P_ * 3, -1);
        h_pk_size_.assign(size_t(G_) * P_, 0);
        h_wsuf_.assign(size_t(G_) * (P_ + 1) * BK_, 0);
        for (int j = 0; j < G_; j++) {
            const auto &pk = gammas_[size_t(j)].packages;
            const int np = int(pk.size());
            for (int q = 0; q < np; q++) {
                h_pk_size_[size_t(j) * P_ + q] = (unsigned char)pk[size_t(q)].size();
                for (size_t m = 0; m < pk[size_t(q)].size(); m++)
                    h_pk_rows_[(size_t(j) * P_ + q) * 3 + m] = short(pk[size_t(q)][m]);
            }
            unsigned long long *ws = h_wsuf_.data() + size_t(j) * (P_ + 1) * BK_;
            ws[size_t(np) * BK_] = 1;
            for (int q = np - 1; q >= 0; q--)
                for (int m = 0; m < BK_; m++) {
                    const unsigned long long a = ws[size_t(q + 1) * BK_ + m],
                                             b = m ? ws[size_t(q + 1) * BK_ + m - 1] * pk[size_t(q)].size() : 0;
                    ws[size_t(q) * BK_ + m] = (a >= cap || b >= cap || a + b >= cap) ? cap : a + b;
                }
        }
        // expanded elements (package members) in forward and reversed package order, and the
        // weighted colex counts F / FR of the packaged tile kernel
        for (int j = 0; j < G_; j++) {
            int e = 0;
            for (const auto &pk : gammas_[size_t(j)].packages) e += int(pk.size());
            E_ = std::max(E_, e);
        }
        h_e_row_.assign(size_t(G_) * E_, -1);
        h_e_pkg_.assign(size_t(G_) * E_, -1);
        h_r_row_.assign(size_t(G_) * E_, -1);
        h_r_pkg_.assign(size_t(G_) * E_, -1);
        h_off_.assign(size_t(G_) * (P_ + 1), 0);
        h_r_off_.assign(size_t(G_) * (P_ + 1), 0);
        h_F_.assign(size_t(G_) * (E_ + 1) * BK_, 0);
        h_FR_.assign(size_t(G_) * (E_ + 1) * BK_, 0);
        for (int j = 0; j < G_; j++) {
            const auto &pk = gammas_[size_t(j)].packages;
            const int np = int(pk.size());
            for (int dir = 0; dir < 2; dir++) {
                short *erow = (dir ? h_r_row_ : h_e_row_).data() + size_t(j) * E_;
                short *epkg = (dir ? h_r_pkg_ : h_e_pkg_).data() + size_t(j) * E_;
                short *off = (dir ? h_r_off_ : h_off_).data() + size_t(j) * (P_ + 1);
                unsigned long long *F = (dir ? h_FR_ : h_F_).data() + size_t(j) * (E_ + 1) * BK_;
                int e = 0;
                for (int qq = 0; qq < np; qq++) {
                    const int q = dir ? np - 1 - qq : qq;  // reversed: package np-1-q' at position q'
                    off[qq] = short(e);
                    for (int r : pk[size_t(q)]) {
                        erow[e] = short(r);
                        epkg[e] = short(qq);
                        e++;
                    }
                }
                for (int qq = np; qq <= P_; qq++) off[qq] = short(e);
                for (int x = 0; x <= e; x++) F[size_t(x) * BK_] = 1;
                for (int x = 1; x <= e; x++)
                    for (int i = 1; i < BK_; i++) {
                        const unsigned long long a = F[size_t(x - 1) * BK_ + i],
                                                 b = F[size_t(off[epkg[x - 1]]) * BK_ + i - 1];
                        F[size_t(x) * BK_ + i] = (a >= cap || b >= cap || a + b >= cap) ? cap : a + b;
                    }
            }
        }
    }
    upload();
    lap("upload");
}

// ---- process-wide caches: repeated distance calls skip cudaMalloc / stream / event creation
namespace {
std::mutex g_cache_mu;
struct FreeBlock {
    int device;
    size_t bytes;
    void *ptr;
};
std::vector<FreeBlock> g_free_blocks;
std::vector<std::pair<int, cudaEvent_t>> g_free_events;

void *workspace_get(int device, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        size_t best = g_free_blocks.size();
        for (size_t i = 0; i < g_free_blocks.size(); i++) {
            const FreeBlock &f = g_free_blocks[i];
            if (f.device == device && f.bytes >= bytes && f.bytes <= 4 * bytes + (1 << 20) &&
                (best == g_free_blocks.size() || f.bytes < g_free_blocks[best].bytes))
                best = i;
        }
        if (best < g_free_blocks.size()) {
            void *p = g_free_blocks[best].ptr;
            g_free_blocks.erase(g_free_blocks.begin() + long(best));
            return p;
        }
    }
    void *p = nullptr;
    check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
    return p;
}

void workspace_put(int device, size_t bytes, void *p) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_free_blocks.push_back(FreeBlock{device, bytes, p});
    if (g_free_blocks.size() > 16) {
        cudaFree(g_free_blocks.front().ptr);
        g_free_blocks.erase(g_free_blocks.begin());
    }
}

cudaEvent_t event_get(int device) {
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (size_t i = 0; i < g_free_events.size(); i++)
            if (g_free_events[i].first == device) {
                cudaEvent_t e = g_free_events[i].second;
                g_free_events.erase(g_free_events.begin() + long(i));
                return e;
            }
    }
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "cudaEventCreate");
    return e;
}

void event_put(int device, cudaEvent_t e) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_free_events.emplace_back(device, e);
}

std::vector<std::pair<size_t, void *>> g_free_pinned;

void *pinned_get(size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (size_t i = 0; i < g_free_pinned.size(); i++)
            if (g_free_pinned[i].first >= bytes && g_free_pinned[i].first <= 4 * bytes + (1 << 20)) {
                void *p = g_free_pinned[i].second;
                g_free_pinned.erase(g_free_pinned.begin() + long(i));
                return p;
            }
    }
    void *p = nullptr;
    check_cuda(cudaMallocHost(&p, bytes), "cudaMallocHost");
    return p;
}

void pinned_put(size_t bytes, void *p) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_free_pinned.emplace_back(bytes, p);
    if (g_free_pinned.size() > 16) {
        cudaFreeHost(g_free_pinned.front().second);
        g_free_pinned.erase(g_free_pinned.begin());
    }
}

// one non-blocking stream per (thread, device), kept for the process lifetime
cudaStream_t thread_stream(int device) {
    thread_local std::vector<std::pair<int, cudaStream_t>> streams;
    for (auto &s : streams)
        if (s.first == device) return s.second;
    cudaStream_t st;
    check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    streams.emplace_back(device, st);
    return st;
}
}  // namespace

Plan::~Plan() {
    if (d_mem_ || h_stage_) cudaStreamSynchronize(stream_);
    if (d_mem_) workspace_put(device_, d_bytes_, d_mem_);
    if (h_stage_) pinned_put(d_bytes_, h_stage_);
    for (cudaEvent_t e : events_)
        if (e) event_put(device_, e);
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

void Plan::upload() {
    // size checks first: a rejected problem must not leave a device block or a pinned image
    // (with an H2D copy in flight) behind, since ~Plan does not run when the constructor throws
    if (problem_smem_bytes(G_, N_, W_, SW_, BK_) > 200 * 1024 ||
        (packaged_ && pkg_smem_bytes(G_, N_, W_, SW_, P_, BK_) > 200 * 1024))
        throw InvalidArgument("problem too large for shared-memory staging");
    device_ = opts_.device;
    check_cuda(cudaSetDevice(device_), "cudaSetDevice");
    check_cuda(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device_), "cudaDeviceGetAttribute");
    stream_ = opts_.stream ? static_cast<cudaStream_t>(opts_.stream) : thread_stream(device_);
    // tile unit tables: level g needs G * (N - g + 1) + 1 entries (boundaries b in [h, N - t])
    table_cap_ = size_t(G_) * size_t(N_ + 1) * size_t(N_ + 2) / 2 + size_t(N_ + 2);
    const size_t b_prows = align256(h_prows_.size() * 4);
    const size_t b_rows = align256(h_rows_.size() * 4), b_syn = align256(std::max<size_t>(h_syn_.size(), 1) * 8),
                 b_binom = align256(h_binom_.size() * 8),
                 b_state = align256(sizeof(LevelState) + size_t(max_weight_ + 1) * 8),
                 b_ctl = align256(sizeof(RunCtl)), b_trace = align256(size_t(N_ + 1) * 4),
                 b_counters = align256(size_t(N_ + 1) * 8), b_tables = align256(table_cap_ * 8);
    const size_t b_pkr = align256(h_pk_rows_.size() * 2 + 2), b_pks = align256(h_pk_size_.size() + 1),
                 b_ws = align256(h_wsuf_.size() * 8 + 8), b_el = align256(h_e_row_.size() * 2 + 2),
                 b_off = align256(h_off_.size() * 2 + 2), b_F = align256(h_F_.size() * 8 + 8);
    if (packaged_) table_cap_ += size_t(G_) * size_t(P_ + 1) * size_t(P_ + 2);  // room for the pair lists
    const size_t b_tables_pk = align256(table_cap_ * 8);
    const size_t b_tc_sign = tc_ok_ ? align256(tc_enc_.sign.size() * 4) : 0,
                 b_tc_mask = tc_ok_ ? align256(tc_enc_.mask.size() * 2) : 0,
                 b_tc_gam = tc_ok_ ? align256(tc_enc_.gam.size() * sizeof(TcGammaDev)) : 0;
    d_bytes_ = b_prows + b_rows + b_syn + b_binom + b_state + b_ctl + b_trace + 2 * b_counters +
               (packaged_ ? b_tables_pk + b_pkr + b_pks + b_ws + 4 * b_el + 2 * b_off + 2 * b_F : b_tables) +
               b_tc_sign + b_tc_mask + b_tc_gam;
    const auto t0 = std::chrono::steady_clock::now();
    d_mem_ = workspace_get(device_, d_bytes_);
    // every input section is laid out in one pinned staging image of the device block and
    // goes over in a single asynchronous copy; the unit tables of later levels are staged in
    // the same image (h_pinned_) and copied level by level
    h_stage_ = static_cast<unsigned char *>(pinned_get(d_bytes_));
    unsigned char *base = static_cast<unsigned char *>(d_mem_);
    size_t at = 0;
    auto place = [&](const void *src, size_t bytes, size_t region) {
        if (bytes) std::memcpy(h_stage_ + at, src, bytes);
        unsigned char *dev = base + at;
        at += region;
        return dev;
    };
    pd_.rows = reinterpret_cast<const uint32_t *>(place(h_rows_.data(), h_rows_.size() * 4, b_rows));
    pd_.syn = reinterpret_cast<const unsigned long long *>(place(h_syn_.data(), h_syn_.size() * 8, b_syn));
    pd_.binom = reinterpret_cast<const unsigned long long *>(place(h_binom_.data(), h_binom_.size() * 8, b_binom));
    upload_bytes = h_rows_.size() * 4 + h_syn_.size() * 8 + h_binom_.size() * 8;
    unsigned char *q = place(nullptr, 0, b_state);
    pd_.state = reinterpret_cast<LevelState *>(q);
    pd_.key_by_w = reinterpret_cast<unsigned long long *>(q + sizeof(LevelState));
    // the host image's ctl section receives the level checks' D2H copies (pinned: asynchronous)
    h_ctl_ = reinterpret_cast<RunCtl *>(h_stage_ + at);
    pd_.ctl = reinterpret_cast<RunCtl *>(place(nullptr, 0, b_ctl));
    pd_.trace_upper = reinterpret_cast<int *>(place(nullptr, 0, b_trace));
    d_counters_ = reinterpret_cast<unsigned long long *>(place(nullptr, 0, b_counters));
    h_counter_init_.assign(size_t(N_ + 1), 0);
    d_counter_init_ = reinterpret_cast<unsigned long long *>(place(h_counter_init_.data(), size_t(N_ + 1) * 8, b_counters));
    h_pinned_ = reinterpret_cast<unsigned long long *>(h_stage_ + at);
    d_tables_ = reinterpret_cast<unsigned long long *>(place(nullptr, 0, packaged_ ? b_tables_pk : b_tables));
    pd_.prows = reinterpret_cast<const uint32_t *>(place(h_prows_.data(), h_prows_.size() * 4, b_prows));
    pd_.K = K_;
    if (packaged_) {
        pk_.pk_rows = reinterpret_cast<const short *>(place(h_pk_rows_.data(), h_pk_rows_.size() * 2, b_pkr));
        pk_.pk_size = reinterpret_cast<const unsigned char *>(place(h_pk_size_.data(), h_pk_size_.size(), b_pks));
        pk_.wsuf = reinterpret_cast<const unsigned long long *>(place(h_wsuf_.data(), h_wsuf_.size() * 8, b_ws));
        pt_.e_row = reinterpret_cast<const short *>(place(h_e_row_.data(), h_e_row_.size() * 2, b_el));
        pt_.e_pkg = reinterpret_cast<const short *>(place(h_e_pkg_.data(), h_e_pkg_.size() * 2, b_el));
        pt_.r_row = reinterpret_cast<const short *>(place(h_r_row_.data(), h_r_row_.size() * 2, b_el));
        pt_.r_pkg = reinterpret_cast<const short *>(place(h_r_pkg_.data(), h_r_pkg_.size() * 2, b_el));
        pt_.off = reinterpret_cast<const short *>(place(h_off_.data(), h_off_.size() * 2, b_off));
        pt_.r_off = reinterpret_cast<const short *>(place(h_r_off_.data(), h_r_off_.size() * 2, b_off));
        pt_.F = reinterpret_cast<const unsigned long long *>(place(h_F_.data(), h_F_.size() * 8, b_F));
        pt_.FR = reinterpret_cast<const unsigned long long *>(place(h_FR_.data(), h_FR_.size() * 8, b_F));
        pt_.E = E_;
        pk_.P = P_;
        for (int j = 0; j < G_; j++) pk_.np[j] = np_[size_t(j)];
        upload_bytes += h_pk_rows_.size() * 2 + h_pk_size_.size() + h_wsuf_.size() * 8;
    }
    upload_bytes += h_prows_.size() * 4;
    if (tc_ok_) {
        d_tc_sign_ = reinterpret_cast<const uint32_t *>(place(tc_enc_.sign.data(), tc_enc_.sign.size() * 4, b_tc_sign));
        d_tc_mask_ = reinterpret_cast<const short *>(place(tc_enc_.mask.data(), tc_enc_.mask.size() * 2, b_tc_mask));
        d_tc_gam_ = reinterpret_cast<const TcGammaDev *>(
            place(tc_enc_.gam.data(), tc_enc_.gam.size() * sizeof(TcGammaDev), b_tc_gam));
        upload_bytes += tc_enc_.sign.size() * 4 + tc_enc_.mask.size() * 2 + tc_enc_.gam.size() * sizeof(TcGammaDev);
    }
    check_cuda(cudaMemcpyAsync(base, h_stage_, at, cudaMemcpyHostToDevice, stream_), "H2D plan");
    h2d_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    pd_.G = G_;
    pd_.N = N_;
    pd_.W = W_;
    pd_.SW = SW_;
    pd_.BK = BK_;
    pd_.scale = scale_;
    pd_.max_weight = max_weight_;
    levels_.assign(size_t(N_ + 1), LevelHost{});
    events_.assign(size_t(2 * (N_ + 1)), nullptr);
}

cudaEvent_t Plan::level_event(int i) {
    if (!events_[size_t(i)]) events_[size_t(i)] = event_get(device_);
    return events_[size_t(i)];
}

size_t tile_smem_bytes(int G, int N, int W, int K, int BK);

// Experiments only: SDB_TILE_FORCE="g:t:tchunk,..." overrides the cost model's (t, tail chunk)
// for the listed levels (t = 0: the walk / package walk kernel).
static void forced_tile(int g, int &t, int &tchunk) {
    const char *force = std::getenv("SDB_TILE_FORCE");
    if (!force) return;
    for (const char *q = force; *q;) {
        int fg = 0, ft = 0, fc = 0, used = 0;
        if (std::sscanf(q, "%d:%d:%d%n", &fg, &ft, &fc, &used) != 3) break;
        if (fg == g && ft >= 0 && ft < g && fc >= 2 && fc <= kTailChunk) {
            t = ft;
            tchunk = fc;
        }
        q += used;
        if (*q == ',') q++;
    }
}

// Cost-model constants of choose_tile, fitted to a (t, tchunk) sweep of config 4 levels 6-8
// and config 2 levels 4-6 (tools/t_tchunk.py, profiles/r01_tchunk_sweep.log): a unit costs
// about 40k candidate-equivalents of dispensing, staging and head generation, and the last
// units leave about 0.4 of the biggest one as tail.
constexpr double kTileUnitCost = 40000;
constexpr double kTileTailFraction = 0.4;

TileChoice choose_tile(int G, int N, int g, int W, int K, unsigned long long per_gamma, int forced_kernel, int num_sms,
                       int world) {
    TileChoice best{0, kTailChunk};
    if (forced_kernel == 1 || g < 2) return best;
    const double total = double(per_gamma) * G;
    if (forced_kernel != 2 && total < double(1 << 16)) return best;
    // Level time in candidate-equivalents per CTA slot: max(total load / slots, the largest
    // unit) — a level with few big units is bound by its slowest CTA. A tile unit costs its
    // padded candidates (every lane of a warp with heads runs H heads) plus kTileUnitCost for
    // the dispenser, tail staging and head generation; the walk kernel costs ~28 per candidate
    // (measured 1.4e11 vs 3.9e12 cand/s) with perfectly fine granularity.
    // K: the launched kernel's probe words per row (W, or W + 1 with the extra probe word): it
    // sets the heads per lane, the head block and the CTAs per SM
    const double Hl = heads_per_lane(W, K), HBk = head_block(W, K);
    const double slots = double(num_sms) * tile_blocks_per_sm(W, K) * std::max(1, world);  // all ranks' CTAs
    std::vector<double> C(size_t(N + 1) * size_t(N + 1), 0.0);  // Pascal's triangle in doubles
    for (int a = 0; a <= N; a++)
        for (int k = 0; k <= a; k++)
            C[size_t(a) * (N + 1) + size_t(k)] =
                (k == 0 || k == a) ? 1.0 : C[size_t(a - 1) * (N + 1) + size_t(k - 1)] + C[size_t(a - 1) * (N + 1) + size_t(k)];
    double best_time = total * 28.0 / slots;
    if (forced_kernel == 2) best_time = 1e300;
    for (int t = 1; t < g; t++) {
        const int h = g - t;
        for (int tchunk = kTailChunk; tchunk >= 64; tchunk /= 2) {
            double sum = 0, biggest = 0;
            for (int b = h; b <= N - t; b++) {
                const double Hb = C[size_t(b) * (N + 1) + size_t(h)], Tb = C[size_t(N - 1 - b) * (N + 1) + size_t(t - 1)];
                const double nH = std::ceil(Hb / HBk), nT = std::ceil(Tb / tchunk);
                const double heads_last = Hb - (nH - 1) * HBk;
                const double warps_full = kTileThreads / 32.0, warps_last = std::ceil(heads_last / (32.0 * Hl));
                const double tc = Tb / nT;  // average tails per unit
                const double unit_full = warps_full * 32 * Hl * tc + kTileUnitCost,
                             unit_last = warps_last * 32 * Hl * tc + kTileUnitCost;
                sum += nT * ((nH - 1) * unit_full + unit_last);
                biggest = std::max(biggest, nH > 1 ? unit_full : unit_last);
            }
            sum *= G;
            // the average load per CTA slot plus the tail: the last units finish unevenly,
            // a fraction of the biggest unit late on average (this matters when sharding leaves
            // few units per CTA)
            const double time = std::max(sum / slots + kTileTailFraction * biggest, biggest);
            if (time < best_time) {
                best_time = time;
                best = TileChoice{t, tchunk};
            }
        }
    }
    return best;
}

int choose_tile_t(int G, int N, int g, int W, unsigned long long per_gamma, int forced_kernel) {
    return choose_tile(G, N, g, W, probe_words(W, false), per_gamma, forced_kernel, 148, 1).t;
}

// Cost model of the tensor-core tile kernel, in SM cycles per CTA (one CTA per SM). A unit
// (128 heads x up to 256 nbt tails) costs the larger of its MMAs (128 cycles per 256-column
// K = 32 step, measured: tools/microbench/tc_i8.cu) and its producer work (the head tile plus
// its share of the tail staging: a restaged chunk serves the run of units that share it).
constexpr double kTcHeadTileCycles = 700, kTcTailRowCycles = 3, kTcUnitCycles = 300, kTcEpiCycles = 200;
TcChoice choose_tc(int G, int N, int g, const std::vector<TcGammaDev> &gam, int kmax, int kw, int W, int BK,
                   int num_sms, int world) {
    TcChoice best{0, 1};
    if (g < 2) return best;
    const int BKs = std::min(BK, g + 2);
    int nbt_max = 0;
    for (int nbt = 1; nbt <= kTcMaxNbt; nbt++)
        if (tc_smem_layout(G, N, W, kmax, kw, nbt, BKs).total <= kTcSmemMax) nbt_max = nbt;
    if (nbt_max == 0) return best;
    std::vector<double> C(size_t(N + 1) * size_t(N + 1), 0.0);
    for (int a = 0; a <= N; a++)
        for (int k = 0; k <= a; k++)
            C[size_t(a) * (N + 1) + size_t(k)] =
                (k == 0 || k == a) ? 1.0 : C[size_t(a - 1) * (N + 1) + size_t(k - 1)] + C[size_t(a - 1) * (N + 1) + size_t(k)];
    const double slots = double(num_sms) * std::max(1, world);
    double best_time = 1e300;
    const double HB = double(kTcHeads) * kTcUnitTiles;
    for (int t = std::max(1, g - kTcMaxPart); t < g && t - 1 <= kTcMaxPart; t++) {
        const int h = g - t;
        for (int nbt = 1; nbt <= nbt_max; nbt++) {
            double sum = 0, biggest = 0;
            for (int j = 0; j < G; j++) {
                const double kt = gam[size_t(j)].K / 32;
                for (int b = h; b <= N - t; b++) {
                    const double Hb = C[size_t(b) * (N + 1) + size_t(h)], Tb = C[size_t(N - 1 - b) * (N + 1) + size_t(t - 1)];
                    const double nH = std::ceil(Hb / HB), nT = std::ceil(Tb / (kTcTileN * nbt));
                    const double na = std::ceil(Hb / nH / kTcHeads);    // head tiles per unit
                    const double tiles = std::ceil(Tb / nT / kTcTileN);  // tail tiles per unit
                    const double mma = na * tiles * std::max(kt * 128, kTcEpiCycles);
                    const double restage = nH > 1 ? 1.0 / std::min(nH, 4.0) : 1.0;
                    const double prod = na * kTcHeadTileCycles + restage * tiles * kTcTileN * kTcTailRowCycles;
                    const double unit = std::max(mma, prod) + kTcUnitCycles;
                    sum += nH * nT * unit;
                    biggest = std::max(biggest, unit);
                }
            }
            const double time = std::max(sum / slots + 0.5 * biggest, biggest);
            if (time < best_time) {
                best_time = time;
                best = TcChoice{t, nbt};
            }
        }
    }
    return best;
}

// L(g - 1) for the kernels' mid-level early exit (kernels.cu early_key); 0 turns it off: for
// g = 1, and for the single-level seam (run_level), whose caller's bound state it cannot see
unsigned Plan::early_bound(int g) const {
    if (g < 2 || single_level_) return 0;
    const long long L = lower_bound(g - 1);
    return L <= 0 ? 0u : unsigned(std::min<long long>(L, 0x7fffffffLL));
}

bool Plan::prepare_tc(int g, LevelHost &lv, int world, int rank) {
    TcChoice c = choose_tc(G_, N_, g, tc_enc_.gam, tc_enc_.kmax, tc_enc_.kw, W_, BK_, num_sms_, world);
    if (const char *force = std::getenv("SDB_TC_FORCE")) {  // experiments: "g:t:nbt,..."
        for (const char *q = force; *q;) {
            int fg = 0, ft = 0, fn = 0, used = 0;
            if (std::sscanf(q, "%d:%d:%d%n", &fg, &ft, &fn, &used) != 3) break;
            if (fg == g && ft > 0 && ft < g && fn >= 1 && fn <= kTcMaxNbt) c = TcChoice{ft, fn};
            q += used;
            if (*q == ',') q++;
        }
    }
    if (c.t == 0) return false;
    const int BKs = std::min(BK_, g + 2);
    if (tc_smem_layout(G_, N_, W_, tc_enc_.kmax, tc_enc_.kw, c.nbt, BKs).total > kTcSmemMax) return false;
    TcPlan &tp = lv.tc;
    TilePlan &tl = tp.tile;
    tl.g = g;
    tl.lprev = early_bound(g);
    tl.t = c.t;
    tl.h = g - c.t;
    tl.thr0 = ~0u;
    tl.nb = N_ - c.t - tl.h + 1;
    tl.tchunk = kTcTileN * c.nbt;
    tl.per_gamma = binom_u64(N_, g);
    const size_t n_entries = size_t(G_) * size_t(tl.nb) + 1;
    if (table_used_ + n_entries > table_cap_) return false;
    unsigned long long *h_table = h_pinned_ + table_used_;
    unsigned long long acc = 0;
    for (int j = 0; j < G_; j++)
        for (int b = tl.h; b <= N_ - c.t; b++) {
            h_table[size_t(j) * tl.nb + (b - tl.h)] = acc;
            const unsigned long long Hb = binom_u64(b, tl.h), Tb = binom_u64(N_ - 1 - b, c.t - 1);
            constexpr unsigned long long kHB = kTcHeads * kTcUnitTiles;
            acc += ((Hb + kHB - 1) / kHB) * ((Tb + tl.tchunk - 1) / tl.tchunk);
        }
    h_table[size_t(G_) * tl.nb] = acc;
    tl.unit_total = acc;
    tl.shard_rank = rank;
    tl.shard_world = world;
    tl.cum = d_tables_ + table_used_;
    tl.counter = d_counters_ + g;
    table_used_ += n_entries;
    check_cuda(cudaMemcpyAsync(const_cast<unsigned long long *>(tl.cum), h_table, n_entries * 8, cudaMemcpyHostToDevice,
                               stream_),
               "H2D unit table");
    tp.nbt = c.nbt;
    tp.kmax = tc_enc_.kmax;
    tp.kw = tc_enc_.kw;
    tp.sign = d_tc_sign_;
    tp.mask = d_tc_mask_;
    tp.gam = d_tc_gam_;
    lv.t = -3;
    return true;
}

long long Plan::lower_bound(int g) const {
    // engine.cpp:31-47 for singleton packages: hamming sums over matrices; symplectic
    // single matrix g+1; two matrices g+1+max(0, g+1+n_pp-n_p) with n_pp = n_p here.
    if (mode_ == Mode::hamming) {
        long long s = 0;
        for (const GammaIn &gm : gammas_) s += std::max(0LL, (long long)g + 1 - gm.rank_deficit);
        return s;
    }
    if (G_ == 1) return (long long)g + 1;
    if (G_ == 2) {
        const GammaIn &d = gammas_[1];
        const long long np = d.packages.empty() ? d.matrix.rows : (long long)d.packages.size();
        const long long npp = d.n_pp < 0 ? np : d.n_pp;
        return (long long)g + 1 + std::max(0LL, (long long)g + 1 + npp - np);
    }
    throw InvalidArgument("lower_bound: symplectic mode takes one or two matrices");
}

// Packaged levels: the head x tail tile kernel when the cost model prefers it to the walk
// (same model as choose_tile, with the weighted element counts F / FR in place of binomials).
bool Plan::prepare_ptile(int g, LevelHost &lv, int world, int rank) {
    if (opts_.kernel == 1 || g < 2) return false;
    const unsigned long long total = level_candidates(g);
    if (opts_.kernel != 2 && total < (1ull << 16)) return false;
    const double Hl = heads_per_lane(W_, pd_.K), HBk = head_block(W_, pd_.K);
    const double slots = double(num_sms_) * tile_blocks_per_sm(W_, pd_.K) * std::max(1, world);
    double best_time = opts_.kernel == 2 ? 1e300 : double(total) * 28.0 / slots;
    int best_t = 0, best_chunk = kTailChunk;
    auto Hb_of = [&](int j, int b, int h) { return double(F_at(j, h_off_[size_t(j) * (P_ + 1) + b], h)); };
    auto Tb_of = [&](int j, int b, int t) {
        const int np = np_[size_t(j)];
        const short *off = h_off_.data() + size_t(j) * (P_ + 1);
        return double(off[b + 1] - off[b]) * double(FR_at(j, h_r_off_[size_t(j) * (P_ + 1) + (np - 1 - b)], t - 1));
    };
    for (int t = 1; t < g; t++) {
        const int h = g - t;
        for (int tchunk = kTailChunk; tchunk >= 64; tchunk /= 2) {
            double sum = 0, biggest = 0;
            for (int j = 0; j < G_; j++)
                for (int b = h; b <= np_[size_t(j)] - t; b++) {
                    const double Hb = Hb_of(j, b, h), Tb = Tb_of(j, b, t);
                    if (Hb <= 0 || Tb <= 0) continue;
                    const double nH = std::ceil(Hb / HBk), nT = std::ceil(Tb / tchunk);
                    const double heads_last = Hb - (nH - 1) * HBk;
                    const double warps_full = kTileThreads / 32.0, warps_last = std::ceil(heads_last / (32.0 * Hl));
                    const double tc = Tb / nT;
                    const double unit_full = warps_full * 32 * Hl * tc + 25000, unit_last = warps_last * 32 * Hl * tc + 25000;
                    sum += nT * ((nH - 1) * unit_full + unit_last);
                    biggest = std::max(biggest, nH > 1 ? unit_full : unit_last);
                }
            // the average load per CTA slot plus the tail: the last units finish unevenly,
            // about half the biggest unit late on average (this matters when sharding leaves
            // few units per CTA)
            const double time = std::max(sum / slots + 0.5 * biggest, biggest);
            if (time < best_time) {
                best_time = time;
                best_t = t;
                best_chunk = tchunk;
            }
        }
    }
    forced_tile(g, best_t, best_chunk);
    if (best_t == 0) return false;
    if (ptile_smem_bytes(G_, N_, W_, K_, P_, E_, std::min(BK_, g + 2)) > 200 * 1024) return false;
    PTilePlan &tp = lv.ptile;
    tp.g = g;
    tp.t = best_t;
    tp.h = g - best_t;
    tp.tchunk = best_chunk;
    tp.thr0 = ~0u;
    // (Gamma, b) pairs with work, their cumulative unit counts, then the pair codes
    std::vector<unsigned long long> cum;
    std::vector<unsigned> pairs;
    unsigned long long acc = 0;
    for (int j = 0; j < G_; j++)
        for (int b = tp.h; b <= np_[size_t(j)] - tp.t; b++) {
            const unsigned long long Hb = F_at(j, h_off_[size_t(j) * (P_ + 1) + b], tp.h);
            const int np = np_[size_t(j)];
            const short *off = h_off_.data() + size_t(j) * (P_ + 1);
            const unsigned long long Tb =
                (unsigned long long)(off[b + 1] - off[b]) * FR_at(j, h_r_off_[size_t(j) * (P_ + 1) + (np - 1 - b)], tp.t - 1);
            if (Hb == 0 || Tb == 0) continue;
            cum.push_back(acc);
            pairs.push_back(unsigned(j) << 16 | unsigned(b));
            acc += ((Hb + head_block(W_, pd_.K) - 1) / head_block(W_, pd_.K)) * ((Tb + tp.tchunk - 1) / tp.tchunk);
        }
    cum.push_back(acc);
    tp.npairs = int(pairs.size());
    const size_t n_entries = cum.size() + (pairs.size() + 1) / 2;
    if (table_used_ + n_entries > table_cap_) return false;
    unsigned long long *h_table = h_pinned_ + table_used_;
    std::copy(cum.begin(), cum.end(), h_table);
    std::memcpy(h_table + cum.size(), pairs.data(), pairs.size() * 4);
    tp.cum = d_tables_ + table_used_;
    tp.pairs = reinterpret_cast<const unsigned *>(d_tables_ + table_used_ + cum.size());
    tp.counter = d_counters_ + g;
    tp.unit_total = acc;
    tp.shard_rank = rank;
    tp.shard_world = world;
    table_used_ += n_entries;
    check_cuda(cudaMemcpyAsync(const_cast<unsigned long long *>(tp.cum), h_table, n_entries * 8, cudaMemcpyHostToDevice,
                               stream_),
               "H2D unit table");
    lv.t = -2;
    return true;
}

unsigned long long Plan::level_candidates(int g) const {
    if (!packaged_) return binom_u64(N_, g) * (unsigned long long)G_;
    unsigned long long t = 0;
    for (int j = 0; j < G_; j++) t += h_wsuf_[size_t(j) * (P_ + 1) * BK_ + size_t(g)];
    return t;
}

void Plan::prepare_level(int g) {
    LevelHost &lv = levels_[size_t(g)];
    if (lv.ready) return;
    // small levels run whole on every rank (identical results, no exchange); big ones shard
    const unsigned long long shard_min = opts_.shard_min > 0 ? (unsigned long long)opts_.shard_min : kDefaultShardMin;
    // (a one-rank communicator with shard_min = 1 takes the exchange path too: the single-GPU
    // test of the NCCL plumbing)
    lv.sharded = (opts_.world > 1 || (opts_.comm && opts_.shard_min == 1)) && level_candidates(g) >= shard_min;
    const int world = lv.sharded ? std::max(1, opts_.world) : 1, rank = lv.sharded ? opts_.rank : 0;
    if (packaged_) {
        if (g >= BK_) throw InvalidArgument("generation beyond the kernels' combination-size limit");
        // both packaged kernels key a candidate as Gamma << 58 | rank: check every Gamma's
        // level size before either is prepared
        for (int j = 0; j < G_; j++)
            if (h_wsuf_[size_t(j) * (P_ + 1) * BK_ + size_t(g)] >= (1ull << kKeyRankBits))
                throw InvalidArgument("level too large for 58-bit combination ranks");
        if (prepare_ptile(g, lv, world, rank)) {
            lv.ready = true;
            return;
        }
        PkgLevel &L = lv.pkg;
        L.g = g;
        L.thr0 = ~0u;
        unsigned long long total = 0;
        for (int j = 0; j < G_; j++) {
            L.total[j] = h_wsuf_[size_t(j) * (P_ + 1) * BK_ + size_t(g)];
            if (L.total[j] >= (1ull << kKeyRankBits))
                throw InvalidArgument("level too large for 58-bit combination ranks");
            total += L.total[j];
        }
        const unsigned long long threads_total = (unsigned long long)num_sms_ * 8 * 256;
        const unsigned long long threads_all = threads_total * (unsigned long long)world;
        L.seg_len = std::max<unsigned long long>(1, (total + threads_all - 1) / threads_all);
        L.seg_total = 0;
        for (int j = 0; j < G_; j++) {
            L.segs[j] = (L.total[j] + L.seg_len - 1) / L.seg_len;
            L.seg_total += L.segs[j];
        }
        L.shard_rank = rank;
        L.shard_world = world;
        lv.t = -1;
        lv.ready = true;
        return;
    }
    const unsigned long long per = binom_u64(N_, g);
    if (per >= (1ull << kKeyRankBits)) throw InvalidArgument("level too large for 58-bit combination ranks");
    const unsigned long long total = per * (unsigned long long)G_;
    if (tc_ok_ && opts_.kernel != 1 && opts_.kernel != 2 && g >= 2 &&
        (opts_.kernel == 4 || total >= kTcMinCandidates) && prepare_tc(g, lv, world, rank)) {
        if (std::getenv("SDB_TRACE_HOST"))
            std::fprintf(stderr, "[sdb] level %d: tensor-core tile t=%d nbt=%d units=%llu sharded=%d\n", g, lv.tc.tile.t,
                         lv.tc.nbt, (unsigned long long)lv.tc.tile.unit_total, int(lv.sharded));
        lv.ready = true;
        return;
    }
    TileChoice tc = choose_tile(G_, N_, g, W_, K_, per, opts_.kernel, num_sms_, world);
    forced_tile(g, tc.t, tc.tchunk);
    lv.t = tc.t;
    if (lv.t == 0) {
        LevelLaunch &LL = lv.walk;
        LL.g = g;
        LL.lprev = early_bound(g);
        LL.thr0 = ~0u;  // the kernels read U from the device (RunCtl)
        LL.per_gamma = per;
        const unsigned long long threads_total = (unsigned long long)num_sms_ * 8 * 256;
        // one segment per thread of the full grid: tiny levels get one candidate per thread
        // instead of a long serial walk on a few threads
        const unsigned long long threads_all = threads_total * (unsigned long long)world;  // every rank's grid
        LL.seg_len = std::max<unsigned long long>(1, (total + threads_all - 1) / threads_all);
        LL.segs_per_gamma = (per + LL.seg_len - 1) / LL.seg_len;
        const unsigned long long S = LL.segs_per_gamma * (unsigned long long)G_;
        LL.seg_total = S;
        LL.shard_rank = rank;
        LL.shard_world = world;
    } else {
        TilePlan &tp = lv.tile;
        tp.g = g;
        tp.lprev = early_bound(g);
        tp.t = lv.t;
        tp.h = g - lv.t;
        tp.thr0 = ~0u;
        tp.nb = N_ - lv.t - tp.h + 1;
        tp.tchunk = tc.tchunk;
        tp.per_gamma = per;
        const size_t n_entries = size_t(G_) * size_t(tp.nb) + 1;
        if (table_used_ + n_entries > table_cap_) throw InternalFailure("tile unit tables overflow");
        // staged in the plan's pinned buffer: the copy is truly asynchronous, no wait here
        unsigned long long *h_table = h_pinned_ + table_used_;
        unsigned long long acc = 0;
        for (int j = 0; j < G_; j++)
            for (int b = tp.h; b <= N_ - lv.t; b++) {
                h_table[size_t(j) * tp.nb + (b - tp.h)] = acc;
                const unsigned long long Hb = binom_u64(b, tp.h), Tb = binom_u64(N_ - 1 - b, lv.t - 1);
                acc += ((Hb + head_block(W_, pd_.K) - 1) / head_block(W_, pd_.K)) * ((Tb + tp.tchunk - 1) / tp.tchunk);
            }
        h_table[size_t(G_) * tp.nb] = acc;
        tp.unit_total = acc;
        tp.shard_rank = rank;
        tp.shard_world = world;
        tp.cum = d_tables_ + table_used_;
        tp.counter = d_counters_ + g;  // zeroed by run_init at the start of every run
        table_used_ += n_entries;
        check_cuda(cudaMemcpyAsync(const_cast<unsigned long long *>(tp.cum), h_table, n_entries * 8,
                                   cudaMemcpyHostToDevice, stream_),
                   "H2D unit table");
        if (tile_smem_bytes(G_, N_, W_, K_, std::min(BK_, g + 2)) > 200 * 1024)
            throw InvalidArgument("problem too large for shared-memory staging");
    }
    if (std::getenv("SDB_TRACE_HOST"))
        std::fprintf(stderr, "[sdb] level %d: %s t=%d tchunk=%d units=%llu segs=%llu seg_len=%llu sharded=%d\n", g,
                     lv.t ? "tile" : "walk", lv.t, lv.t ? lv.tile.tchunk : 0,
                     lv.t ? (unsigned long long)lv.tile.unit_total : 0ull,
                     lv.t ? 0ull : (unsigned long long)lv.walk.seg_total, lv.t ? 0ull : (unsigned long long)lv.walk.seg_len,
                     int(lv.sharded));
    lv.ready = true;
}

int Plan::launch_level(int g) {
    const LevelHost &lv = levels_[size_t(g)];
    const int nl = lv.t == -3  ? launch_tc_level(pd_, lv.tc, stream_, num_sms_)
                   : lv.t == -2 ? launch_ptile_level(pd_, pk_, pt_, lv.ptile, stream_, num_sms_)
                   : lv.t == -1 ? launch_pkg_level(pd_, pk_, lv.pkg, stream_, num_sms_)
                   : lv.t == 0  ? launch_walk_level(pd_, lv.walk, stream_, num_sms_)
                                : launch_tile_level(pd_, lv.tile, stream_, num_sms_);
    if (nl < 0) throw InvalidArgument("unsupported row width");
    check_cuda(cudaGetLastError(), "level kernel launch");
    return nl;
}

bool Plan::run_level(int g, long long upper, long long *upper_out, unsigned long long *candidates,
                     uint64_t *best_out) {
    check_cuda(cudaSetDevice(device_), "cudaSetDevice");
    if (G_ != 1) throw InvalidArgument("enumerate_generation: one generator matrix");
    const int np = packaged_ ? np_[0] : N_;
    if (g < 1 || g > np) throw InvalidArgument("enumerate_generation: generation out of range");
    if (g > kMaxLevel) throw InvalidArgument("generation beyond the kernels' combination-size limit");
    if (upper == 0) upper = sentinel_;  // BoundsState.upper == 0: unset (engine.cpp:299)
    *candidates = level_candidates(g);
    *upper_out = upper;
    if (upper < 0) return false;  // no weight lies below it
    // every weight is below the sentinel, so a larger incoming bound starts the device at it
    const unsigned start = unsigned(std::min<long long>(upper, sentinel_));
    launch_run_init(pd_, start, d_counter_init_, d_counters_, N_ + 1, stream_);
    check_cuda(cudaGetLastError(), "run init launch");
    single_level_ = true;
    prepare_level(g);
    launch_level(g);
    launch_level_close(pd_, g, 0, 0, stream_);  // lower 0: the close never terminates
    check_cuda(cudaGetLastError(), "level close launch");
    RunCtl ctl{};
    check_cuda(cudaMemcpyAsync(&ctl, pd_.ctl, sizeof ctl, cudaMemcpyDeviceToHost, stream_), "D2H ctl");
    check_cuda(cudaStreamSynchronize(stream_), "level sync");
    const bool improved = ctl.best_g == g && (long long)ctl.U < upper;
    *upper_out = improved ? (long long)ctl.U : upper;
    if (improved && best_out) {
        const unsigned long long r = ctl.best_key & ((1ull << kKeyRankBits) - 1);
        std::vector<uint64_t> acc(size_t(gammas_[0].matrix.stride), 0);
        unrank_best(g, 0, r, acc);
        std::copy(acc.begin(), acc.end(), best_out);
    }
    return improved;
}

// The level loop (reference run_bz, engine.cpp:303-343) with the bound state on the device:
// levels are enqueued without waiting; level_close folds each level into U, writes the
// trace entry and raises `done` once L(g) >= U, and every later kernel returns at once.
// The host waits only after levels big enough to matter (and, with several ranks, after
// every level for the min-allreduce of the level minimum).
void Plan::run(sdb_report *rep, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out, double *level_seconds) {
    check_cuda(cudaSetDevice(device_), "cudaSetDevice");
    const int world = std::max(1, opts_.world), rank = opts_.rank;
    if (rank < 0 || rank >= world) throw InvalidArgument("rank outside [0, world)");
    if (world > 1 && !opts_.allreduce_min && !opts_.comm)
        throw InvalidArgument("world > 1 needs a communicator (comm) or an allreduce_min callback");
    // every matrix generates the full code: the smallest package count closes the search
    // (engine.cpp:322-325)
    int g_limit = N_;
    if (packaged_) g_limit = *std::min_element(np_.begin(), np_.end());
    if (opts_.max_generation > 0) g_limit = std::min(g_limit, opts_.max_generation);
    if (g_limit > kMaxLevel) g_limit = kMaxLevel;  // checked again below if the run gets there
    constexpr unsigned long long kSyncCandidates = 1ull << 28;  // ~0.1 ms of kernel time
    // levels enqueued past the last check: a level after termination costs its (empty) launches,
    // so small codes (whose levels are all tiny) check every few levels
#ifndef SDB_MAX_UNCHECKED_LEVELS
#define SDB_MAX_UNCHECKED_LEVELS 4
#endif
    constexpr int kMaxUncheckedLevels = SDB_MAX_UNCHECKED_LEVELS;
    int launches = 0, last_g = 0, checked_g = 0;
    // A big level's termination check is deferred: its ctl copy and event are enqueued behind
    // it, the next level is prepared and enqueued, and only then does the host wait. The
    // device then never idles on the host's preparation of the next level; a level enqueued
    // after termination returns at once on the device (RunCtl.done).
    int pending_g = 0;
    cudaEvent_t check_ev = level_event(0);
    unsigned long long h2d = 0, d2h = 0;
    launches += launch_run_init(pd_, unsigned(sentinel_), d_counter_init_, d_counters_, N_ + 1, stream_);
    check_cuda(cudaGetLastError(), "run init launch");
    RunCtl ctl{};
    std::vector<unsigned char> h_state;
    bool stopped_early = false;  // a deferred check found the run done while level g failed to set up
    for (int g = 1; g <= g_limit; g++) {
        // Level g is set up before the previous big level's check resolves (deferred check).
        // If the setup fails (size limits, launch errors), resolve that check first: a run
        // that already terminated must report its result, not this level's error.
        try {
            prepare_level(g);
        } catch (...) {
            if (pending_g) {
                check_cuda(cudaEventSynchronize(check_ev), "level check");
                pending_g = 0;
                if (h_ctl_->done) {
                    stopped_early = true;
                    break;
                }
            }
            throw;
        }
        const LevelHost &lv = levels_[size_t(g)];
        // per-level events only when the caller wants per-level times; else one pair
        // around all levels (fewer API calls on small codes)
        if (level_seconds || g == 1) check_cuda(cudaEventRecord(level_event(2 * g), stream_), "event");
        try {
            launches += launch_level(g);
        } catch (...) {
            if (pending_g) {
                check_cuda(cudaEventSynchronize(check_ev), "level check");
                pending_g = 0;
                if (h_ctl_->done) {
                    stopped_early = true;
                    break;
                }
            }
            throw;
        }
        int from_keys = 0;
        if (lv.sharded && opts_.comm) {
            // stream-ordered NCCL min-allreduce of the per-weight best keys; level_close reads
            // the level minimum off them
            comm_allreduce_min_u64(opts_.comm, pd_.key_by_w, size_t(max_weight_ + 1), stream_);
            from_keys = 1;
        } else if (lv.sharded) {
            // min-allreduce of (level minimum, its key) across ranks through the host
            // callback, then hand the result to level_close through the same state fields
            const size_t sb = sizeof(LevelState) + size_t(max_weight_ + 1) * 8;
            h_state.resize(sb);
            check_cuda(cudaMemcpyAsync(h_state.data(), pd_.state, sb, cudaMemcpyDeviceToHost, stream_), "D2H state");
            check_cuda(cudaStreamSynchronize(stream_), "level sync");
            d2h += sb;
            LevelState st;
            std::memcpy(&st, h_state.data(), sizeof st);
            const unsigned long long *keys = reinterpret_cast<const unsigned long long *>(h_state.data() + sizeof st);
            uint64_t wmin = st.wmin == ~0u ? ~uint64_t(0) : uint64_t(st.wmin);
            uint64_t key = wmin != ~uint64_t(0) ? keys[wmin] : kNoKey;
            uint64_t v = wmin;
            if (opts_.allreduce_min(opts_.allreduce_ctx, &v, 1) != 0) throw DeviceFailure("allreduce_min failed");
            if (v != wmin) key = kNoKey;
            if (opts_.allreduce_min(opts_.allreduce_ctx, &key, 1) != 0) throw DeviceFailure("allreduce_min failed");
            static thread_local unsigned hw[2];
            static thread_local unsigned long long hk;
            hw[0] = v == ~uint64_t(0) ? ~0u : unsigned(v);
            hk = key;
            check_cuda(cudaMemcpyAsync(&pd_.state->wmin, &hw[0], 4, cudaMemcpyHostToDevice, stream_), "H2D wmin");
            h2d += 4;
            if (v != ~uint64_t(0)) {
                check_cuda(cudaMemcpyAsync(pd_.key_by_w + v, &hk, 8, cudaMemcpyHostToDevice, stream_), "H2D key");
                h2d += 8;
            }
        }
        launches += launch_level_close(pd_, g, lower_bound(g), from_keys, stream_);
        check_cuda(cudaGetLastError(), "level close launch");
        if (level_seconds) check_cuda(cudaEventRecord(level_event(2 * g + 1), stream_), "event");
        last_g = g;
        const unsigned long long total = level_candidates(g);
        if (pending_g) {
            // the previous big level's check, now that this level is queued behind it
            check_cuda(cudaEventSynchronize(check_ev), "level check");
            checked_g = pending_g;
            pending_g = 0;
            if (h_ctl_->done) break;
        }
        const bool last = g == g_limit;
        if (total >= kSyncCandidates && !last && !(lv.sharded && !opts_.comm)) {
            check_cuda(cudaMemcpyAsync(h_ctl_, pd_.ctl, sizeof ctl, cudaMemcpyDeviceToHost, stream_), "D2H ctl");
            check_cuda(cudaEventRecord(check_ev, stream_), "event");
            d2h += sizeof ctl;
            pending_g = g;
        } else if ((lv.sharded && !opts_.comm) || last || g - checked_g >= kMaxUncheckedLevels) {
            check_cuda(cudaMemcpyAsync(h_ctl_, pd_.ctl, sizeof ctl, cudaMemcpyDeviceToHost, stream_), "D2H ctl");
            check_cuda(cudaStreamSynchronize(stream_), "level sync");
            d2h += sizeof ctl;
            checked_g = g;
            if (h_ctl_->done) break;
        }
        if (!packaged_ && g == kMaxLevel && g < N_ && (opts_.max_generation <= 0 || opts_.max_generation > g))
            throw InvalidArgument("generation beyond the kernels' combination-size limit");
    }
    (void)stopped_early;  // the trace below ends at the last level launched either way
    if (!level_seconds) check_cuda(cudaEventRecord(level_event(1), stream_), "event");
    std::vector<int> tu(size_t(last_g + 1));
    check_cuda(cudaMemcpyAsync(&ctl, pd_.ctl, sizeof ctl, cudaMemcpyDeviceToHost, stream_), "D2H ctl");
    check_cuda(cudaMemcpyAsync(tu.data(), pd_.trace_upper, tu.size() * 4, cudaMemcpyDeviceToHost, stream_), "D2H trace");
    check_cuda(cudaStreamSynchronize(stream_), "run sync");
    d2h += sizeof ctl + tu.size() * 4;

    long long U = sentinel_;
    unsigned long long candidates = 0;
    double enum_s = 0;
    int generation = 0, n_levels = 0;
    bool complete = false;
    for (int g = 1; g <= last_g; g++) {
        if (tu[size_t(g)] < 0) break;  // enqueued after termination: skipped on the device
        U = tu[size_t(g)];
        const long long L = lower_bound(g);
        float ms = 0;
        if (level_seconds) {
            check_cuda(cudaEventElapsedTime(&ms, level_event(2 * g), level_event(2 * g + 1)), "event time");
            enum_s += ms * 1e-3;
        }
        candidates += level_candidates(g);
        generation = g;
        if (n_levels < trace_cap && trace) trace[n_levels] = sdb_trace_entry{g, L, U};
        if (level_seconds && n_levels < trace_cap) level_seconds[n_levels] = ms * 1e-3;
        n_levels++;
        if (L >= U) { complete = true; break; }
        if (g == (packaged_ ? *std::min_element(np_.begin(), np_.end()) : N_)) complete = true;
    }
    if (!level_seconds && last_g >= 1) {
        float ms = 0;
        check_cuda(cudaEventElapsedTime(&ms, level_event(2), level_event(1)), "event time");
        enum_s = ms * 1e-3;
    }
    if (complete && U >= sentinel_)
        throw InternalFailure("run_bz: no admissible codeword after complete enumeration; "
                              "input is not a valid normalizer matrix");
    const int best_g = ctl.best_g;
    const int best_j = best_g > 0 ? int(ctl.best_key >> kKeyRankBits) : -1;
    const unsigned long long best_r = best_g > 0 ? (ctl.best_key & ((1ull << kKeyRankBits) - 1)) : 0;
    rep->generations = generation;
    rep->candidates_enumerated = candidates;
    rep->trace_len = n_levels;
    rep->complete = complete ? 1 : 0;
    rep->upper = U;
    rep->candidates_visited = ctl.visited;
    rep->candidates_skipped = ctl.skipped;
    rep->enum_seconds = enum_s;
    rep->n_gammas = G_;
    rep->kernel_launches = launches;
    rep->best_generation = best_g;
    rep->best_gamma = best_j;
    rep->best_rank = best_r;
    rep->h2d_bytes += h2d;
    rep->d2h_bytes += d2h;
    if (generation >= 1) {
        const int t = levels_[size_t(generation)].t;
        rep->last_level_kernel = t == -3 ? 3 : t == -2 ? 5 : t == -1 ? 4 : t == 0 ? 1 : 2;
    }
    if (best_out) {
        const BitMat &m = gammas_[size_t(std::max(0, best_j))].matrix;
        std::vector<uint64_t> acc(size_t(m.stride), 0);
        if (best_g > 0) unrank_best(best_g, best_j, best_r, acc);
        std::copy(acc.begin(), acc.end(), best_out);
    }
}

// Host twin of the kernels' unranking: the codeword at lexicographic rank r of level g of
// Gamma j, in the reference's visiting order (engine.cpp:202-219).
void Plan::unrank_best(int g, int j, unsigned long long r, std::vector<uint64_t> &acc) const {
    const BitMat &m = gammas_[size_t(j)].matrix;
    if (!packaged_) {
        int v = 0;
        for (int i = 0; i < g; i++) {
            for (;; v++) {
                const unsigned long long cnt = binom_u64(N_ - 1 - v, g - 1 - i);
                if (r < cnt) break;
                r -= cnt;
            }
            for (int w = 0; w < m.stride; w++) acc[size_t(w)] ^= m.row(v)[w];
            v++;
        }
        return;
    }
    const auto &pk = gammas_[size_t(j)].packages;
    const unsigned long long *ws = h_wsuf_.data() + size_t(j) * (P_ + 1) * BK_;
    int q = 0;
    for (int i = 0; i < g; i++) {
        for (;; q++) {
            const unsigned long long sub = ws[size_t(q + 1) * BK_ + size_t(g - 1 - i)];
            const unsigned long long cnt = pk[size_t(q)].size() * sub;
            if (r < cnt) {
                const int row = pk[size_t(q)][size_t(r / sub)];
                r %= sub;
                for (int w = 0; w < m.stride; w++) acc[size_t(w)] ^= m.row(row)[w];
                break;
            }
            r -= cnt;
        }
        q++;
    }
}

// ------------------------------------------------------------------------------- batch

int run_brute(const BitMat &a, const sdb_run_options &o, double *device_seconds) {
    const int rows = a.rows, n = a.cols / 2, k = rows - n;
    if (rows > 28) throw InvalidArgument("brute_force_distance: 2^(n+k) enumeration is limited to n+k <= 28 rows");
    if (rows == 0) throw InvalidArgument("brute_force_distance: matrix has no rows");
    const int W = (n + 31) / 32;
    if (W > 4) throw InvalidArgument("brute_force_distance: rows too wide for the brute-force kernel (n > 128)");
    const bool filter = o.dual_filter && k >= 1;
    std::vector<uint32_t> h_rows(size_t(rows) * 2 * W, 0);
    std::vector<unsigned long long> h_syn(size_t(rows), 0);
    for (int r = 0; r < rows; r++) {
        extract_bits(a, r, 0, n, h_rows.data() + size_t(r) * 2 * W, W);
        extract_bits(a, r, n, n, h_rows.data() + size_t(r) * 2 * W + W, W);
        if (filter)
            for (int j = 0; j < rows; j++)
                if (symplectic_ip(a.row(r), a.row(j), n)) h_syn[size_t(r)] |= 1ull << j;
    }
    check_cuda(cudaSetDevice(o.device), "cudaSetDevice");
    int num_sms = 148;
    check_cuda(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, o.device), "cudaDeviceGetAttribute");
    cudaStream_t st = o.stream ? static_cast<cudaStream_t>(o.stream) : thread_stream(o.device);
    const size_t b_rows = align256(h_rows.size() * 4), b_syn = align256(h_syn.size() * 8), bytes = b_rows + b_syn + 256;
    void *mem = workspace_get(o.device, bytes);
    unsigned char *base = static_cast<unsigned char *>(mem);
    BruteDev b{};
    b.rows = reinterpret_cast<const uint32_t *>(base);
    b.syn = reinterpret_cast<const unsigned long long *>(base + b_rows);
    b.best = reinterpret_cast<unsigned int *>(base + b_rows + b_syn);
    b.n_rows = rows;
    b.W = W;
    b.filter = filter ? 1 : 0;
    b.block_log2 = rows > 20 ? 10 : 4;
    unsigned best = ~0u;
    cudaEvent_t e0 = event_get(o.device), e1 = event_get(o.device);
    try {
        check_cuda(cudaMemcpyAsync(base, h_rows.data(), h_rows.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
        check_cuda(cudaMemcpyAsync(base + b_rows, h_syn.data(), h_syn.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
        check_cuda(cudaMemsetAsync(b.best, 0xFF, 4, st), "memset");
        check_cuda(cudaEventRecord(e0, st), "event");
        if (launch_brute(b, st, num_sms) < 0) throw InvalidArgument("unsupported row width");
        check_cuda(cudaGetLastError(), "brute kernel launch");
        check_cuda(cudaEventRecord(e1, st), "event");
        check_cuda(cudaMemcpyAsync(&best, b.best, 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "brute sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (device_seconds) *device_seconds = ms * 1e-3;
    } catch (...) {
        event_put(o.device, e0);
        event_put(o.device, e1);
        workspace_put(o.device, bytes, mem);
        throw;
    }
    event_put(o.device, e0);
    event_put(o.device, e1);
    workspace_put(o.device, bytes, mem);
    if (best == ~0u) throw InternalFailure("brute_force_distance: no admissible codeword exists");
    return int(best);
}

// Batch with the prep on the device (one warp per code). Returns false, having written
// nothing, when some code needs more Gamma slots than the prep kernel keeps (the caller then
// runs the host-prep path).
// Device path of the batch: prep and the level loops both on the device, one H2D of the
// normalizers (with the binomial table) from pinned staging, one D2H of every result, and no
// host round trip in between (each code reads its own matrix count from the prep).
static void run_batch_device(const uint64_t *rows, int n_codes, int n_rows, int n_cols, int row_words,
                             const sdb_run_options &o, int *distances, int *statuses, int *generations,
                             sdb_trace_entry *traces, int *trace_lens, int trace_cap, double *device_seconds,
                             std::vector<int> &host_prep) {
    const int n = n_cols / 2, k = n_rows - n, N = n_rows, W = (n + 31) / 32;
    const int Gs = kPrepGammaSlots, SW = (o.dual_filter && k >= 1) ? 1 : 0, BK = std::min(N, kMaxLevel) + 2;
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    check_cuda(cudaSetDevice(o.device), "cudaSetDevice");
    cudaStream_t st = o.stream ? static_cast<cudaStream_t>(o.stream) : thread_stream(o.device);
    const std::vector<unsigned long long> h_binom = binom_table(N, BK);
    const size_t nc = size_t(n_codes);
    const size_t in_bytes = nc * N * row_words * 8, binom_bytes = h_binom.size() * 8;
    const size_t b_in = align256(in_bytes), b_binom = align256(binom_bytes), b_rows = align256(nc * Gs * N * 2 * W * 4),
                 b_syn = align256(std::max<size_t>(nc * Gs * N * SW, 1) * 8), b_def = align256(nc * Gs * 4),
                 b_int = align256(nc * 4), b_tr = align256(nc * N * 4);
    const size_t b_up = b_in + b_binom, b_out = 3 * b_int + 2 * b_tr;
    const size_t bytes = b_up + b_rows + b_syn + b_def + 2 * b_int + b_out;
    void *mem = workspace_get(o.device, bytes);
    unsigned char *h_up = static_cast<unsigned char *>(pinned_get(b_up));
    unsigned char *h_out = static_cast<unsigned char *>(pinned_get(b_out));
    cudaEvent_t e0 = event_get(o.device), e1 = event_get(o.device);
    struct Release {
        int dev;
        size_t bytes, b_up, b_out;
        void *p;
        unsigned char *h_up, *h_out;
        cudaEvent_t e0, e1;
        cudaStream_t st;
        ~Release() {
            cudaStreamSynchronize(st);
            workspace_put(dev, bytes, p);
            pinned_put(b_up, h_up);
            pinned_put(b_out, h_out);
            event_put(dev, e0);
            event_put(dev, e1);
        }
    } release{o.device, bytes, b_up, b_out, mem, h_up, h_out, e0, e1, st};
    unsigned char *q = static_cast<unsigned char *>(mem);
    auto take = [&q](size_t b) {
        unsigned char *p = q;
        q += b;
        return p;
    };
    unsigned char *d_up = take(b_up);
    BatchPrepDev pd{};
    pd.normalizers = reinterpret_cast<const unsigned long long *>(d_up);
    pd.rows = reinterpret_cast<uint32_t *>(take(b_rows));
    pd.syn = reinterpret_cast<unsigned long long *>(take(b_syn));
    pd.deficits = reinterpret_cast<int *>(take(b_def));
    pd.n_gammas = reinterpret_cast<int *>(take(b_int));
    pd.status = reinterpret_cast<int *>(take(b_int));
    unsigned char *d_out = take(b_out);
    BatchDev bd{};
    bd.binom = reinterpret_cast<const unsigned long long *>(d_up + b_in);
    bd.out_upper = reinterpret_cast<int *>(d_out);
    bd.out_generations = reinterpret_cast<int *>(d_out + b_int);
    bd.out_status = reinterpret_cast<int *>(d_out + 2 * b_int);
    bd.out_trace_lower = reinterpret_cast<int *>(d_out + 3 * b_int);
    bd.out_trace_upper = reinterpret_cast<int *>(d_out + 3 * b_int + b_tr);
    pd.in_words = row_words;
    pd.codes = n_codes;
    pd.N = N;
    pd.n = n;
    pd.W = W;
    pd.validate = o.validate;
    pd.filter = SW;
    pd.Gs = Gs;
    pd.force_rows = o.kernel == 1;
    const auto t1 = clk::now();
    std::memcpy(h_up, rows, in_bytes);
    std::memcpy(h_up + b_in, h_binom.data(), binom_bytes);
    const auto t2 = clk::now();
    check_cuda(cudaMemcpyAsync(d_up, h_up, b_up, cudaMemcpyHostToDevice, st), "H2D normalizers");
    check_cuda(cudaEventRecord(e0, st), "event");
    launch_batch_prep(pd, st);
    check_cuda(cudaGetLastError(), "batch prep launch");
    bd.rows = pd.rows;
    bd.syn = pd.syn;
    bd.deficits = pd.deficits;
    bd.in_status = pd.status;
    bd.n_gammas = pd.n_gammas;
    bd.codes = n_codes;
    bd.G = Gs;
    bd.Gs = Gs;
    bd.N = N;
    bd.W = W;
    bd.SW = SW;
    bd.BK = BK;
    bd.scale = 2;
    bd.sentinel = 3 * n + 1;
    bd.max_g = o.max_generation;
    // enough resident codes per SM to cover the per-code level barriers
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device);
    bd.threads = n_codes >= 4 * sms ? 128 : 256;
    bd.no_mitm = o.kernel == 1;
    if (problem_smem_bytes(Gs, N, W, SW, BK) > 200 * 1024) throw InvalidArgument("batch codes too large");
    if (launch_batch(bd, st) < 0) throw InvalidArgument("unsupported row width");
    check_cuda(cudaGetLastError(), "batch kernel launch");
    check_cuda(cudaEventRecord(e1, st), "event");
    check_cuda(cudaMemcpyAsync(h_out, d_out, b_out, cudaMemcpyDeviceToHost, st), "D2H results");
    const auto t3 = clk::now();
    check_cuda(cudaStreamSynchronize(st), "batch sync");
    const auto t4 = clk::now();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (device_seconds) *device_seconds = ms * 1e-3;
    const int *up = reinterpret_cast<const int *>(h_out), *gen = reinterpret_cast<const int *>(h_out + b_int),
              *stt = reinterpret_cast<const int *>(h_out + 2 * b_int),
              *tl = reinterpret_cast<const int *>(h_out + 3 * b_int),
              *tu = reinterpret_cast<const int *>(h_out + 3 * b_int + b_tr);
    for (int c = 0; c < n_codes; c++) {
        const size_t cc = size_t(c);
        distances[c] = -1;
        generations[c] = 0;
        trace_lens[c] = 0;
        statuses[c] = 0;
        if (stt[cc] == kBatchNeedsHostPrep) {
            host_prep.push_back(c);
            continue;
        }
        if (stt[cc] == 2) {  // the prep's validation / information_sets failure
            statuses[c] = SDB_ERR_VALIDATION;
            continue;
        }
        generations[c] = gen[cc];
        trace_lens[c] = gen[cc];
        for (int g = 0; g < gen[cc] && g < trace_cap; g++)
            traces[cc * trace_cap + g] = sdb_trace_entry{g + 1, tl[cc * N + g], tu[cc * N + g]};
        if (stt[cc] != 0 || up[cc] % 2 != 0)
            statuses[c] = SDB_ERR_INTERNAL;
        else
            distances[c] = up[cc] / 2;
    }
    if (std::getenv("SDB_TRACE_HOST")) {
        auto ms = [](clk::time_point a, clk::time_point b) { return 1e3 * std::chrono::duration<double>(b - a).count(); };
        std::fprintf(stderr, "[sdb] batch: setup %.3f, stage %.3f, launch %.3f, wait %.3f, unpack %.3f ms\n", ms(t0, t1),
                     ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, clk::now()));
    }
}

void run_batch(const uint64_t *rows, int n_codes, int n_rows, int n_cols, int row_words, const sdb_run_options &o,
               int *distances, int *statuses, int *generations, sdb_trace_entry *traces, int *trace_lens,
               int trace_cap, double *device_seconds) {
    if (n_codes <= 0) return;
    if (n_cols % 2 != 0 || n_cols == 0)
        throw InvalidArgument("StabilizerInstance: column count must be even and nonzero");
    {
        const int n = n_cols / 2, k = n_rows - n;
        // validate_normalizer's shape checks (distance.cpp:71-79) are per batch: one shape
        if (o.validate && (n_rows == 0 || k < 0 || n_rows > 2 * n)) {
            for (int c = 0; c < n_codes; c++) {
                statuses[c] = SDB_ERR_VALIDATION;
                distances[c] = -1;
                generations[c] = 0;
                trace_lens[c] = 0;
            }
            if (device_seconds) *device_seconds = 0;
            return;
        }
        if (o.kernel != 3 && n_rows >= 1 && n_rows <= kPrepMaxRows && n <= kPrepMaxN) {
            std::vector<int> redo;
            run_batch_device(rows, n_codes, n_rows, n_cols, row_words, o, distances, statuses, generations, traces,
                             trace_lens, trace_cap, device_seconds, redo);
            if (redo.empty()) return;
            // codes with more information sets than the device prep has slots: host prep
            std::vector<uint64_t> sub(redo.size() * size_t(n_rows) * size_t(row_words));
            for (size_t i = 0; i < redo.size(); i++)
                std::memcpy(sub.data() + i * n_rows * row_words, rows + size_t(redo[i]) * n_rows * row_words,
                            size_t(n_rows) * row_words * 8);
            const size_t m = redo.size();
            std::vector<int> d(m), s(m), g(m), tl(m);
            std::vector<sdb_trace_entry> tr(m * size_t(std::max(trace_cap, 1)));
            sdb_run_options oh = o;
            oh.kernel = 3;
            double dev2 = 0;
            run_batch(sub.data(), int(m), n_rows, n_cols, row_words, oh, d.data(), s.data(), g.data(), tr.data(),
                      tl.data(), trace_cap, &dev2);
            for (size_t i = 0; i < m; i++) {
                const int c = redo[i];
                distances[c] = d[i];
                statuses[c] = s[i];
                generations[c] = g[i];
                trace_lens[c] = tl[i];
                for (int e = 0; e < trace_cap; e++) traces[size_t(c) * trace_cap + e] = tr[i * trace_cap + e];
            }
            if (device_seconds) *device_seconds += dev2;
            return;
        }
    }
    if (n_cols % 2 != 0 || n_cols == 0)
        throw InvalidArgument("StabilizerInstance: column count must be even and nonzero");
    const int n = n_cols / 2, k = n_rows - n, N = n_rows;
    const int W = (n + 31) / 32;
    if (W > kMaxW) throw InvalidArgument("rows too wide for the enumeration kernels (n > 256)");
    struct Prepped {
        int status = 0;
        std::vector<GammaIn> gammas;
        std::vector<uint64_t> syn;
        int SW = 0;
    };
    std::vector<Prepped> pp(static_cast<size_t>(n_codes));
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nthreads = int(std::min<unsigned>(hw, unsigned(n_codes)));
    auto work = [&](int t) {
        for (int c = t; c < n_codes; c += nthreads) {
            Prepped &p = pp[size_t(c)];
            try {
                BitMat a = BitMat::from_words(rows + size_t(c) * n_rows * row_words, n_rows, n_cols, row_words);
                if (o.validate) {
                    Validation v = validate_normalizer(a);
                    if (!v.ok) { p.status = SDB_ERR_VALIDATION; continue; }
                }
                std::vector<InfoSet> is = information_sets(isometry_transform(a));
                for (InfoSet &s : is) p.gammas.push_back(GammaIn{std::move(s.matrix), s.rank_deficit});
                Filter f;
                f.enabled = o.dual_filter && k >= 1;
                if (f.enabled) f.rows = a;
                p.SW = build_syndromes(p.gammas, n, f, p.syn);
            } catch (const ValidationFailure &) {
                p.status = SDB_ERR_VALIDATION;
            } catch (const std::exception &) {
                p.status = SDB_ERR_INTERNAL;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nthreads; t++) pool.emplace_back(work, t);
    work(0);
    for (std::thread &t : pool) t.join();

    int G = 0, SW = 0;
    std::vector<int> live;
    for (int c = 0; c < n_codes; c++)
        if (pp[size_t(c)].status == 0) {
            live.push_back(c);
            G = std::max(G, int(pp[size_t(c)].gammas.size()));
            SW = std::max(SW, pp[size_t(c)].SW);
        }
    for (int c = 0; c < n_codes; c++) {
        statuses[c] = pp[size_t(c)].status;
        distances[c] = -1;
        generations[c] = 0;
        trace_lens[c] = 0;
    }
    if (device_seconds) *device_seconds = 0;
    if (live.empty()) return;
    const int nl = int(live.size());
    const int BK = std::min(N, kMaxLevel) + 2;
    std::vector<uint32_t> h_rows(size_t(nl) * G * N * 2 * W, 0);
    std::vector<uint64_t> h_syn(size_t(nl) * G * N * SW, 0);
    std::vector<int> h_def(size_t(nl) * G, 1 << 20);
    for (int li = 0; li < nl; li++) {
        const Prepped &p = pp[size_t(live[size_t(li)])];
        for (int j = 0; j < G; j++) {
            // codes with fewer matrices repeat their first one with a deficit that never
            // contributes to L (duplicates cannot lower the minimum)
            const int src = j < int(p.gammas.size()) ? j : 0;
            const BitMat &m = p.gammas[size_t(src)].matrix;
            if (j < int(p.gammas.size())) h_def[size_t(li) * G + j] = p.gammas[size_t(j)].rank_deficit;
            for (int r = 0; r < N; r++) {
                uint32_t *dst = h_rows.data() + ((size_t(li) * G + j) * N + r) * 2 * W;
                extract_bits(m, r, 0, n, dst, W);
                extract_bits(m, r, n, n, dst + W, W);
                for (int s = 0; s < p.SW; s++)
                    h_syn[((size_t(li) * G + j) * N + r) * SW + s] = p.syn[(size_t(src) * N + r) * p.SW + s];
            }
        }
    }
    std::vector<unsigned long long> h_binom = binom_table(N, BK);
    check_cuda(cudaSetDevice(o.device), "cudaSetDevice");
    cudaStream_t st;
    check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    const size_t b_rows = align256(h_rows.size() * 4), b_syn = align256(std::max<size_t>(h_syn.size(), 1) * 8),
                 b_def = align256(h_def.size() * 4), b_binom = align256(h_binom.size() * 8),
                 b_out = align256(size_t(nl) * 4);
    const size_t b_tr = align256(size_t(nl) * N * 4);
    void *mem = nullptr;
    check_cuda(cudaMalloc(&mem, b_rows + b_syn + b_def + b_binom + 3 * b_out + 2 * b_tr), "cudaMalloc");
    unsigned char *base = static_cast<unsigned char *>(mem);
    BatchDev bd{};
    bd.rows = reinterpret_cast<const uint32_t *>(base);
    bd.syn = reinterpret_cast<const unsigned long long *>(base + b_rows);
    bd.deficits = reinterpret_cast<const int *>(base + b_rows + b_syn);
    bd.binom = reinterpret_cast<const unsigned long long *>(base + b_rows + b_syn + b_def);
    unsigned char *outp = base + b_rows + b_syn + b_def + b_binom;
    bd.out_upper = reinterpret_cast<int *>(outp);
    bd.out_generations = reinterpret_cast<int *>(outp + b_out);
    bd.out_status = reinterpret_cast<int *>(outp + 2 * b_out);
    bd.out_trace_lower = reinterpret_cast<int *>(outp + 3 * b_out);
    bd.out_trace_upper = reinterpret_cast<int *>(outp + 3 * b_out + b_tr);
    bd.codes = nl;
    bd.G = G;
    bd.N = N;
    bd.W = W;
    bd.SW = SW;
    bd.BK = BK;
    bd.scale = 2;
    bd.sentinel = 3 * n + 1;
    bd.Gs = G;
    bd.in_status = nullptr;
    bd.max_g = o.max_generation;
    try {
        check_cuda(cudaMemcpyAsync(base, h_rows.data(), h_rows.size() * 4, cudaMemcpyHostToDevice, st), "H2D");
        if (!h_syn.empty())
            check_cuda(cudaMemcpyAsync(base + b_rows, h_syn.data(), h_syn.size() * 8, cudaMemcpyHostToDevice, st), "H2D");
        check_cuda(cudaMemcpyAsync(base + b_rows + b_syn, h_def.data(), h_def.size() * 4, cudaMemcpyHostToDevice, st),
                   "H2D");
        check_cuda(cudaMemcpyAsync(base + b_rows + b_syn + b_def, h_binom.data(), h_binom.size() * 8,
                                   cudaMemcpyHostToDevice, st),
                   "H2D");
        if (problem_smem_bytes(G, N, W, SW, BK) > 200 * 1024) throw InvalidArgument("batch codes too large");
        cudaEvent_t e0, e1;
        check_cuda(cudaEventCreate(&e0), "event");
        check_cuda(cudaEventCreate(&e1), "event");
        check_cuda(cudaEventRecord(e0, st), "event");
        if (launch_batch(bd, st) < 0) throw InvalidArgument("unsupported row width");
        check_cuda(cudaGetLastError(), "batch kernel launch");
        check_cuda(cudaEventRecord(e1, st), "event");
        const size_t nls = static_cast<size_t>(nl);
        std::vector<int> up(nls), gen(nls), stt(nls), tl(nls * N), tu(nls * N);
        check_cuda(cudaMemcpyAsync(up.data(), bd.out_upper, size_t(nl) * 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaMemcpyAsync(gen.data(), bd.out_generations, size_t(nl) * 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaMemcpyAsync(stt.data(), bd.out_status, size_t(nl) * 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaMemcpyAsync(tl.data(), bd.out_trace_lower, size_t(nl) * N * 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaMemcpyAsync(tu.data(), bd.out_trace_upper, size_t(nl) * N * 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "batch sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (device_seconds) *device_seconds = ms * 1e-3;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        for (int li = 0; li < nl; li++) {
            const int c = live[size_t(li)];
            generations[c] = gen[size_t(li)];
            trace_lens[c] = gen[size_t(li)];
            for (int g = 0; g < gen[size_t(li)] && g < trace_cap; g++)
                traces[size_t(c) * trace_cap + g] =
                    sdb_trace_entry{g + 1, tl[size_t(li) * N + g], tu[size_t(li) * N + g]};
            if (stt[size_t(li)] != 0) {
                statuses[c] = SDB_ERR_INTERNAL;
            } else if (up[size_t(li)] % 2 != 0) {
                statuses[c] = SDB_ERR_INTERNAL;
            } else {
                distances[c] = up[size_t(li)] / 2;
            }
        }
    } catch (...) {
        cudaFree(mem);
        cudaStreamDestroy(st);
        throw;
    }
    cudaFree(mem);
    cudaStreamDestroy(st);
}

}  // namespace sdb
