// sm_100a enumeration kernels for the symplectic Brouwer-Zimmermann hot path.
//
//   walk_kernel<W>   small / mid levels: each thread unranks the first combination of
//                    a segment of consecutive lexicographic ranks (combinatorial number
//                    system) and walks the segment with the lexicographic successor,
//                    updating the running XOR of its rows; weight = scale * sum popc(x|z).
//   batch_kernel<W>  one code per CTA, the whole level loop (U, L, trace) on the device
//                    (BASELINE config 3).
//
// Improving candidates (weight <= running threshold) take the rare path: compressed
// admissibility syndrome (reference AdmissibilityFilter, engine.cpp:14-29), then
// atomicMin on the level minimum and on the per-weight best key (Gamma << 58 | rank),
// so the reported best codeword is the first one in the reference's visiting order.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.hpp"
#include "tc_ptx.cuh"

namespace sdb {

namespace {

// Opt a kernel into up to 200 KB of dynamic shared memory, once per device (the attribute
// is per device; a process may drive several GPUs).
template <auto Kernel>
void allow_big_smem() {
    static std::atomic<unsigned long long> done{0};  // one per kernel (Kernel is a value)
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done.fetch_or(bit, std::memory_order_acq_rel);
}

__device__ __forceinline__ unsigned long long binom_at(const unsigned long long *b, int BK, int a, int k) {
    if (k < 0 || a < 0 || k > a) return 0ull;
    return b[a * BK + k];
}

// lexicographic unrank of `r` into g ascending elements of [0, N)
__device__ __forceinline__ void unrank_lex(unsigned long long r, int g, int N, const unsigned long long *binom,
                                           int BK, int *c) {
    int v = 0;
    for (int i = 0; i < g; i++) {
        for (;; v++) {
            const unsigned long long cnt = binom_at(binom, BK, N - 1 - v, g - 1 - i);
            if (r < cnt) break;
            r -= cnt;
        }
        c[i] = v++;
    }
}

template <int W>
__device__ __forceinline__ void xor_row(uint32_t (&acc)[2 * W], const uint32_t *row) {
#pragma unroll
    for (int i = 0; i < 2 * W; i++) acc[i] ^= row[i];
}

template <int W>
__device__ __forceinline__ int weight_of(const uint32_t (&acc)[2 * W]) {
    int w = 0;
#pragma unroll
    for (int i = 0; i < W; i++) w += __popc(acc[i] | acc[W + i]);
    return w;
}

__device__ __forceinline__ bool admissible_combo(const unsigned long long *syn, int SW, const int *c, int g) {
    if (SW == 0) return true;
    for (int s = 0; s < SW; s++) {
        unsigned long long x = 0;
        for (int i = 0; i < g; i++) x ^= syn[c[i] * SW + s];
        if (x) return true;
    }
    return false;
}

__device__ __forceinline__ bool run_done(const ProblemDev &p) { return *(volatile int *)&p.ctl->done != 0; }

// threshold at kernel start: weights <= U - 1 can still lower U (engine units)
// Mid-level early exit. Every codeword not enumerated by levels < g weighs at least L(g-1),
// and U > L(g-1) when level g starts, so a level-g candidate never weighs less than L(g-1);
// once the level minimum reaches L(g-1) it is the distance and level g's close will stop the
// run with the same (g, L, U). What may still change is `best`, the first minimal candidate in
// the reference's order (Gamma, lexicographic rank): work whose keys all exceed the current
// key of that weight cannot lower it. Returns that key, or ~0 while the exit does not apply.
__device__ __forceinline__ unsigned long long early_key(const ProblemDev &p, unsigned lprev) {
    const unsigned w = *(volatile unsigned *)&p.state->wmin;
    if (lprev == 0 || w > lprev) return ~0ull;
    return *(volatile unsigned long long *)&p.key_by_w[w];
}

__device__ __forceinline__ unsigned start_threshold(const ProblemDev &p, unsigned thr0) {
    const unsigned U = *(volatile unsigned *)&p.ctl->U;
    return min(min(thr0, U - 1u), *(volatile unsigned *)&p.state->wmin);
}

__global__ void run_init_kernel(ProblemDev p, unsigned sentinel, const unsigned long long *counter_init,
                                unsigned long long *counters, int n_counters) {
    if (threadIdx.x == 0) {
        p.ctl->U = sentinel;
        p.ctl->done = 0;
        p.ctl->best_g = -1;
        p.ctl->best_key = ~0ull;
        p.ctl->visited = 0;
        p.ctl->skipped = 0;
        p.state->wmin = ~0u;
        p.state->visited = 0;
        p.state->skipped = 0;
    }
    for (int i = threadIdx.x; i <= p.max_weight; i += blockDim.x) p.key_by_w[i] = ~0ull;
    for (int i = threadIdx.x; i <= p.N; i += blockDim.x) p.trace_upper[i] = -1;
    for (int i = threadIdx.x; i < n_counters; i += blockDim.x) counters[i] = counter_init[i];
}

// Reference run_bz level barrier (engine.cpp:327-335): U from the level minimum (admissible
// candidates only, already filtered in the kernels), trace entry, stop when L >= U.
__global__ void level_close_kernel(ProblemDev p, int g, long long lower, int from_keys) {
    __shared__ unsigned s_w;
    if (from_keys) {
        // after the cross-rank min-allreduce of key_by_w: the level minimum is the smallest
        // weight any rank keyed
        if (threadIdx.x == 0) s_w = ~0u;
        __syncthreads();
        for (int i = threadIdx.x; i <= p.max_weight; i += blockDim.x)
            if (p.key_by_w[i] != ~0ull) atomicMin(&s_w, unsigned(i));
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        RunCtl *c = p.ctl;
        if (!c->done) {
            const unsigned w = from_keys ? s_w : p.state->wmin;
            if (w != ~0u && w < c->U) {
                c->U = w;
                c->best_g = g;
                c->best_key = p.key_by_w[w];
            }
            p.trace_upper[g] = int(c->U);
            c->visited += p.state->visited;
            c->skipped += p.state->skipped;
            if (lower >= (long long)c->U) c->done = 1;
        }
        p.state->wmin = ~0u;
        p.state->visited = 0;
        p.state->skipped = 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= p.max_weight; i += blockDim.x) p.key_by_w[i] = ~0ull;
}

template <int W>
__global__ void __launch_bounds__(256) walk_kernel(ProblemDev p, LevelLaunch L) {
    if (run_done(p)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const int rowlen = 2 * W;
    const int nrow_words = p.G * p.N * rowlen;
    // rows, syndromes and the binomial columns C(., k < g) the level's unranks read (a small
    // level would spend most of its time staging the whole table)
    const int BKs = max(1, min(p.BK, L.g));
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem);
    unsigned long long *s_syn = reinterpret_cast<unsigned long long *>(smem + ((nrow_words * 4 + 15) & ~15));
    const int nsyn = p.G * p.N * p.SW;
    unsigned long long *s_binom = s_syn + nsyn;
    const int nbinom = (p.N + 1) * BKs;
    for (int i = threadIdx.x; i < nrow_words; i += blockDim.x) s_rows[i] = p.rows[i];
    for (int i = threadIdx.x; i < nsyn; i += blockDim.x) s_syn[i] = p.syn[i];
    for (int i = threadIdx.x; i < nbinom; i += blockDim.x) s_binom[i] = p.binom[(i / BKs) * p.BK + i % BKs];
    __syncthreads();

    const int g = L.g, N = p.N;
    unsigned int thr = start_threshold(p, L.thr0);
    unsigned long long visited = 0, skipped = 0;
    int c[kMaxLevel];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long it = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;; it += stride) {
        const unsigned long long seg = it * L.shard_world + L.shard_rank;
        if (seg >= L.seg_total) break;
        const int j = int(seg / L.segs_per_gamma);
        const unsigned long long r0 = (seg % L.segs_per_gamma) * L.seg_len;
        const unsigned long long r1 = min(r0 + L.seg_len, L.per_gamma);
        if ((((unsigned long long)j << kKeyRankBits) | r0) > early_key(p, L.lprev)) {
            skipped += r1 - r0;  // every key of the segment exceeds the best one (early exit)
            continue;
        }
        const uint32_t *grows = s_rows + j * N * rowlen;
        const unsigned long long *gsyn = s_syn + j * N * p.SW;
        unrank_lex(r0, g, N, s_binom, BKs, c);
        for (int i = 0; i < g; i++) SDB_CHECK(c[i] >= 0 && c[i] < N && (i == 0 || c[i] > c[i - 1]));
        uint32_t acc[2 * W];
#pragma unroll
        for (int i = 0; i < 2 * W; i++) acc[i] = 0;
        for (int i = 0; i < g; i++) xor_row<W>(acc, grows + c[i] * rowlen);
        unsigned long long r = r0;
        for (;;) {
            const unsigned int w = unsigned(p.scale * weight_of<W>(acc));
            if (w <= thr) {
                if (admissible_combo(gsyn, p.SW, c, g)) {
                    atomicMin(&p.state->wmin, w);
                    atomicMin(&p.key_by_w[w], ((unsigned long long)j << kKeyRankBits) | r);
                    thr = w;
                }
            }
            if (++r >= r1) break;
            // lexicographic successor: bump the rightmost element that can move
            int i = g - 1;
            while (c[i] == N - g + i) i--;
            for (int m = i; m < g; m++) xor_row<W>(acc, grows + c[m] * rowlen);
            c[i]++;
            for (int m = i + 1; m < g; m++) c[m] = c[m - 1] + 1;
            for (int m = i; m < g; m++) xor_row<W>(acc, grows + c[m] * rowlen);
        }
        visited += r1 - r0;
        thr = min(thr, *(volatile unsigned int *)&p.state->wmin);
    }
    // one atomic per warp for the visit counter
    for (int o = 16; o > 0; o >>= 1) {
        visited += __shfl_down_sync(0xffffffffu, visited, o);
        skipped += __shfl_down_sync(0xffffffffu, skipped, o);
    }
    if ((threadIdx.x & 31) == 0 && visited) atomicAdd(&p.state->visited, visited);
    if ((threadIdx.x & 31) == 0 && skipped) atomicAdd(&p.state->skipped, skipped);
}

// ---------------------------------------------------------------- packages (1/3-packages)

__host__ __device__ size_t pkg_layout(int G, int N, int W, int SW, int P, int BK, size_t *o_syn, size_t *o_pr, size_t *o_ps,
                                      size_t *o_ws) {
    size_t off = ((size_t(G) * N * 2 * W * 4) + 15) & ~size_t(15);
    *o_syn = off;
    off += size_t(G) * N * SW * 8;
    *o_pr = off;
    off += ((size_t(G) * P * 3 * 2) + 15) & ~size_t(15);
    *o_ps = off;
    off += ((size_t(G) * P) + 15) & ~size_t(15);
    *o_ws = off;
    off += size_t(G) * (P + 1) * BK * 8;
    return off;
}

template <int W>
__global__ void __launch_bounds__(256) pkg_kernel(ProblemDev p, PkgDev k, PkgLevel L) {
    if (run_done(p)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const int rowlen = 2 * W, G = p.G, N = p.N, SW = p.SW, P = k.P, BK = p.BK;
    size_t o_syn, o_pr, o_ps, o_ws;
    pkg_layout(G, N, W, SW, P, BK, &o_syn, &o_pr, &o_ps, &o_ws);
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem);
    unsigned long long *s_syn = reinterpret_cast<unsigned long long *>(smem + o_syn);
    short *s_pr = reinterpret_cast<short *>(smem + o_pr);
    unsigned char *s_ps = smem + o_ps;
    unsigned long long *s_ws = reinterpret_cast<unsigned long long *>(smem + o_ws);
    for (int i = threadIdx.x; i < G * N * rowlen; i += blockDim.x) s_rows[i] = p.rows[i];
    for (int i = threadIdx.x; i < G * N * SW; i += blockDim.x) s_syn[i] = p.syn[i];
    for (int i = threadIdx.x; i < G * P * 3; i += blockDim.x) s_pr[i] = k.pk_rows[i];
    for (int i = threadIdx.x; i < G * P; i += blockDim.x) s_ps[i] = k.pk_size[i];
    for (int i = threadIdx.x; i < G * (P + 1) * BK; i += blockDim.x) s_ws[i] = k.wsuf[i];
    __syncthreads();

    const int g = L.g;
    unsigned thr = start_threshold(p, L.thr0);
    unsigned long long visited = 0;
    int pk[kMaxLevel], d[kMaxLevel];
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long it = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;; it += stride) {
        unsigned long long seg = it * L.shard_world + L.shard_rank;
        if (seg >= L.seg_total) break;
        int j = 0;
        while (seg >= L.segs[j]) seg -= L.segs[j++];
        const int np = k.np[j];
        const unsigned long long r0 = seg * L.seg_len, r1 = min(r0 + L.seg_len, L.total[j]);
        const uint32_t *grows = s_rows + j * N * rowlen;
        const unsigned long long *gsyn = s_syn + j * N * SW;
        const short *prow = s_pr + j * P * 3;
        const unsigned char *psz = s_ps + j * P;
        const unsigned long long *ws = s_ws + size_t(j) * (P + 1) * BK;  // ws[q * BK + m]
        // unrank r0 in the reference's order: (package, member) pairs, lexicographic
        uint32_t acc[2 * W];
#pragma unroll
        for (int i = 0; i < 2 * W; i++) acc[i] = 0;
        {
            unsigned long long rho = r0;
            int q = 0;
            for (int i = 0; i < g; i++) {
                for (;; q++) {
                    const unsigned long long sub = ws[(q + 1) * BK + (g - 1 - i)];
                    const unsigned long long cnt = psz[q] * sub;
                    if (rho < cnt) {
                        pk[i] = q;
                        d[i] = int(rho / sub);
                        rho %= sub;
                        break;
                    }
                    rho -= cnt;
                }
                xor_row<W>(acc, grows + prow[q * 3 + d[i]] * rowlen);
                q++;
            }
        }
        unsigned long long r = r0;
        for (;;) {
            const unsigned w = unsigned(p.scale * weight_of<W>(acc));
            if (w <= thr) {
                bool adm = SW == 0;
                for (int s = 0; s < SW && !adm; s++) {
                    unsigned long long x = 0;
                    for (int i = 0; i < g; i++) x ^= gsyn[prow[pk[i] * 3 + d[i]] * SW + s];
                    adm = x != 0;
                }
                if (adm) {
                    atomicMin(&p.state->wmin, w);
                    atomicMin(&p.key_by_w[w], ((unsigned long long)j << kKeyRankBits) | r);
                    thr = w;
                }
            }
            if (++r >= r1) break;
            // successor: the deepest position that can take its next member or next package
            int i = g - 1;
            while (d[i] + 1 >= psz[pk[i]] && pk[i] + 1 > np - (g - i)) i--;
            for (int m = i; m < g; m++) xor_row<W>(acc, grows + prow[pk[m] * 3 + d[m]] * rowlen);
            if (d[i] + 1 < psz[pk[i]]) {
                d[i]++;
            } else {
                pk[i]++;
                d[i] = 0;
            }
            for (int m = i + 1; m < g; m++) {
                pk[m] = pk[m - 1] + 1;
                d[m] = 0;
            }
            for (int m = i; m < g; m++) xor_row<W>(acc, grows + prow[pk[m] * 3 + d[m]] * rowlen);
        }
        visited += r1 - r0;
        thr = min(thr, *(volatile unsigned int *)&p.state->wmin);
    }
    for (int o = 16; o > 0; o >>= 1) visited += __shfl_down_sync(0xffffffffu, visited, o);
    if ((threadIdx.x & 31) == 0 && visited) atomicAdd(&p.state->visited, visited);
}

template <int W>
int launch_pkg_impl(const ProblemDev &p, const PkgDev &k, const PkgLevel &L, cudaStream_t st, int num_sms) {
    size_t a, b, c, d;
    const size_t smem = pkg_layout(p.G, p.N, W, p.SW, k.P, p.BK, &a, &b, &c, &d);
    allow_big_smem<pkg_kernel<W>>();
    const unsigned long long segs = (L.seg_total + L.shard_world - 1 - L.shard_rank) / L.shard_world;
    unsigned long long blocks = (segs + 255) / 256;
    const unsigned long long cap = (unsigned long long)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) return 0;
    pkg_kernel<W><<<unsigned(blocks), 256, smem, st>>>(p, k, L);
    return 1;
}

// ---------------------------------------------------------------- brute force (Gray walk)

template <int W>
__global__ void __launch_bounds__(256) brute_kernel(BruteDev b) {
    __shared__ uint32_t s_rows[32 * 2 * W];
    __shared__ unsigned long long s_syn[32];
    for (int i = threadIdx.x; i < b.n_rows * 2 * W; i += blockDim.x) s_rows[i] = b.rows[i];
    for (int i = threadIdx.x; i < b.n_rows; i += blockDim.x) s_syn[i] = b.filter ? b.syn[i] : 0ull;
    __syncthreads();
    const unsigned long long total = (1ull << b.n_rows) - 1;  // m = 1 .. total
    const unsigned long long nblk = (total + (1ull << b.block_log2)) >> b.block_log2;
    unsigned best = ~0u;
    for (unsigned long long blk = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; blk < nblk;
         blk += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long m0 = max(1ull, blk << b.block_log2);
        const unsigned long long m1 = min(total + 1, (blk + 1) << b.block_log2);
        // state after index m0 - 1: the rows of gray(m0 - 1)
        uint32_t acc[2 * W];
#pragma unroll
        for (int w = 0; w < 2 * W; w++) acc[w] = 0;
        unsigned long long syn = 0;
        const unsigned long long g0 = (m0 - 1) ^ ((m0 - 1) >> 1);
        for (int r = 0; r < b.n_rows; r++)
            if ((g0 >> r) & 1ull) {
                xor_row<W>(acc, s_rows + r * 2 * W);
                syn ^= s_syn[r];
            }
        for (unsigned long long m = m0; m < m1; m++) {
            const int flip = __ffsll((long long)m) - 1;
            xor_row<W>(acc, s_rows + flip * 2 * W);
            syn ^= s_syn[flip];
            if (b.filter && syn == 0) continue;
            best = min(best, unsigned(weight_of<W>(acc)));
        }
    }
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_down_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0u) atomicMin(b.best, best);
}

// ---------------------------------------------------------------- batch: one code per CTA

// Meet-in-the-middle levels of the batch kernel. The rows of one matrix split into halves
// A = [0, nA) and B = [nA, N); list L_h of a half holds the XOR sums and the admissibility
// syndromes of its h-subsets in colex order, so the g-combinations are exactly the pairs
// A_h x B_(g-h), h = 0..g. The lists stay resident from level to level (level g adds L_g).
// Pairs with an empty side (h = 0 or h = g) are the new L_g entries themselves: they are
// scored while L_g is built, and the deepest level scores its L_g without storing it.
template <int W>
struct MitmEnt;
template <>
struct MitmEnt<1> {
    using T = uint2;
    static __device__ __forceinline__ T load_row(const uint32_t *r) { return make_uint2(r[0], r[1]); }
    static __device__ __forceinline__ T x(T a, T b) { return make_uint2(a.x ^ b.x, a.y ^ b.y); }
    static __device__ __forceinline__ unsigned weight(T a) { return __popc(a.x | a.y); }
    static __device__ __forceinline__ unsigned weight(T a, T b) { return __popc((a.x ^ b.x) | (a.y ^ b.y)); }
};
template <>
struct MitmEnt<2> {
    using T = uint4;  // (x0, x1, z0, z1)
    static __device__ __forceinline__ T load_row(const uint32_t *r) { return make_uint4(r[0], r[1], r[2], r[3]); }
    static __device__ __forceinline__ T x(T a, T b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }
    static __device__ __forceinline__ unsigned weight(T a) { return __popc(a.x | a.z) + __popc(a.y | a.w); }
    static __device__ __forceinline__ unsigned weight(T a, T b) {
        return __popc((a.x ^ b.x) | (a.z ^ b.z)) + __popc((a.y ^ b.y) | (a.w ^ b.w));
    }
};

// matrices whose lists stay resident: the device prep's slots
constexpr int kMitmSlots = kPrepGammaSlots;

// first entry of L_h in an n-element half: sum of C(n, s), s < h
__device__ __forceinline__ int mitm_off(const unsigned long long *binom, int BK, int n, int h) {
    int e = 0;
    for (int s = 0; s < h; s++) e += int(binom[n * BK + s]);
    return e;
}

// where the lists of one matrix live: A's L_0..L_(stored-1), then B's
constexpr int kMitmMaxLevel = 15;
struct MitmView {
    int nA, nB;
    int stored;   // lists L_0 .. L_(stored-1) are resident (stored = mitm_g: L_mitm_g never is)
    int blockB;   // first entry of B's lists
    int stride;   // entries per matrix
    const int *cnt;  // [2][kMitmMaxLevel + 1]: C(n_half, h)
    const int *off;  // [2][kMitmMaxLevel + 1]: first entry of L_h (B's include blockB)
};

__device__ __forceinline__ void mitm_candidate(unsigned w, unsigned long long syn, int SW, unsigned scale,
                                               unsigned &best, unsigned &wlim) {
    if (w < wlim && (SW == 0 || syn != 0ull)) {
        best = scale * w;
        wlim = w;
    }
}

// L_g of both halves of every matrix from the resident L_(g-1), each entry scored as a
// candidate on its own (its pair with the other half's empty subset), and stored when a
// deeper level will read it. In colex order the g-subsets with maximum m come after those
// with maximum < m, and their first g - 1 elements are the first C(m, g-1) entries of L_(g-1).
template <int W>
__device__ __forceinline__ void mitm_build(int g, int G, int N, const uint32_t *s_rows, const unsigned long long *s_syn,
                                           int SW, const unsigned long long *binom, int BK, const MitmView &v,
                                           typename MitmEnt<W>::T *ent, unsigned long long *esyn, unsigned scale,
                                           unsigned &best, unsigned &wlim) {
    using E = MitmEnt<W>;
    const bool store = g < v.stored;
    constexpr int K = kMitmMaxLevel + 1;
    for (int j = 0; j < G; j++) {
        typename E::T *L = ent + j * v.stride;
        unsigned long long *S = esyn + j * v.stride;
        const uint32_t *rows = s_rows + j * N * 2 * W;
        const unsigned long long *syn = s_syn + j * N * SW;
        for (int half = 0; half < 2; half++) {
            const int n = half ? v.nB : v.nA, base = half ? v.nA : 0;
            const int c = v.cnt[half * K + g], dst0 = v.off[half * K + g], src0 = v.off[half * K + g - 1];
            // entries ascend with the thread's stride, so the maximum m only moves up
            int m = g - 1;
            for (int e = threadIdx.x; e < c; e += blockDim.x) {
                while (binom[(m + 1) * BK + g] <= (unsigned long long)e) m++;
                const int r = base + m;
                typename E::T x = E::load_row(rows + r * 2 * W);
                unsigned long long sy = SW ? syn[r] : 0ull;
                if (g > 1) {
                    const int src = src0 + e - int(binom[m * BK + g]);
                    x = E::x(L[src], x);
                    if (SW) sy ^= S[src];
                }
                mitm_candidate(E::weight(x), sy, SW, scale, best, wlim);
                if (store) {
                    L[dst0 + e] = x;
                    if (SW) S[dst0 + e] = sy;
                }
            }
            (void)n;
        }
    }
    __syncthreads();
}

// the pairs A_h x B_(g-h), 0 < h < g, of one level and all G matrices. A warp takes a block of
// R rows of the shorter list (round robin over the blocks of every segment, so the warps stay
// balanced without a barrier) and its lanes stride the longer one: each lane loads one entry
// per step and scores it against the R rows it holds in registers.
constexpr int kMitmRows = 4;

template <int W, int R>
__device__ __forceinline__ void mitm_rows(int oy, int ny, int ox, int nx, int yb, const typename MitmEnt<W>::T *L,
                                          const unsigned long long *S, int SW, unsigned scale, unsigned &best,
                                          unsigned &wlim) {
    using E = MitmEnt<W>;
    typename E::T a[R];
#pragma unroll
    for (int i = 0; i < R; i++) a[i] = L[oy + min(yb * R + i, ny - 1)];
    for (int x = threadIdx.x & 31; x < nx; x += 32) {
        const typename E::T u = L[ox + x];
#pragma unroll
        for (int i = 0; i < R; i++) {
            const unsigned w = E::weight(a[i], u);
            if (w < wlim && (SW == 0 || (S[oy + min(yb * R + i, ny - 1)] ^ S[ox + x]) != 0ull)) {
                best = scale * w;
                wlim = w;
            }
        }
    }
}

template <int W>
__device__ __forceinline__ void mitm_scan(int g, int G, const unsigned long long *binom, int BK, const MitmView &v,
                                          const typename MitmEnt<W>::T *ent, const unsigned long long *esyn, int SW,
                                          unsigned scale, unsigned &best, unsigned &wlim) {
    constexpr int R = kMitmRows;
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int t0 = warp;  // block index carried across segments
    for (int j = 0; j < G; j++) {
        const typename MitmEnt<W>::T *L = ent + j * v.stride;
        const unsigned long long *S = esyn + j * v.stride;
        constexpr int K = kMitmMaxLevel + 1;
        for (int h = 1; h < g; h++) {
            const int cA = v.cnt[h], cB = v.cnt[K + g - h];
            if (cA == 0 || cB == 0) continue;
            const int oA = v.off[h], oB = v.off[K + g - h];
            const bool xa = cA >= cB;  // lanes stride the longer list
            const int oy = xa ? oB : oA, ny = xa ? cB : cA, ox = xa ? oA : oB, nx = xa ? cA : cB;
            const bool wide = ny >= R;
            const int blocks = wide ? (ny + R - 1) / R : ny;
            int t = t0;
            for (; t < blocks; t += nwarps) {
                if (wide)
                    mitm_rows<W, R>(oy, ny, ox, nx, t, L, S, SW, scale, best, wlim);
                else
                    mitm_rows<W, 1>(oy, ny, ox, nx, t, L, S, SW, scale, best, wlim);
            }
            t0 = t - blocks;
        }
    }
}

// One code per CTA, its whole level loop (U, L, trace, termination) in shared memory. Levels
// whose meet-in-the-middle lists fit (BatchDev.mitm_g) run mitm_build + mitm_scan; deeper ones
// fall back to a per-thread walk: each thread takes one contiguous lex-rank segment, and since
// the lex order varies the last element fastest, its loop is one row XOR onto the (g-1)-prefix
// accumulator and one POPC per word, the prefix advancing once per run of last elements (the
// syndrome is rebuilt only for candidates below the best).
template <int W>
__global__ void __launch_bounds__(256) batch_kernel(BatchDev b) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int code = blockIdx.x;
    const int rowlen = 2 * W;
    const int N = b.N;
    __shared__ unsigned int s_wmin;
    __shared__ int s_done;
    if (b.in_status && b.in_status[code] != 0) {
        if (threadIdx.x == 0) {
            b.out_upper[code] = b.sentinel;
            b.out_generations[code] = 0;
            b.out_status[code] = b.in_status[code];
        }
        return;
    }
    // matrices of this code: its own count from the device prep, else the batch-wide G
    const int G = b.n_gammas ? b.n_gammas[code] : b.G;
    if (G > b.G) {  // more matrices than slots: the host redoes this code with host prep
        if (threadIdx.x == 0) {
            b.out_upper[code] = b.sentinel;
            b.out_generations[code] = 0;
            b.out_status[code] = kBatchNeedsHostPrep;
        }
        return;
    }
    const int nrow_words = b.G * N * rowlen;
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem);
    unsigned long long *s_binom =
        reinterpret_cast<unsigned long long *>(smem + ((nrow_words * 4 + 15) & ~15));
    const int nbinom = (N + 1) * b.BK;
    unsigned long long *s_syn = s_binom + nbinom;
    // 16-byte aligned offset into the dynamic shared block (pointer arithmetic on smem keeps
    // the shared address space visible to the compiler)
    unsigned char *s_mitm =
        smem + ((reinterpret_cast<unsigned char *>(s_syn + b.G * N * b.SW) - smem + 15) & ~ptrdiff_t(15));
    const uint32_t *grow = b.rows + (size_t)code * b.Gs * N * rowlen;
    const unsigned long long *gsyn = b.syn + (size_t)code * b.Gs * N * b.SW;
    for (int i = threadIdx.x; i < G * N * rowlen; i += blockDim.x) s_rows[i] = grow[i];
    for (int i = threadIdx.x; i < nbinom; i += blockDim.x) s_binom[i] = b.binom[i];
    for (int i = threadIdx.x; i < G * N * b.SW; i += blockDim.x) s_syn[i] = gsyn[i];
    // list sizes and offsets of the meet-in-the-middle levels: [half][h]
    __shared__ int s_mcnt[2 * (kMitmMaxLevel + 1)], s_moff[2 * (kMitmMaxLevel + 1)];
    if (b.mitm_g > 0 && threadIdx.x < 2) {
        const int half = threadIdx.x, n = half ? N - (N >> 1) : (N >> 1);
        int at = half ? mitm_off(b.binom, b.BK, N >> 1, b.mitm_g) : 0;  // s_binom is not loaded yet
        for (int h = 0; h <= kMitmMaxLevel; h++) {
            const int c = h <= b.mitm_g ? int(binom_at(b.binom, b.BK, n, h)) : 0;
            s_mcnt[half * (kMitmMaxLevel + 1) + h] = c;
            s_moff[half * (kMitmMaxLevel + 1) + h] = at;
            at += h < b.mitm_g ? c : 0;
        }
    }
    // the rank deficits, read once: the level close below is a serial section of thread 0
    __shared__ int s_def[kPrepGammaSlots];
    if (threadIdx.x < kPrepGammaSlots) s_def[threadIdx.x] = int(threadIdx.x) < G ? b.deficits[(size_t)code * b.Gs + threadIdx.x] : 0;
    if (threadIdx.x == 0) { s_wmin = unsigned(b.sentinel); s_done = 0; }
    __syncthreads();

    const int SW = b.SW;
    const unsigned scale = unsigned(b.scale);
    int U = b.sentinel;
    int gen = 0;
    int c[kMaxLevel];
    const int g_last = b.max_g > 0 ? min(N, b.max_g) : N;
    for (int g = 1; g <= g_last; g++) {
        // thread-local minimum of the admissible candidates below U (engine units); one shared
        // atomic per warp at the end instead of one per improving candidate
        unsigned best = unsigned(U);
        unsigned wlim = (best + scale - 1) / scale;  // popc < wlim  <=>  scale * popc < best
        // levels whose half-lists fit stay resident and grow by one size per level
        const bool mitm = W <= 2 && g <= b.mitm_g && G <= kMitmSlots;
        if constexpr (W <= 2) {
            if (mitm) {
                using T = typename MitmEnt<W>::T;
                MitmView v;
                v.nA = N >> 1;
                v.nB = N - v.nA;
                v.stored = b.mitm_g;
                v.blockB = s_moff[v.stored];
                v.stride = s_moff[kMitmMaxLevel + 1 + v.stored];
                v.cnt = s_mcnt;
                v.off = s_moff;
                T *ent = reinterpret_cast<T *>(s_mitm);
                unsigned long long *esyn = reinterpret_cast<unsigned long long *>(s_mitm + size_t(b.mitm_cap) * sizeof(T));
                mitm_build<W>(g, G, N, s_rows, s_syn, SW, s_binom, b.BK, v, ent, esyn, scale, best, wlim);
                mitm_scan<W>(g, G, s_binom, b.BK, v, ent, esyn, SW, scale, best, wlim);
            }
        }
        // one segment per thread: tiny levels get a candidate or two per thread, not a long
        // serial walk on a few of them
        const unsigned long long per = mitm ? 0ull : binom_at(s_binom, b.BK, N, g);
        const unsigned long long seg_len = mitm ? 1ull : max(1ull, (per * G + blockDim.x - 1) / blockDim.x);
        const unsigned long long segs_per = mitm ? 0ull : (per + seg_len - 1) / seg_len;
        for (unsigned long long seg = threadIdx.x; seg < segs_per * G; seg += blockDim.x) {
            const int j = int(seg / segs_per);
            const unsigned long long r0 = (seg % segs_per) * seg_len;
            const uint32_t *rows = s_rows + j * N * rowlen;
            const unsigned long long *syn = s_syn + j * N * SW;
            unrank_lex(r0, g, N, s_binom, b.BK, c);
            uint32_t pre[2 * W];
#pragma unroll
            for (int i = 0; i < 2 * W; i++) pre[i] = 0;
            for (int i = 0; i < g - 1; i++) xor_row<W>(pre, rows + c[i] * rowlen);
            int m = c[g - 1];
            unsigned long long left = min(r0 + seg_len, per) - r0;
            for (;;) {
                const int lim = int(min((unsigned long long)N, (unsigned long long)m + left));
                left -= (unsigned long long)(lim - m);
                const uint32_t *row = rows + m * rowlen;
                for (; m < lim; m++, row += rowlen) {
                    unsigned w = 0;
#pragma unroll
                    for (int i = 0; i < W; i++) w += __popc((pre[i] ^ row[i]) | (pre[W + i] ^ row[W + i]));
                    if (w < wlim) {
                        bool ok = SW == 0;
                        for (int s = 0; s < SW && !ok; s++) {
                            unsigned long long x = syn[m * SW + s];
                            for (int i = 0; i < g - 1; i++) x ^= syn[c[i] * SW + s];
                            ok = x != 0;
                        }
                        if (ok) {
                            best = scale * w;
                            wlim = w;
                        }
                    }
                }
                if (left == 0 || g == 1) break;
                // next (g-1)-prefix in lex order; its last element restarts right after it
                int i = g - 2;
                while (c[i] == N - g + i) i--;
                for (int q = i; q < g - 1; q++) xor_row<W>(pre, rows + c[q] * rowlen);
                c[i]++;
                for (int q = i + 1; q < g - 1; q++) c[q] = c[q - 1] + 1;
                for (int q = i; q < g - 1; q++) xor_row<W>(pre, rows + c[q] * rowlen);
                m = c[g - 2] + 1;
            }
        }
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_down_sync(0xffffffffu, best, o));
        if ((threadIdx.x & 31) == 0 && best < unsigned(U)) atomicMin(&s_wmin, best);
        __syncthreads();
        if (threadIdx.x == 0) {
            if (int(s_wmin) < U) U = int(s_wmin);
            long lower = 0;
            for (int j = 0; j < G; j++) {
                const int t = g + 1 - (j < kPrepGammaSlots ? s_def[j] : b.deficits[(size_t)code * b.Gs + j]);
                lower += t > 0 ? t : 0;
            }
            b.out_trace_lower[(size_t)code * N + g - 1] = int(lower);
            b.out_trace_upper[(size_t)code * N + g - 1] = U;
            if (lower >= U) s_done = 1;
            s_wmin = unsigned(U);
        }
        __syncthreads();
        U = int(s_wmin);
        gen = g;
        if (s_done) break;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        b.out_upper[code] = U;
        b.out_generations[code] = gen;
        b.out_status[code] = (U >= b.sentinel && (s_done || gen == N)) ? 3 : 0;
    }
}


// ---------------------------------------------------------------- tile: heads x tails

// log2(i!) for i <= kMaxLevel: the starting estimate of unrank_colex_est
__constant__ float c_log2fact[kMaxLevel + 1] = {0.0000000f, 0.0000000f, 1.0000000f, 2.5849625f, 4.5849625f, 6.9068906f, 9.4918531f, 12.2992080f, 15.2992080f, 18.4691330f, 21.7910611f, 25.2504927f, 28.8354552f, 32.5358950f, 36.3432499f, 40.2501405f, 44.2501405f, 48.3376033f, 52.5075283f, 56.7554558f, 61.0773839f, 65.4697013f, 69.9291330f, 74.4526949f, 79.0376574f, 83.6815136f, 88.3819533f, 93.1368408f, 97.9441958f, 102.8021767f, 107.7090673f, 112.6632637f, 117.6632637f, 122.7076578f, 127.7951206f, 132.9244036f, 138.0943286f, 143.3037820f, 148.5517095f, 153.8371117f, 159.1590398f, 164.5165918f, 169.9089093f, 175.3351740f, 180.7946056f, 186.2864587f, 191.8100207f, 197.3646095f, 202.9495720f, 208.5642819f, 214.2081381f, 219.8805634f, 225.5810031f, 231.3089236f, 237.0638111f, 242.8451708f, 248.6525257f, 254.4854157f, 260.3433967f, 266.2260398f, 272.1329304f, 278.0636677f, 284.0178640f};

// 1 / i for the same i (a multiply instead of a division in the estimate)
__constant__ float c_inv[kMaxLevel + 1] = {0.0f, 1.0f / 1, 1.0f / 2, 1.0f / 3, 1.0f / 4, 1.0f / 5, 1.0f / 6, 1.0f / 7, 1.0f / 8, 1.0f / 9,
    1.0f / 10, 1.0f / 11, 1.0f / 12, 1.0f / 13, 1.0f / 14, 1.0f / 15, 1.0f / 16, 1.0f / 17, 1.0f / 18, 1.0f / 19, 1.0f / 20,
    1.0f / 21, 1.0f / 22, 1.0f / 23, 1.0f / 24, 1.0f / 25, 1.0f / 26, 1.0f / 27, 1.0f / 28, 1.0f / 29, 1.0f / 30, 1.0f / 31,
    1.0f / 32, 1.0f / 33, 1.0f / 34, 1.0f / 35, 1.0f / 36, 1.0f / 37, 1.0f / 38, 1.0f / 39, 1.0f / 40, 1.0f / 41, 1.0f / 42,
    1.0f / 43, 1.0f / 44, 1.0f / 45, 1.0f / 46, 1.0f / 47, 1.0f / 48, 1.0f / 49, 1.0f / 50, 1.0f / 51, 1.0f / 52, 1.0f / 53,
    1.0f / 54, 1.0f / 55, 1.0f / 56, 1.0f / 57, 1.0f / 58, 1.0f / 59, 1.0f / 60, 1.0f / 61, 1.0f / 62};

// colex unrank of rho into an m-subset of [0, lim), ascending into e[0..m-1]: for i = m..1 the
// largest c below the previous element with C(c, i) <= rho. Each search starts at an estimate
// instead of scanning down from the previous element: C(c, i) <= rho < C(c + 1, i) puts c in (x - 1, x + i - 1] with
// x = (rho * i!)^(1/i), so a start at x + (i - 1)/2 is off by a step or two, where the scan
// costs up to `lim` dependent shared-memory loads per unrank.
__device__ __forceinline__ void unrank_colex_est(unsigned long long rho, int m, int lim,
                                                 const unsigned long long *binom, int BK, int *e) {
    int c = lim - 1;
    for (int i = m; i >= 1; i--) {
        int cc;
        if (i == 1) {
            cc = int(min(rho, (unsigned long long)c));  // C(cc, 1) = cc
        } else {
            const float lx = (__log2f(float(rho) + 1.0f) + c_log2fact[i]) * c_inv[i];
            const float est = exp2f(lx) + 0.5f * float(i - 1);
            cc = max(est >= float(c) ? c : int(est), i - 1);  // clamped before the conversion
            while (binom_at(binom, BK, cc, i) > rho) cc--;
            while (cc < c && binom_at(binom, BK, cc + 1, i) <= rho) cc++;
        }
        e[i - 1] = cc;
        rho -= binom_at(binom, BK, cc, i);
        c = cc - 1;
    }
}

// lexicographic rank of ascending c[0..g-1] among g-subsets of [0, N): the reference's
// visiting order inside one generation (engine.cpp:202-219)
__device__ __forceinline__ unsigned long long lexrank(const int *c, int g, int N, const unsigned long long *binom,
                                                      int BK, unsigned long long per) {
    unsigned long long s = 0;
    for (int i = 1; i <= g; i++) s += binom_at(binom, BK, N - 1 - c[g - i], i);
    return per - 1 - s;
}

// One work unit of the tile kernel, decoded once per CTA and kept in shared memory so the
// hot loop carries no per-unit registers (they would spill at 64 registers per thread).
struct TileUnit {
    int j, b, tcount, pad;
    unsigned long long t0;      // first tail (colex rank among (t-1)-subsets of (b, N))
    unsigned long long hbase0;  // first head of the block (colex rank among h-subsets of [0, b))
};

// Rare path: a candidate whose fast-path lower bound passed the threshold. Rebuilds its
// element list from the head rank and the tail rank, computes the exact weight from the
// rows, applies the admissibility syndrome (reference AdmissibilityFilter,
// engine.cpp:14-29) and publishes (weight, key). Returns the updated threshold.
template <int W>
__device__ __noinline__ unsigned tile_exact(const ProblemDev p, const TilePlan tp, const uint32_t *s_rows,
                                            const unsigned long long *s_binom, int BKs, const TileUnit *un,
                                            int head_off, int tix, unsigned thrH) {
    const int N = p.N, h = tp.h, t = tp.t, g = tp.g, j = un->j, b = un->b;
    const uint32_t *grows = s_rows + j * N * 2 * W;
    int c[kMaxLevel];
    unrank_colex_est(un->hbase0 + head_off, h, b, s_binom, BKs, c);
    c[h] = b;
    unrank_colex_est(un->t0 + tix, t - 1, N - 1 - b, s_binom, BKs, c + h + 1);
    for (int k = h + 1; k < g; k++) c[k] += b + 1;
    for (int k = 0; k < g; k++) SDB_CHECK(c[k] >= 0 && c[k] < N && (k == 0 || c[k] > c[k - 1]));
    uint32_t acc[2 * W];
#pragma unroll
    for (int w = 0; w < 2 * W; w++) acc[w] = 0;
    for (int k = 0; k < g; k++) xor_row<W>(acc, grows + c[k] * 2 * W);
    const unsigned wv = unsigned(p.scale * weight_of<W>(acc));
    if (wv > thrH) return thrH;
    if (p.SW) {
        const unsigned long long *syn = p.syn + (size_t)j * N * p.SW;
        bool adm = false;
        for (int s = 0; s < p.SW; s++) {
            unsigned long long x = 0;
            for (int k = 0; k < g; k++) x ^= syn[c[k] * p.SW + s];
            adm |= x != 0;
        }
        if (!adm) return thrH;
    }
    const unsigned long long key =
        ((unsigned long long)j << kKeyRankBits) | lexrank(c, g, N, s_binom, BKs, tp.per_gamma);
    atomicMin(&p.state->wmin, wv);
    atomicMin(&p.key_by_w[wv], key);
    return wv;
}

// Fast-path lower bound on a candidate's weight (in symbols), one POPC whatever W is: the OR
// of the probe-word differences. The probe words of a row (ProblemDev.prows, K per row) are
// the oriented word of each 32-symbol block, plus — for Gammas whose probe words alone are
// sparse — the partner word of one block; W = 1 keeps both words of its block. Bit b of the
// fold is set only if a symbol 32w+b of the candidate is nonzero, so popc(fold) <= popc(x|z)
// (exact for W = 1).
template <int K>
__device__ __forceinline__ uint32_t probe_fold(const uint32_t (&hp)[K], const uint32_t *t) {
    uint32_t u = hp[0] ^ t[0];
#pragma unroll
    for (int w = 1; w < K; w++) u |= hp[w] ^ t[w];
    return u;
}


// colex successor of the ascending m-subset e (m >= 1) with the row sum kept in acc:
// the lowest element that can move up by one moves, the ones below it reset to 0..q-1.
// rows(i) = base + (off + i) * rowlen; NW words of each row take part.
template <int NW>
__device__ __forceinline__ void colex_step(int *e, int m, uint32_t (&acc)[NW], const uint32_t *base, int off,
                                           int rowlen) {
    int q = 0;
    while (q < m - 1 && e[q] + 1 == e[q + 1]) q++;
    for (int k = 0; k <= q; k++)
#pragma unroll
        for (int w = 0; w < NW; w++) acc[w] ^= base[(off + e[k]) * rowlen + w];
    e[q]++;
    for (int k = 0; k < q; k++) e[k] = k;
    for (int k = 0; k <= q; k++)
#pragma unroll
        for (int w = 0; w < NW; w++) acc[w] ^= base[(off + e[k]) * rowlen + w];
}

template <int W, bool XP>
__global__ void __launch_bounds__(kTileThreads, tile_blocks_per_sm(W, probe_words(W, XP)))
    tile_kernel(ProblemDev p, TilePlan tp) {
    constexpr int K = probe_words(W, XP);  // probe words per row / head / tail
    constexpr int H = heads_per_lane(W, K);
    constexpr int HB = head_block(W, K);
    constexpr int PW = probe_stride(K);
    if (run_done(p)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const int rowlen = 2 * W;
    const int G = p.G, N = p.N;
    // binomials C(a, k) for k <= g + 1 only: the level needs no wider ones, and the slice keeps
    // shared memory small enough for many resident CTAs
    const int BKs = min(p.BK, tp.g + 2);
    const TileSmem lay = tile_smem_layout(G, N, W, K, BKs);
    const int nrow_words = G * N * rowlen;
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem + lay.rows);
    unsigned long long *s_binom = reinterpret_cast<unsigned long long *>(smem + lay.binom);
    const int nbinom = (N + 1) * BKs;
    uint32_t *s_tp = reinterpret_cast<uint32_t *>(smem + lay.tp);
    uint32_t *s_prows = reinterpret_cast<uint32_t *>(smem + lay.prows);
    __shared__ TileUnit s_un;
    __shared__ unsigned long long s_visited, s_skipped;
    // units are claimed in runs of consecutive indices (fewer near the end of the level); the
    // head blocks of one tail chunk are consecutive, so a run mostly reuses the staged tails
    __shared__ unsigned long long s_claim, s_claim_end;
    __shared__ int s_restage, s_staged_j, s_staged_b;
    __shared__ unsigned long long s_staged_t0;
    for (int i = threadIdx.x; i < nrow_words; i += blockDim.x) s_rows[i] = p.rows[i];
    for (int i = threadIdx.x; i < G * N * K; i += blockDim.x) s_prows[i] = p.prows[i];
    // adjacent-row table: adj[r] = prows[r] ^ prows[r + 1] within each Gamma
    uint32_t *s_adj = reinterpret_cast<uint32_t *>(smem + lay.adj);
    for (int i = threadIdx.x; i < G * N * K; i += blockDim.x)
        s_adj[i] = (i / K) % N < N - 1 ? p.prows[i] ^ p.prows[i + K] : 0u;
    for (int i = threadIdx.x; i < nbinom; i += blockDim.x) s_binom[i] = p.binom[(i / BKs) * p.BK + i % BKs];
    if (threadIdx.x == 0) {
        s_visited = 0;
        s_skipped = 0;
        s_claim = s_claim_end = 0;
        s_staged_b = -1;
    }
    // this rank's units: local index u is global unit u * world + rank
    const unsigned long long local_units = (tp.unit_total + tp.shard_world - 1 - tp.shard_rank) / tp.shard_world;

    const unsigned sshift = p.scale == 2 ? 1u : 0u;
    const int lane_head = (threadIdx.x >> 5) * (32 * H) + (threadIdx.x & 31) * H;
    unsigned thrH = start_threshold(p, tp.thr0);
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_claim == s_claim_end) {
#ifndef SDB_UNIT_BATCH
#define SDB_UNIT_BATCH 4
#endif
                // runs of SDB_UNIT_BATCH while plenty remain; single units for the last few
                // per CTA, which bound the level's tail
                const unsigned long long seen = *(volatile unsigned long long *)tp.counter;
                const unsigned long long run =
                    seen + 4ull * SDB_UNIT_BATCH * gridDim.x < local_units ? SDB_UNIT_BATCH : 1ull;
                s_claim = atomicAdd(tp.counter, run);
                s_claim_end = s_claim + run;
            }
            const unsigned long long unit = (s_claim++) * tp.shard_world + tp.shard_rank;
            s_un.tcount = 0;
            s_restage = 0;
            if (unit < tp.unit_total) {
                // (j, b): the last q with cum[q] <= unit
                int lo = 0, hi = G * tp.nb - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (__ldg(tp.cum + mid) <= unit) lo = mid; else hi = mid - 1;
                }
                const int b = tp.h + lo % tp.nb;
                const unsigned long long u = unit - __ldg(tp.cum + lo);
                const unsigned long long Hb = binom_at(s_binom, BKs, b, tp.h);
                const unsigned long long Tb = binom_at(s_binom, BKs, N - 1 - b, tp.t - 1);
                const unsigned long long nH = (Hb + HB - 1) / HB;
                // head blocks vary fastest: consecutive units share their tail chunk
                const unsigned long long tc = u / nH, hc = u % nH;
                s_un.j = lo / tp.nb;
                s_un.b = b;
                s_un.t0 = tc * tp.tchunk;
                s_un.tcount = int(min((unsigned long long)tp.tchunk, Tb - s_un.t0));
                s_un.hbase0 = hc * HB;
                s_un.pad = int(min((unsigned long long)HB, Hb - hc * HB));  // heads in this block
                if ((unsigned long long)s_un.j > (early_key(p, tp.lprev) >> kKeyRankBits)) {
                    // early exit: a later Gamma's keys all exceed the best one; -1 skips the unit
                    s_skipped += (unsigned long long)s_un.pad * (unsigned long long)s_un.tcount;
                    s_un.tcount = -1;
                } else {
                    s_visited += (unsigned long long)s_un.pad * (unsigned long long)s_un.tcount;
                    if (s_un.j != s_staged_j || b != s_staged_b || s_un.t0 != s_staged_t0) {
                        s_restage = 1;
                        s_staged_j = s_un.j;
                        s_staged_b = b;
                        s_staged_t0 = s_un.t0;
                    }
                }
            }
        }
        __syncthreads();
        const int tcount = s_un.tcount;
        if (tcount == 0) break;
        if (tcount < 0) continue;  // skipped (the loop top syncs before s_un is rewritten)
        const int t = tp.t, h = tp.h;
        {
            const int b = s_un.b;
            const uint32_t *pg = s_prows + s_un.j * N * K;  // probe words of this Gamma's rows
            // stage the tail chunk's probe words: {b} + colex (t-1)-subsets of (b, N);
            // each thread takes a contiguous run and walks it with colex successors
            const int R = (tcount + blockDim.x - 1) / blockDim.x;
            const int i0 = threadIdx.x * R, i1 = min(i0 + R, tcount);
            if (s_restage && i0 < i1) {
                int e[kMaxLevel];
                unrank_colex_est(s_un.t0 + i0, t - 1, N - 1 - b, s_binom, BKs, e);
                uint32_t acc[K];
#pragma unroll
                for (int w = 0; w < K; w++) acc[w] = pg[b * K + w];
                for (int k = 0; k < t - 1; k++)
#pragma unroll
                    for (int w = 0; w < K; w++) acc[w] ^= pg[(b + 1 + e[k]) * K + w];
                for (int i = i0;;) {
#pragma unroll
                    for (int w = 0; w < K; w++) s_tp[i * PW + w] = acc[w];
                    if (i == tcount - 1 && (tcount & 1))  // odd counts: duplicate the last tail
#pragma unroll
                        for (int w = 0; w < K; w++) s_tp[(i + 1) * PW + w] = acc[w];
                    if (++i >= i1) break;
                    colex_step<K>(e, t - 1, acc, pg, b + 1, K);
                }
            }
        }
        __syncthreads();

        // this lane's heads: H consecutive colex ranks of h-subsets of [0, b)
        const int nvalid = max(0, min(H, s_un.pad - lane_head));
        if (!__any_sync(0xffffffffu, nvalid > 0)) continue;
        uint32_t hp[H][K];
        {
            const int b = s_un.b;
            const uint32_t *pg = s_prows + s_un.j * N * K;
            int e[kMaxLevel];
            uint32_t acc[K];
            // e0, e1: the two lowest elements in registers (e1 = b for h = 1): most colex
            // successors just move e0 up by one, one XOR of the adjacent-row table
            int e0 = 0, e1 = b;
            if (nvalid > 0) {
                unrank_colex_est(s_un.hbase0 + lane_head, h, b, s_binom, BKs, e);
#pragma unroll
                for (int w = 0; w < K; w++) acc[w] = 0;
                for (int k = 0; k < h; k++)
#pragma unroll
                    for (int w = 0; w < K; w++) acc[w] ^= pg[e[k] * K + w];
                e0 = e[0];
                if (h > 1) e1 = e[1];
            } else {
                // lanes without heads: all-ones probe words, the fold never passes the check
#pragma unroll
                for (int w = 0; w < K; w++) acc[w] = 0xffffffffu;
            }
            const uint32_t *ag = s_adj + s_un.j * N * K;
#pragma unroll
            for (int i = 0; i < H; i++) {
                if (i > 0 && i < nvalid) {
                    if (e0 + 1 < e1) {
#pragma unroll
                        for (int w = 0; w < K; w++) acc[w] ^= ag[e0 * K + w];
                        e0++;
                    } else {
                        e[0] = e0;
                        colex_step<K>(e, h, acc, pg, 0, K);
                        e0 = e[0];
                        e1 = h > 1 ? e[1] : b;
                    }
                }
                // heads past the valid count repeat the last valid head (same candidates)
#pragma unroll
                for (int w = 0; w < K; w++) hp[i][w] = acc[w];
            }
        }

        unsigned thr0 = thrH >> sshift;
        int ti = 0;
        for (;;) {
            // hot loop: no calls inside, so the heads stay in registers
            for (; ti < tcount; ti += 2) {
                // both tails' probe words: 2 * PW words, whole 16-byte broadcast loads
                uint32_t tt[2 * PW];
#pragma unroll
                for (int v = 0; v < 2 * PW; v += 4) {
                    const uint4 q4 = *reinterpret_cast<const uint4 *>(s_tp + ti * PW + v);
                    tt[v] = q4.x;
                    tt[v + 1] = q4.y;
                    tt[v + 2] = q4.z;
                    tt[v + 3] = q4.w;
                }
                unsigned m = 0xffffffffu;
#pragma unroll
                for (int i = 0; i < H; i++) {
                    const unsigned a = __popc(probe_fold<K>(hp[i], tt));
                    const unsigned c = __popc(probe_fold<K>(hp[i], tt + PW));
                    m = min(m, min(a, c));
                }
                // warp-uniform exit: a lone lane leaving the loop would finish it alone later
                if (__any_sync(0xffffffffu, m <= thr0 && nvalid > 0)) break;
            }
            if (ti >= tcount) break;
            // rare: which of this lane's 2H candidates passed the bound; one call site
            unsigned fire = 0;
#pragma unroll
            for (int i = 0; i < H; i++) {
#pragma unroll
                for (int r = 0; r < 2; r++)
                    if (i < nvalid && ti + r < tcount &&
                        __popc(probe_fold<K>(hp[i], s_tp + (ti + r) * PW)) <= thr0)
                        fire |= 1u << (2 * i + r);
            }
            while (fire) {
                const int k = __ffs(fire) - 1;
                fire &= fire - 1;
                thrH = tile_exact<W>(p, tp, s_rows, s_binom, BKs, &s_un, lane_head + (k >> 1), ti + (k & 1), thrH);
            }
            thr0 = thrH >> sshift;
            ti += 2;
        }
        thrH = min(thrH, *(volatile unsigned int *)&p.state->wmin);
    }
    if (threadIdx.x == 0 && s_skipped) atomicAdd(&p.state->skipped, s_skipped);
    if (threadIdx.x == 0 && s_visited) atomicAdd(&p.state->visited, s_visited);
}

// ---------------------------------------------------------------- tensor-core tile (tcgen05)

#include "tc_tile.cuh"

// ---------------------------------------------------------------- packaged tile (1/3-packages)

struct PtileSmem {
    size_t rows, prows, el, off, F, FR, tp, total;
};
__host__ __device__ inline PtileSmem ptile_layout(int G, int N, int W, int K, int P, int E, int BKs) {
    PtileSmem L{};
    L.rows = 0;
    L.prows = align16(size_t(G) * N * 2 * W * 4);
    L.el = align16(L.prows + size_t(G) * N * K * 4);                 // e_row, e_pkg, r_row, r_pkg
    L.off = align16(L.el + size_t(4) * G * E * 2);                   // off, r_off
    L.F = align16(L.off + size_t(2) * G * (P + 1) * 2);              // F sliced to BKs columns
    L.FR = align16(L.F + size_t(G) * (E + 1) * BKs * 8);
    L.tp = align16(L.FR + size_t(G) * (E + 1) * BKs * 8);
    L.total = align16(L.tp + size_t(kTailChunk + 1) * probe_stride(K) * 4);
    return L;
}

// colex unrank of rho into m elements with distinct packages inside elements [0, lim):
// the largest x with F(x, i) <= rho is the i-th element; the rest lie below its package.
// F(., i) is nondecreasing and F(0, i) = 0, so each element is a binary search (a scan down
// from the previous element costs up to `lim` dependent shared-memory loads per unrank).
__device__ __forceinline__ void unrank_pcolex(unsigned long long rho, int m, int lim, const unsigned long long *F,
                                              int BKs, const short *epkg, const short *off, int *e) {
    int hi = lim - 1;
    for (int i = m; i >= 1; i--) {
        int lo = 0;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (F[mid * BKs + i] <= rho) lo = mid; else hi = mid - 1;
        }
        e[i - 1] = lo;
        rho -= F[lo * BKs + i];
        hi = off[epkg[lo]] - 1;
    }
}

// The same unrank scanning down from the bound: the tail staging keeps it, because a tail
// chunk's first tail mostly sits at the top of its range (measured on config 4's Saved_2_Gamma:
// bisecting there cost 2%, while bisecting the heads and the rare path gained 0.7%).
__device__ __forceinline__ void unrank_pcolex_scan(unsigned long long rho, int m, int lim, const unsigned long long *F,
                                                   int BKs, const short *epkg, const short *off, int *e) {
    int x = lim - 1;
    for (int i = m; i >= 1; i--) {
        while (F[x * BKs + i] > rho) x--;
        e[i - 1] = x;
        rho -= F[x * BKs + i];
        x = off[epkg[x]] - 1;
    }
}

// colex successor of the element set e[0..m) (distinct packages, all below lim) with the
// row sum kept in acc: the lowest element that can move to the next element (next member,
// or the first member of the next package, as long as it stays below the package of the
// element above it); the ones below restart at the first members of packages 0, 1, ...
template <int NW>
__device__ __forceinline__ void pcolex_step(int *e, int m, int lim, const short *epkg, const short *off,
                                            const short *erow, uint32_t (&acc)[NW], const uint32_t *rows,
                                            int rowlen) {
    int i = 0;
    for (;; i++) {
        const int v = e[i] + 1;
        if (i + 1 < m ? (v < e[i + 1] && epkg[v] != epkg[e[i + 1]]) : v < lim) break;
    }
    for (int k = 0; k <= i; k++)
#pragma unroll
        for (int w = 0; w < NW; w++) acc[w] ^= rows[erow[e[k]] * rowlen + w];
    e[i]++;
    for (int k = 0; k < i; k++) e[k] = off[k];
    for (int k = 0; k <= i; k++)
#pragma unroll
        for (int w = 0; w < NW; w++) acc[w] ^= rows[erow[e[k]] * rowlen + w];
}

struct PtileUnit {
    int j, b, tcount, heads;
    int np, lim_h, lim_t, sb;             // packages, head / tail element limits, members of b
    unsigned long long t0, hbase0, tsub;  // first tail, first head, tail sets per member of b
};

// Per-Gamma views of the packaged tables in shared memory.
struct PtileView {
    const short *erow, *epkg, *rrow, *rpkg, *off, *roff;
    const unsigned long long *F, *FR;
};
__device__ __forceinline__ PtileView ptile_view(const short *s_el, const short *s_off, const unsigned long long *s_F,
                                                const unsigned long long *s_FR, int G, int E, int P, int BKs, int j) {
    PtileView v;
    v.erow = s_el + j * E;
    v.epkg = s_el + G * E + j * E;
    v.rrow = s_el + 2 * G * E + j * E;
    v.rpkg = s_el + 3 * G * E + j * E;
    v.off = s_off + j * (P + 1);
    v.roff = s_off + G * (P + 1) + j * (P + 1);
    v.F = s_F + size_t(j) * (E + 1) * BKs;
    v.FR = s_FR + size_t(j) * (E + 1) * BKs;
    return v;
}

// Rare path: rebuild the candidate's (package, member) list from the ranks, exact weight,
// admissibility, key = the reference's lexicographic rank over (p_1, m_1, p_2, m_2, ...)
// (engine.cpp:202-219) through the weighted suffix counts.
template <int W>
__device__ __noinline__ unsigned ptile_exact(const ProblemDev p, const PkgDev k, const PTilePlan tp,
                                             const uint32_t *s_rows, const PtileView v, int BKs, const PtileUnit *un,
                                             int head_off, int tix, unsigned thrH) {
    const int N = p.N, h = tp.h, t = tp.t, g = tp.g, j = un->j, b = un->b, np = un->np;
    int e[kMaxLevel], pk[kMaxLevel], mm[kMaxLevel], row[kMaxLevel];
    unrank_pcolex(un->hbase0 + head_off, h, un->lim_h, v.F, BKs, v.epkg, v.off, e);
    for (int i = 0; i < h; i++) {
        pk[i] = v.epkg[e[i]];
        mm[i] = e[i] - v.off[pk[i]];
        row[i] = v.erow[e[i]];
    }
    const unsigned long long tau = un->t0 + tix;
    const int mb = int(tau / un->tsub);
    pk[h] = b;
    mm[h] = mb;
    row[h] = v.erow[v.off[b] + mb];
    unrank_pcolex(tau % un->tsub, t - 1, un->lim_t, v.FR, BKs, v.rpkg, v.roff, e);
    for (int i = 0; i < t - 1; i++) {  // reversed order: the last reversed element is the next package
        const int er = e[t - 2 - i], rq = v.rpkg[er];
        pk[h + 1 + i] = np - 1 - rq;
        mm[h + 1 + i] = er - v.roff[rq];
        row[h + 1 + i] = v.rrow[er];
    }
    uint32_t acc[2 * W];
#pragma unroll
    for (int w = 0; w < 2 * W; w++) acc[w] = 0;
    const uint32_t *grows = s_rows + j * N * 2 * W;
    for (int i = 0; i < g; i++) xor_row<W>(acc, grows + row[i] * 2 * W);
    const unsigned wv = unsigned(p.scale * weight_of<W>(acc));
    if (wv > thrH) return thrH;
    if (p.SW) {
        const unsigned long long *syn = p.syn + (size_t)j * N * p.SW;
        bool adm = false;
        for (int s = 0; s < p.SW; s++) {
            unsigned long long x = 0;
            for (int i = 0; i < g; i++) x ^= syn[row[i] * p.SW + s];
            adm |= x != 0;
        }
        if (!adm) return thrH;
    }
    const unsigned long long *ws = k.wsuf + size_t(j) * (k.P + 1) * p.BK;
    const unsigned char *psz = k.pk_size + j * k.P;
    unsigned long long rank = 0;
    int prev = -1;
    for (int i = 0; i < g; i++) {
        for (int q = prev + 1; q < pk[i]; q++) rank += psz[q] * ws[(q + 1) * p.BK + (g - 1 - i)];
        rank += (unsigned long long)mm[i] * ws[(pk[i] + 1) * p.BK + (g - 1 - i)];
        prev = pk[i];
    }
    const unsigned long long key = ((unsigned long long)j << kKeyRankBits) | rank;
    atomicMin(&p.state->wmin, wv);
    atomicMin(&p.key_by_w[wv], key);
    return wv;
}

template <int W, bool XP>
__global__ void __launch_bounds__(kTileThreads, tile_blocks_per_sm(W, probe_words(W, XP)))
    ptile_kernel(ProblemDev p, PkgDev k, PtileDev d, PTilePlan tp) {
    constexpr int K = probe_words(W, XP);
    constexpr int H = heads_per_lane(W, K);
    constexpr int HB = head_block(W, K);
    constexpr int PW = probe_stride(K);
    if (run_done(p)) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const int rowlen = 2 * W, G = p.G, N = p.N, P = k.P, E = d.E;
    const int BKs = min(p.BK, tp.g + 2);
    const PtileSmem lay = ptile_layout(G, N, W, K, P, E, BKs);
    uint32_t *s_rows = reinterpret_cast<uint32_t *>(smem + lay.rows);
    short *s_el = reinterpret_cast<short *>(smem + lay.el);
    short *s_off = reinterpret_cast<short *>(smem + lay.off);
    unsigned long long *s_F = reinterpret_cast<unsigned long long *>(smem + lay.F);
    unsigned long long *s_FR = reinterpret_cast<unsigned long long *>(smem + lay.FR);
    uint32_t *s_tp = reinterpret_cast<uint32_t *>(smem + lay.tp);
    uint32_t *s_prows = reinterpret_cast<uint32_t *>(smem + lay.prows);
    __shared__ PtileUnit s_un;
    __shared__ unsigned long long s_visited;
    for (int i = threadIdx.x; i < G * N * rowlen; i += blockDim.x) s_rows[i] = p.rows[i];
    for (int i = threadIdx.x; i < G * N * K; i += blockDim.x) s_prows[i] = p.prows[i];
    for (int i = threadIdx.x; i < G * E; i += blockDim.x) {
        s_el[i] = d.e_row[i];
        s_el[G * E + i] = d.e_pkg[i];
        s_el[2 * G * E + i] = d.r_row[i];
        s_el[3 * G * E + i] = d.r_pkg[i];
    }
    for (int i = threadIdx.x; i < G * (P + 1); i += blockDim.x) {
        s_off[i] = d.off[i];
        s_off[G * (P + 1) + i] = d.r_off[i];
    }
    for (int i = threadIdx.x; i < G * (E + 1) * BKs; i += blockDim.x) {
        const int x = i / BKs, c = i % BKs;
        s_F[i] = d.F[size_t(x) * p.BK + c];
        s_FR[i] = d.FR[size_t(x) * p.BK + c];
    }
    if (threadIdx.x == 0) s_visited = 0;

    const unsigned sshift = p.scale == 2 ? 1u : 0u;
    const int lane_head = (threadIdx.x >> 5) * (32 * H) + (threadIdx.x & 31) * H;
    unsigned thrH = start_threshold(p, tp.thr0);
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long unit = atomicAdd(tp.counter, 1ull) * tp.shard_world + tp.shard_rank;
            s_un.tcount = 0;
            if (unit < tp.unit_total) {
                int lo = 0, hi = tp.npairs - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (__ldg(tp.cum + mid) <= unit) lo = mid; else hi = mid - 1;
                }
                const unsigned pr = __ldg(tp.pairs + lo);
                const int j = int(pr >> 16), b = int(pr & 0xffffu);
                const PtileView v = ptile_view(s_el, s_off, s_F, s_FR, G, E, P, BKs, j);
                const int np = k.np[j];
                const unsigned long long u = unit - __ldg(tp.cum + lo);
                s_un.j = j;
                s_un.b = b;
                s_un.np = np;
                s_un.lim_h = v.off[b];
                s_un.lim_t = v.roff[np - 1 - b];
                s_un.sb = v.off[b + 1] - v.off[b];
                const unsigned long long Hb = v.F[s_un.lim_h * BKs + tp.h];
                s_un.tsub = v.FR[s_un.lim_t * BKs + (tp.t - 1)];
                const unsigned long long Tb = (unsigned long long)s_un.sb * s_un.tsub;
                const unsigned long long nT = (Tb + tp.tchunk - 1) / tp.tchunk;
                const unsigned long long hc = u / nT, tc = u % nT;
                s_un.t0 = tc * tp.tchunk;
                s_un.tcount = int(min((unsigned long long)tp.tchunk, Tb - s_un.t0));
                s_un.hbase0 = hc * HB;
                s_un.heads = int(min((unsigned long long)HB, Hb - hc * HB));
                s_visited += (unsigned long long)s_un.heads * (unsigned long long)s_un.tcount;
            }
        }
        __syncthreads();
        const int tcount = s_un.tcount;
        if (tcount == 0) break;
        const int t = tp.t, h = tp.h, j = s_un.j;
        const PtileView v = ptile_view(s_el, s_off, s_F, s_FR, G, E, P, BKs, j);
        const uint32_t *pg = s_prows + j * N * K;  // probe words of this Gamma's rows
        {
            // stage tails: member mb of package b plus a (t-1)-set above b (reversed colex)
            const int R = (tcount + blockDim.x - 1) / blockDim.x;
            const int i0 = threadIdx.x * R, i1 = min(i0 + R, tcount);
            if (i0 < i1) {
                int e[kMaxLevel];
                unsigned long long tau = s_un.t0 + i0;
                int mb = int(tau / s_un.tsub);
                unsigned long long rest = tau % s_un.tsub;
                uint32_t acc[K];
                auto restart = [&]() {
                    unrank_pcolex_scan(rest, t - 1, s_un.lim_t, v.FR, BKs, v.rpkg, v.roff, e);
#pragma unroll
                    for (int w = 0; w < K; w++) acc[w] = pg[v.erow[v.off[s_un.b] + mb] * K + w];
                    for (int q = 0; q < t - 1; q++)
#pragma unroll
                        for (int w = 0; w < K; w++) acc[w] ^= pg[v.rrow[e[q]] * K + w];
                };
                restart();
                for (int i = i0;;) {
#pragma unroll
                    for (int w = 0; w < K; w++) s_tp[i * PW + w] = acc[w];
                    if (i == tcount - 1 && (tcount & 1))
#pragma unroll
                        for (int w = 0; w < K; w++) s_tp[(i + 1) * PW + w] = acc[w];
                    if (++i >= i1) break;
                    if (++rest == s_un.tsub) {  // next member of package b
                        rest = 0;
                        mb++;
                        restart();
                    } else {
                        pcolex_step<K>(e, t - 1, s_un.lim_t, v.rpkg, v.roff, v.rrow, acc, pg, K);
                    }
                }
            }
        }
        __syncthreads();

        const int nvalid = max(0, min(H, s_un.heads - lane_head));
        if (!__any_sync(0xffffffffu, nvalid > 0)) continue;
        uint32_t hp[H][K];
        {
            int e[kMaxLevel];
            uint32_t acc[K];
#pragma unroll
            for (int w = 0; w < K; w++) acc[w] = nvalid > 0 ? 0u : 0xffffffffu;
            if (nvalid > 0) {
                unrank_pcolex(s_un.hbase0 + lane_head, h, s_un.lim_h, v.F, BKs, v.epkg, v.off, e);
                for (int q = 0; q < h; q++)
#pragma unroll
                    for (int w = 0; w < K; w++) acc[w] ^= pg[v.erow[e[q]] * K + w];
            }
#pragma unroll
            for (int i = 0; i < H; i++) {
                if (i > 0 && i < nvalid) pcolex_step<K>(e, h, s_un.lim_h, v.epkg, v.off, v.erow, acc, pg, K);
#pragma unroll
                for (int w = 0; w < K; w++) hp[i][w] = acc[w];
            }
        }

        unsigned thr0 = thrH >> sshift;
        int ti = 0;
        for (;;) {
            for (; ti < tcount; ti += 2) {
                uint32_t tt[2 * PW];
#pragma unroll
                for (int vv = 0; vv < 2 * PW; vv += 4) {
                    const uint4 q4 = *reinterpret_cast<const uint4 *>(s_tp + ti * PW + vv);
                    tt[vv] = q4.x;
                    tt[vv + 1] = q4.y;
                    tt[vv + 2] = q4.z;
                    tt[vv + 3] = q4.w;
                }
                unsigned m = 0xffffffffu;
#pragma unroll
                for (int i = 0; i < H; i++) {
                    const unsigned a = __popc(probe_fold<K>(hp[i], tt));
                    const unsigned c = __popc(probe_fold<K>(hp[i], tt + PW));
                    m = min(m, min(a, c));
                }
                if (__any_sync(0xffffffffu, m <= thr0 && nvalid > 0)) break;
            }
            if (ti >= tcount) break;
            unsigned fire = 0;
#pragma unroll
            for (int i = 0; i < H; i++) {
#pragma unroll
                for (int r = 0; r < 2; r++)
                    if (i < nvalid && ti + r < tcount &&
                        __popc(probe_fold<K>(hp[i], s_tp + (ti + r) * PW)) <= thr0)
                        fire |= 1u << (2 * i + r);
            }
            while (fire) {
                const int kk = __ffs(fire) - 1;
                fire &= fire - 1;
                thrH = ptile_exact<W>(p, k, tp, s_rows, v, BKs, &s_un, lane_head + (kk >> 1), ti + (kk & 1), thrH);
            }
            thr0 = thrH >> sshift;
            ti += 2;
        }
        thrH = min(thrH, *(volatile unsigned int *)&p.state->wmin);
    }
    if (threadIdx.x == 0 && s_visited) atomicAdd(&p.state->visited, s_visited);
}

template <int W, bool XP>
int launch_ptile_impl(const ProblemDev &p, const PkgDev &k, const PtileDev &d, const PTilePlan &tp, cudaStream_t st,
                      int num_sms) {
    const size_t smem = ptile_layout(p.G, p.N, W, probe_words(W, XP), k.P, d.E, min(p.BK, tp.g + 2)).total;
    allow_big_smem<ptile_kernel<W, XP>>();
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ptile_kernel<W, XP>, kTileThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const unsigned long long units = (tp.unit_total + tp.shard_world - 1 - tp.shard_rank) / tp.shard_world;
    unsigned long long blocks = (unsigned long long)num_sms * per_sm;
    if (blocks > units) blocks = units;
    if (blocks == 0) return 0;
    ptile_kernel<W, XP><<<unsigned(blocks), kTileThreads, smem, st>>>(p, k, d, tp);
    return 1;
}

size_t tile_smem(int G, int N, int W, int K, int BK) { return tile_smem_layout(G, N, W, K, BK).total; }

template <int W, bool XP>
int launch_tile_impl(const ProblemDev &p, const TilePlan &tp, cudaStream_t st, int num_sms) {
    const size_t smem = tile_smem(p.G, p.N, W, probe_words(W, XP), min(p.BK, tp.g + 2));
    allow_big_smem<tile_kernel<W, XP>>();
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_kernel<W, XP>, kTileThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const unsigned long long units = (tp.unit_total + tp.shard_world - 1 - tp.shard_rank) / tp.shard_world;
    unsigned long long blocks = (unsigned long long)num_sms * per_sm;
    if (blocks > units) blocks = units;
    if (blocks == 0) return 0;
    tile_kernel<W, XP><<<unsigned(blocks), kTileThreads, smem, st>>>(p, tp);
    return 1;
}

size_t problem_smem(int G, int N, int W, int SW, int BK) {
    return ((size_t(G) * N * 2 * W * 4 + 15) & ~size_t(15)) + size_t(N + 1) * BK * 8 + size_t(G) * N * SW * 8;
}

size_t walk_smem(int G, int N, int W, int SW, int BKs) {
    return ((size_t(G) * N * 2 * W * 4 + 15) & ~size_t(15)) + size_t(G) * N * SW * 8 + size_t(N + 1) * BKs * 8;
}

template <int W>
int launch_walk_impl(const ProblemDev &p, const LevelLaunch &L, cudaStream_t st, int num_sms) {
    const size_t smem = walk_smem(p.G, p.N, W, p.SW, max(1, min(p.BK, L.g)));
    allow_big_smem<walk_kernel<W>>();
    const unsigned long long segs = (L.seg_total + L.shard_world - 1 - L.shard_rank) / L.shard_world;
    const int threads = 256;
    unsigned long long blocks = (segs + threads - 1) / threads;
    const unsigned long long cap = (unsigned long long)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) return 0;
    walk_kernel<W><<<unsigned(blocks), threads, smem, st>>>(p, L);
    return 1;
}

// deepest meet-in-the-middle level: level g reads L_0..L_(g-1) of both halves of every slot,
// resident in shared memory (x|z sums and syndromes); returns it and the entries per slot set
constexpr size_t kMitmBytes = 40 * 1024;
static void mitm_plan(int N, int W, int SW, int BK, int &g_out, int &cap_out) {
    g_out = 0;
    cap_out = 0;
    if (W > 2 || SW > 1 || N < 2) return;
    const size_t ent = (size_t(8 * W) + size_t(8 * SW)) * kMitmSlots;
    auto C = [](int n, int k) {
        if (k < 0 || k > n) return 0.0;
        double c = 1;
        for (int i = 1; i <= k; i++) c = c * (n - k + i) / i;
        return c;
    };
    const int nA = N / 2, nB = N - nA;
    double e = 0;  // entries of L_0..L_(g-1), both halves
    for (int g = 1; g <= N && g + 1 < BK && g <= kMitmMaxLevel; g++) {
        e += C(nA, g - 1) + C(nB, g - 1);
        if (e * double(ent) > double(kMitmBytes)) break;
        g_out = g;
        cap_out = int(e) * kMitmSlots;
    }
}

template <int W>
int launch_batch_impl(const BatchDev &b_in, cudaStream_t st) {
    BatchDev b = b_in;
    mitm_plan(b.N, W, b.SW, b.BK, b.mitm_g, b.mitm_cap);
    if (b.no_mitm) b.mitm_g = 0;
    const size_t smem = problem_smem(b.G, b.N, W, b.SW, b.BK) +
                        (b.mitm_g > 0 ? size_t(b.mitm_cap) * size_t(8 * W + 8 * b.SW) + 16 : 0);
    allow_big_smem<batch_kernel<W>>();
    // one code per CTA; small CTAs when there are many codes, so that every SM holds enough of
    // them to cover the per-code level barriers (codes finish at different levels)
    const int threads = b.threads > 0 ? b.threads : 256;
    if (std::getenv("SDB_TRACE_HOST"))
        std::fprintf(stderr, "[sdb] batch kernel: %d codes x %d threads, %zu B smem, meet-in-the-middle levels <= %d (%d entries)\n",
                     b.codes, threads, smem, b.mitm_g, b.mitm_cap);
    batch_kernel<W><<<b.codes, threads, smem, st>>>(b);
    return 1;
}

}  // namespace

size_t problem_smem_bytes(int G, int N, int W, int SW, int BK) { return problem_smem(G, N, W, SW, BK); }

int launch_run_init(const ProblemDev &p, unsigned sentinel, const unsigned long long *counter_init,
                    unsigned long long *counters, int n_counters, void *stream) {
    run_init_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, sentinel, counter_init, counters, n_counters);
    return 1;
}

int launch_level_close(const ProblemDev &p, int g, long long lower, int from_keys, void *stream) {
    level_close_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, g, lower, from_keys);
    return 1;
}
size_t tile_smem_bytes(int G, int N, int W, int K, int BK) { return tile_smem(G, N, W, K, BK); }

int launch_tile_level(const ProblemDev &p, const TilePlan &tp, void *stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool xp = p.K > p.W && p.W > 1;
#define SDB_TILE_CASE(w)                                                                                 \
    case w: return xp ? launch_tile_impl<w, true>(p, tp, st, num_sms) : launch_tile_impl<w, false>(p, tp, st, num_sms);
    switch (p.W) {
        case 1: return launch_tile_impl<1, false>(p, tp, st, num_sms);
        SDB_TILE_CASE(2)
        SDB_TILE_CASE(3)
        SDB_TILE_CASE(4)
        SDB_TILE_CASE(5)
        SDB_TILE_CASE(6)
        SDB_TILE_CASE(7)
        SDB_TILE_CASE(8)
    }
#undef SDB_TILE_CASE
    return -1;
}

int launch_tc_level(const ProblemDev &p, const TcPlan &tp, void *stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (p.W) {
        case 1: return launch_tc_w<1>(p, tp, st, num_sms);
        case 2: return launch_tc_w<2>(p, tp, st, num_sms);
        case 3: return launch_tc_w<3>(p, tp, st, num_sms);
        case 4: return launch_tc_w<4>(p, tp, st, num_sms);
    }
    return -1;
}

int launch_walk_level(const ProblemDev &p, const LevelLaunch &L, void *stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (p.W) {
        case 1: return launch_walk_impl<1>(p, L, st, num_sms);
        case 2: return launch_walk_impl<2>(p, L, st, num_sms);
        case 3: return launch_walk_impl<3>(p, L, st, num_sms);
        case 4: return launch_walk_impl<4>(p, L, st, num_sms);
        case 5: return launch_walk_impl<5>(p, L, st, num_sms);
        case 6: return launch_walk_impl<6>(p, L, st, num_sms);
        case 7: return launch_walk_impl<7>(p, L, st, num_sms);
        case 8: return launch_walk_impl<8>(p, L, st, num_sms);
    }
    return -1;
}

size_t pkg_smem_bytes(int G, int N, int W, int SW, int P, int BK) {
    size_t a, b, c, d;
    return pkg_layout(G, N, W, SW, P, BK, &a, &b, &c, &d);
}

int launch_pkg_level(const ProblemDev &p, const PkgDev &k, const PkgLevel &L, void *stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (p.W) {
        case 1: return launch_pkg_impl<1>(p, k, L, st, num_sms);
        case 2: return launch_pkg_impl<2>(p, k, L, st, num_sms);
        case 3: return launch_pkg_impl<3>(p, k, L, st, num_sms);
        case 4: return launch_pkg_impl<4>(p, k, L, st, num_sms);
        case 5: return launch_pkg_impl<5>(p, k, L, st, num_sms);
        case 6: return launch_pkg_impl<6>(p, k, L, st, num_sms);
        case 7: return launch_pkg_impl<7>(p, k, L, st, num_sms);
        case 8: return launch_pkg_impl<8>(p, k, L, st, num_sms);
    }
    return -1;
}

int launch_brute(const BruteDev &b, void *stream, int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned long long total = (1ull << b.n_rows) - 1;
    const unsigned long long nblk = (total + (1ull << b.block_log2)) >> b.block_log2;
    unsigned long long blocks = (nblk + 255) / 256;
    if (blocks > (unsigned long long)num_sms * 8) blocks = (unsigned long long)num_sms * 8;
    if (blocks == 0) blocks = 1;
    switch (b.W) {
        case 1: brute_kernel<1><<<unsigned(blocks), 256, 0, st>>>(b); return 1;
        case 2: brute_kernel<2><<<unsigned(blocks), 256, 0, st>>>(b); return 1;
        case 3: brute_kernel<3><<<unsigned(blocks), 256, 0, st>>>(b); return 1;
        case 4: brute_kernel<4><<<unsigned(blocks), 256, 0, st>>>(b); return 1;
    }
    return -1;
}

size_t ptile_smem_bytes(int G, int N, int W, int K, int P, int E, int BKs) {
    return ptile_layout(G, N, W, K, P, E, BKs).total;
}

int launch_ptile_level(const ProblemDev &p, const PkgDev &k, const PtileDev &d, const PTilePlan &tp, void *stream,
                       int num_sms) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool xp = p.K > p.W && p.W > 1;
#define SDB_PTILE_CASE(w)                                                                                \
    case w:                                                                                              \
        return xp ? launch_ptile_impl<w, true>(p, k, d, tp, st, num_sms)                                 \
                  : launch_ptile_impl<w, false>(p, k, d, tp, st, num_sms);
    switch (p.W) {
        case 1: return launch_ptile_impl<1, false>(p, k, d, tp, st, num_sms);
        SDB_PTILE_CASE(2)
        SDB_PTILE_CASE(3)
        SDB_PTILE_CASE(4)
        SDB_PTILE_CASE(5)
        SDB_PTILE_CASE(6)
        SDB_PTILE_CASE(7)
        SDB_PTILE_CASE(8)
    }
#undef SDB_PTILE_CASE
    return -1;
}

int launch_batch(const BatchDev &b, void *stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (b.W) {
        case 1: return launch_batch_impl<1>(b, st);
        case 2: return launch_batch_impl<2>(b, st);
        case 3: return launch_batch_impl<3>(b, st);
        case 4: return launch_batch_impl<4>(b, st);
        case 5: return launch_batch_impl<5>(b, st);
        case 6: return launch_batch_impl<6>(b, st);
        case 7: return launch_batch_impl<7>(b, st);
        case 8: return launch_batch_impl<8>(b, st);
    }
    return -1;
}

}  // namespace sdb
