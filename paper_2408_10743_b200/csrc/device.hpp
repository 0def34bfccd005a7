// Shared host/device description of one enumeration problem (all Gamma_j of one code,
// singleton packages) and the kernel entry points in kernels.cu.
//
// HBM layout (one allocation per plan, all 16-byte aligned):
//   rows  u32 [G][N][2W]   row r of Gamma_j: W probe words then W partner words. Word w
//                          of the pair holds symbols 32w..32w+31 of the x block or the z
//                          block (the reference's EnumMatrix symplectic split,
//                          engine.cpp:58-97); per (Gamma, w) the host puts the denser of the
//                          two in the probe slot (orient_probe_words) — popc(x|z) is symmetric
//   syn   u64 [G][N][SW]   compressed admissibility syndrome of each row (SW=0: no filter)
//   binom u64 [N+1][BK]    saturating binomials C(a,b), b < BK
//   state LevelState       per-level running minimum + per-weight best keys
// Weight of a candidate = scale * sum_i popc(x_i | z_i); scale = 2 on the isometry
// route (Hamming weight of (a|b|a^b) = 2 popc(a|b), prep.hpp:66-68), 1 otherwise.
#pragma once

#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define SDB_HD __host__ __device__
#else
#define SDB_HD
#endif

// Bounds checks of the kernels' shared-memory and combination indexing, compiled in only for
// the checked build (tools/build_variant.sh checked "-DSDB_DEBUG_CHECKS", run under the GPU
// test suite with SDB_TEST_VARIANT=checked): compute-sanitizer is not available on the GPU
// pool, so out-of-range indices trap here instead.
#if defined(SDB_DEBUG_CHECKS) && defined(__CUDA_ARCH__)
#define SDB_CHECK(cond)                                                                          \
    do {                                                                                         \
        if (!(cond)) {                                                                           \
            printf("SDB_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   int(blockIdx.x), int(threadIdx.x));                                           \
            __trap();                                                                            \
        }                                                                                        \
    } while (0)
#else
#define SDB_CHECK(cond) ((void)0)
#endif

namespace sdb {

constexpr int kMaxW = 8;         // u32 words per half: n <= 256
constexpr int kMaxSW = 4;        // u64 syndrome words: 2k <= 256
constexpr int kMaxG = 64;        // matrices per code
constexpr int kMaxLevel = 62;    // combination size handled by the kernels
constexpr int kKeyRankBits = 58; // key = gamma << 58 | lexicographic rank
constexpr uint64_t kNoKey = ~uint64_t(0);

struct LevelState {
    unsigned int wmin;           // min weight found this level (engine units), ~0u: none
    unsigned int pad;
    unsigned long long visited;  // candidates the kernels enumerated
    unsigned long long skipped;  // candidates left out by the mid-level early exit (early_skip)
    // followed in memory by key_by_w[max_weight + 1] (u64)
};

// Device-resident level-loop state (reference BoundsState, engine.hpp:26-33): the host
// enqueues levels without waiting for each one; level_close folds a level's minimum into
// U, writes the trace entry and raises `done` once L(g) >= U, after which every later
// level kernel returns at once.
struct RunCtl {
    unsigned int U;                 // upper bound in engine units
    int done;                       // 1 once L(g) >= U (reference run_bz break, engine.cpp:334)
    int best_g;                     // level of the best candidate (-1: none)
    int pad;
    unsigned long long best_key;    // gamma << 58 | lexicographic rank
    unsigned long long visited;     // candidates the kernels enumerated, all levels
    unsigned long long skipped;     // candidates the mid-level early exit left out, all levels
};

struct ProblemDev {
    const uint32_t *rows;
    const unsigned long long *syn;
    const unsigned long long *binom;
    LevelState *state;
    unsigned long long *key_by_w;
    RunCtl *ctl;
    int *trace_upper;               // [N + 1]: U after level g (-1: level skipped)
    const uint32_t *prows;          // [G][N][K] the tile kernels' probe words of every row
    int K;                          // probe words per row (W, W + 1 with an extra probe, 2 when W = 1)
    int G, N, W, SW, BK;
    int scale;
    int max_weight;
};

struct LevelLaunch {
    int g;
    unsigned int thr0;            // only candidates with weight <= thr0 are considered (U - 1)
    unsigned long long per_gamma; // C(N, g)
    unsigned long long seg_len;   // lexicographic ranks per walk segment
    unsigned long long segs_per_gamma;
    // sharding: this rank takes segments rank, rank + world, ... of [0, seg_total)
    unsigned long long seg_total;
    int shard_rank, shard_world;
    unsigned int lprev;           // L(g - 1): the mid-level early exit's bound (0: off)
};

// Level-loop control kernels (one CTA each): reset U / best / counters for a run, and
// close one level (fold the level minimum into U, trace, termination, reset the level).
int launch_run_init(const ProblemDev &p, unsigned sentinel, const unsigned long long *counter_init,
                    unsigned long long *counters, int n_counters, void *stream);
int launch_level_close(const ProblemDev &p, int g, long long lower, int from_keys, void *stream);

// One level, all matrices, lexicographic-walk kernel. Returns the number of kernels launched.
int launch_walk_level(const ProblemDev &p, const LevelLaunch &L, void *stream, int num_sms);

// One level, all matrices, head x tail tile kernel (large levels).
//
// Every g-subset S of the N rows splits at b = the smallest of its last t elements into a
// head (h = g - t elements, all < b) and a tail ({b} plus t-1 elements > b). For fixed
// (Gamma j, b) the candidates are the outer product Heads_b x Tails_b, with
// |Heads_b| = C(b, h) (colex ranks of h-subsets of [0, b)) and |Tails_b| = C(N-1-b, t-1).
// A work unit is (j, b, head block of head_block(W) heads, tail chunk of kTailChunk tails):
// the CTA stages the tail chunk in shared memory, each lane holds heads_per_lane(W) heads in
// registers and streams the tails as warp-uniform broadcast loads, so one candidate is
// one XOR of two precomputed sums fused with the OR (2 LOP3) plus one POPC.
#ifndef SDB_TILE_THREADS
#define SDB_TILE_THREADS 256
#endif
constexpr int kTileThreads = SDB_TILE_THREADS;
// heads held in registers per lane (2W words each); fewer for wide rows to avoid spills
#ifndef SDB_HEADS_W2
#define SDB_HEADS_W2 8
#endif
// K = 3 probe words (W = 3, or W = 2 with the extra probe): 6 heads, so 18 head registers
// fit 4 CTAs/SM
#ifndef SDB_HEADS_K3
#define SDB_HEADS_K3 6
#endif
SDB_HD constexpr int heads_per_lane(int W, int K) {
    return K == 3 ? SDB_HEADS_K3 : W <= 2 ? SDB_HEADS_W2 : W <= 3 ? 8 : (W <= 5 ? 4 : 2);
}
SDB_HD constexpr int head_block(int W, int K) { return kTileThreads * heads_per_lane(W, K); }
#ifndef SDB_TAIL_CHUNK
#define SDB_TAIL_CHUNK 1024
#endif
constexpr int kTailChunk = SDB_TAIL_CHUNK;
// resident CTAs per SM (the register cap: 64 registers at 4, 80 at 3), by the head registers
// per lane, K probe words (W, or W + 1 with the extra probe) x heads_per_lane(W, K); measured
// on B200 (profiles/): K <= 2 with 8 heads runs best at 4, K = 3 with 8 heads spills there and
// runs best at 3, K = 3 with 6 heads (W = 3) runs 1.8% faster at 4 than 8 heads at 3
#ifndef SDB_TILE_BLOCKS_W2
#define SDB_TILE_BLOCKS_W2 4
#endif
#ifndef SDB_TILE_BLOCKS
#define SDB_TILE_BLOCKS 3
#endif
SDB_HD constexpr int probe_words(int W, bool XP) { return W == 1 ? 2 : W + (XP ? 1 : 0); }
SDB_HD constexpr int tile_blocks_per_sm(int W, int K) {
    return (K * heads_per_lane(W, K) <= 18 ? SDB_TILE_BLOCKS_W2 : SDB_TILE_BLOCKS) *
           (256 / kTileThreads);
}
// Staged tail chunk: the probe words of each tail, [kTailChunk+1][probe_stride(K)] with K =
// probe words per row (ProblemDev.prows). probe_stride is even so two tails are whole 16-byte
// loads. The rare exact path rebuilds candidates from the full rows, so nothing else is
// staged per tail.
SDB_HD constexpr int probe_stride(int K) { return (K + 1) & ~1; }
SDB_HD constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
struct TileSmem {
    size_t rows, prows, adj, binom, tp, total;
};
SDB_HD inline TileSmem tile_smem_layout(int G, int N, int W, int K, int BK) {
    TileSmem L{};
    L.rows = 0;
    L.prows = align16(size_t(G) * N * 2 * W * 4);
    L.adj = align16(L.prows + size_t(G) * N * K * 4);  // prows[r] ^ prows[r + 1]
    L.binom = align16(L.adj + size_t(G) * N * K * 4);
    L.tp = align16(L.binom + size_t(N + 1) * BK * 8);
    L.total = align16(L.tp + size_t(kTailChunk + 1) * probe_stride(K) * 4);
    return L;
}

struct TilePlan {
    int g, t, h;
    int tchunk;                     // tails per unit (<= kTailChunk; smaller for mid-size levels)
    unsigned int thr0;              // candidates with weight <= thr0 are considered (U - 1)
    int nb;                         // number of boundaries b in [h, N - t]
    const unsigned long long *cum;  // [G * nb + 1] cumulative unit counts over (j, b)
    unsigned long long *counter;    // dynamic dispenser of this rank's units (starts at 0)
    // sharding: dispensed value i is unit i * shard_world + shard_rank of [0, unit_total);
    // interleaving keeps neighbouring (similar-sized) units on different ranks
    unsigned long long unit_total;
    int shard_rank, shard_world;
    unsigned long long per_gamma;   // C(N, g): lexicographic-rank base
    unsigned int lprev;             // L(g - 1): the mid-level early exit's bound (0: off)
};
int launch_tile_level(const ProblemDev &p, const TilePlan &tp, void *stream, int num_sms);

// Tensor-core tile kernel (tc_tile_kernel, tc_tile.cuh): the same head x tail units, scored as
// an int8 GEMM on tcgen05 with the accumulators in TMEM. Per Gamma the host (tcenc.cpp) maps
// every symbol s to one or three ±1 coordinates so that, for a candidate split into a head
// S_h and a tail S_t,
//     S * popc(x|z) = C0 + c_h + sum_k head_k * tail_k
// exactly: a symbol whose a, b or a^b column is a unit column (one row p holds its 1) is
// nonzero iff p is chosen or its other component is odd, one coordinate with the component's
// sign, zeroed on the side that chose p ("mask"), c = alpha * |S ∩ mask rows|; a symbol with
// no unit column takes three coordinates (a, b, a^b), (3 - sum s_h s_t) / 4. The CTA pipeline
// (one CTA per SM): a unit warp claims units, eight producer warps write their tail tiles (B,
// double-buffered) and head tiles (A, a ring of four), one thread issues tcgen05.mma
// kind::i8 into two 256-column TMEM stages, and 8 epilogue warps read the s32 accumulators
// back as packed 16-bit pairs (tcgen05.ld pack::16b) with a running VIMNMX.S16x2 minimum; only
// a pair at or below the row's threshold takes the exact rare path (tile_exact), so results
// are bit-identical to the POPC kernels.
constexpr int kTcHeads = 128;      // heads per head tile (MMA M)
#ifndef SDB_TC_UNIT_TILES
#define SDB_TC_UNIT_TILES 16
#endif
constexpr int kTcUnitTiles = SDB_TC_UNIT_TILES;  // head tiles per unit (a unit holds up to 128 x this many heads)
constexpr int kTcMaxPart = 8;      // h <= 8 and t - 1 <= 8 (element lists live in registers)
constexpr int kTcTileN = 256;      // tails per B tile = MMA N = TMEM columns per stage
constexpr int kTcStages = 2;       // TMEM stages (512 columns)
constexpr int kTcProdWarps = 8;    // producer warps: two groups of 4 (alternate head tiles; 128 rows each)
#ifndef SDB_TC_SLOTS
#define SDB_TC_SLOTS 4
#endif
constexpr int kTcSlots = SDB_TC_SLOTS;  // head tiles in flight (A ring)
constexpr int kTcUnitQ = 8;        // unit descriptors in flight
constexpr int kTcEpiWarps = 8;
constexpr int kTcThreads = 32 * (1 + kTcEpiWarps + 1 + kTcProdWarps);
constexpr int kTcMaxK = 128;       // coordinates per operand row
constexpr int kTcMaxNbt = 12;      // B tiles per unit (tail tiles a head tile meets)
constexpr int kTcMaxBSlots = kTcMaxNbt + 1;  // B tile ring: one spare slot lets the next chunk start early
struct TcGammaDev {
    int K;       // coordinates of this Gamma (multiple of 32; MMA K steps = K / 32)
    int W1;      // 4-coordinate words whose tail coefficient is alpha (S = 4: 2), the rest 1
    int C0;      // constant of S * weight
    int kc;      // the coordinate carrying -c_t on the tail side (head side -1)
    int S;       // weight scale (2: only unit-column symbols, 4: otherwise)
    int alpha;   // S / 2
    int kt;      // threshold coordinates kt, kt + 1: tail bytes 1, 16; head bytes r, q with
                 // 16 q + r = -(T + 1), so the accumulator is val - T - 1 (< 0 iff val <= T)
};
// One unit in flight. Head row r of tile a (a < na) is head rank hbase0 + r * na + a; tail
// row y of the unit's B tiles is tail rank t0 + (y % 256) * nbt + y / 256 (each producer
// thread walks consecutive ranks with colex successors and writes them to rows that keep its
// stores conflict-free).
struct TcUnitDesc {
    unsigned long long hbase0, t0;
    int j, b, nheads, ntails, nbt, na, chunk_last, restage, end, pad;  // chunk_last: the next unit restages
};
// What the MMA warp needs of a unit, in one word (TcUnitDesc::pad) it makes warp-uniform with
// one redux.sync: na | nbt << 8 | K / 32 << 16 | flags.
constexpr unsigned kTcWordRestage = 1u << 20, kTcWordChunkLast = 1u << 21, kTcWordEnd = 1u << 22;
SDB_HD inline unsigned tc_unit_word(const TcUnitDesc &d, int kt) {
    return unsigned(d.na) | unsigned(d.nbt) << 8 | unsigned(kt) << 16 | (d.restage ? kTcWordRestage : 0u) |
           (d.chunk_last ? kTcWordChunkLast : 0u) | (d.end ? kTcWordEnd : 0u);
}
// -(T + 1) as the head's two threshold bytes (r at kt, q at kt + 1; the tail holds 1, 16),
// clamped to what they can carry: a larger T only sends more pairs down the exact path, a
// T below -2048 passes nothing either way (|val| <= 2 K)
SDB_HD inline void tc_threshold_bytes(int T, int &r, int &q) {
    int m = -(T + 1);
    m = m < -2048 ? -2048 : m > 2047 ? 2047 : m;
    q = m >> 4;  // floor division: -2048 .. 2047 -> -128 .. 127
    r = m & 15;
}
struct TcPlan {
    TilePlan tile;            // unit table over head blocks of kTcHeads * kTcUnitTiles, tchunk = kTcTileN * nbt
    int nbt;                  // B tiles per unit
    int kmax, kw;             // bytes (coordinates) per operand row, sign words per row
    const uint32_t *sign;     // [G][N][kw] coordinate sign bits (bit 8i + j of word w: coordinate 32w + 4j + i)
    const short *mask;        // [G][N] coordinate a row masks (-1: none)
    const TcGammaDev *gam;    // [G]
};
struct TcSmem {
    size_t a, b, sign, mask, rows, binom, uq, gam, cum, total;
};
SDB_HD inline TcSmem tc_smem_layout(int G, int N, int W, int kmax, int kw, int nbt, int BKs) {
    TcSmem L{};
    L.a = 0;
    L.b = L.a + size_t(kTcSlots) * kTcHeads * kmax;
    L.sign = L.b + size_t(nbt + 1) * kTcTileN * kmax;  // the B ring: nbt + 1 tail tiles
    L.mask = align16(L.sign + size_t(G) * N * kw * 4);
    L.rows = align16(L.mask + size_t(G) * N * 2);
    L.binom = align16(L.rows + size_t(G) * N * 2 * W * 4);
    L.uq = align16(L.binom + size_t(N + 1) * BKs * 8);
    L.gam = align16(L.uq + size_t(kTcUnitQ) * sizeof(TcUnitDesc));
    L.cum = align16(L.gam + size_t(G) * sizeof(TcGammaDev));       // the level's unit table
    L.total = align16(L.cum + (size_t(G) * (N + 1) + 1) * 8);
    return L;
}
constexpr size_t kTcSmemMax = 224 * 1024;  // dynamic; the kernel adds ~1 KB of static shared memory
int launch_tc_level(const ProblemDev &p, const TcPlan &tp, void *stream, int num_sms);

// Package routes (Saved_1_Gamma / Saved_2_Gamma): a level-g
// candidate picks g packages p_1 < ... < p_g and one member row of each; the reference
// visits them in lexicographic order of (p_1, m_1, p_2, m_2, ...) (engine.cpp:202-219).
// pkg_kernel<W> walks segments of that order: unrank through weighted suffix counts
// wsuf(q, m) = number of m-package choices with members among packages [q, P), then the
// lexicographic successor (next member of the deepest package that has one, else the next
// package), one or a few row XORs per step.
constexpr int kMaxPkgG = 4;
struct PkgDev {
    const short *pk_rows;              // [G][P][3] member rows, -1 padding
    const unsigned char *pk_size;      // [G][P] members per package (1 or 3)
    const unsigned long long *wsuf;    // [G][P + 1][BK]
    int P;                             // package slots per Gamma (max over Gammas)
    int np[kMaxPkgG];                  // packages of each Gamma
};
struct PkgLevel {
    int g;
    unsigned int thr0;
    unsigned long long seg_len;
    unsigned long long total[kMaxPkgG];  // candidates of each Gamma at this level
    unsigned long long segs[kMaxPkgG];   // segments of each Gamma
    unsigned long long seg_total;
    int shard_rank, shard_world;
    unsigned int lprev;           // L(g - 1): the mid-level early exit's bound (0: off)
};
size_t pkg_smem_bytes(int G, int N, int W, int SW, int P, int BK);

// Packaged head x tail tile kernel (ptile_kernel<W>). A package member is an "element"
// e = off(q) + m of Gamma j; a candidate is a set of g elements from distinct packages.
// Element sets are enumerated in colex order with weighted counts
//   F(x, i) = number of i-element sets with distinct packages inside elements [0, x)
//           = F(x-1, i) + F(off(pkg(x-1)), i-1),
// forward for heads (packages < b) and over the reversed package order for tails (packages
// > b), so heads and tails unrank and step exactly like the singleton tile kernel.
struct PtileDev {
    const short *e_row, *e_pkg;          // [G][E] forward: row / package of element e
    const short *r_row, *r_pkg;          // [G][E] reversed package order
    const short *off, *r_off;            // [G][P + 1] first element of package q
    const unsigned long long *F, *FR;    // [G][E + 1][BK]
    int E;                               // element slots per Gamma
};
struct PTilePlan {
    int g, t, h, tchunk;
    unsigned int thr0;
    int npairs;                          // (Gamma, b) pairs with work
    const unsigned long long *cum;       // [npairs + 1] cumulative unit counts
    const unsigned int *pairs;           // [npairs] j << 16 | b
    unsigned long long *counter;
    unsigned long long unit_total;
    int shard_rank, shard_world;
};
size_t ptile_smem_bytes(int G, int N, int W, int K, int P, int E, int BKs);
int launch_ptile_level(const ProblemDev &p, const PkgDev &k, const PtileDev &d, const PTilePlan &tp, void *stream,
                       int num_sms);
int launch_pkg_level(const ProblemDev &p, const PkgDev &k, const PkgLevel &L, void *stream, int num_sms);

// Brute force (reference brute_force_distance, distance.cpp:151-224): the Gray-code walk over
// all 2^rows - 1 combinations of the normalizer rows, one row XOR per step, the C-membership
// syndrome accumulated alongside; minimum symplectic weight of the admissible ones.
struct BruteDev {
    const uint32_t *rows;               // [rows][2W]
    const unsigned long long *syn;      // [rows] (filter on) bit j = <row_i, row_j>_s
    unsigned int *best;                 // min weight (atomicMin), ~0u: none
    int n_rows, W, filter;
    int block_log2;                     // Gray indices per thread = 2^block_log2
};
int launch_brute(const BruteDev &b, void *stream, int num_sms);

// Batch: one code per CTA, the whole level loop on the device.
struct BatchDev {
    const uint32_t *rows;      // [codes][G][N][2W]
    const unsigned long long *syn;       // [codes][G][N][SW]
    const int *deficits;       // [codes][G]
    const unsigned long long *binom;     // [N+1][BK]
    int *out_upper;            // [codes] final U (engine units)
    int *out_generations;      // [codes]
    int *out_status;           // [codes] 0 ok, 3 no admissible codeword
    int *out_trace_lower;      // [codes][N]
    int *out_trace_upper;      // [codes][N]
    const int *in_status;      // [codes] or null: codes with a nonzero prep status are skipped
    int codes, G, N, W, SW, BK, scale, sentinel;
    int Gs;                    // Gamma slots per code in rows/syn/deficits (>= G)
    int max_g;                 // last level to run (RunOptions.max_generation; N when 0)
    const int *n_gammas;       // [codes] matrices per code (device prep) or null: G for all
    int threads;               // CTA size (a multiple of 32; 0 = 256)
    int no_mitm;               // 1: every level on the per-thread walk (tests)
    int mitm_g, mitm_cap;      // set by the launcher: meet-in-the-middle levels and list entries
};
// out_status of a code whose prep produced more matrices than the batch has slots
constexpr int kBatchNeedsHostPrep = 5;
int launch_batch(const BatchDev &b, void *stream);

// Batch prep on the device, one warp per code (BASELINE config 3):
// validate_normalizer, isometry_transform, information_sets and the admissibility
// syndromes with the host's (= reference's) pivot rules, writing the batch kernel's inputs.
// Limits: n + k <= 64 rows, n <= 64; codes needing more than Gs matrices report G > Gs and
// the host redoes the batch with host prep.
constexpr int kPrepMaxRows = 64;
constexpr int kPrepMaxN = 64;
constexpr int kPrepGammaSlots = 4;
struct BatchPrepDev {
    const unsigned long long *normalizers;  // [codes][N][in_words]
    int in_words;
    int codes, N, n, W;
    int validate, filter;                   // filter: dual_filter && k >= 1
    uint32_t *rows;                         // [codes][Gs][N][2W]
    unsigned long long *syn;                // [codes][Gs][N] (filter) — raw N-bit syndromes
    int *deficits;                          // [codes][Gs]
    int *n_gammas;                          // [codes]
    int *status;                            // [codes]: 0 ok, 2 validation
    int Gs;
    int force_rows;                         // 1: the row-major kernel even for small codes (tests)
};
int launch_batch_prep(const BatchPrepDev &d, void *stream);

}  // namespace sdb
