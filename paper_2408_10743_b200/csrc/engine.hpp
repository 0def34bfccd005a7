// Host engine: builds device problems from Gamma_j, runs the level loop
// (reference run_bz, engine.cpp:303-343) with one kernel launch per level, and the
// batch path (one code per CTA).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

#include "device.hpp"
#include "gf2.hpp"
#include "tcenc.hpp"
#include "../../include/symdist_b200.h"

namespace sdb {

enum class Mode { symplectic = 0, hamming = 1 };

// One prepared matrix (singleton packages, prep.hpp:25-35 with packages[i] = {pivot, {i}}).
struct GammaIn {
    GammaIn() = default;
    GammaIn(BitMat m, int deficit) : matrix(std::move(m)), rank_deficit(deficit) {}
    BitMat matrix;
    int rank_deficit = 0;
    // package routes: member rows of each package (1 or 3 rows); empty = every row is its
    // own package, in row order. n_pp: packages pivoted on principal columns (-1: all)
    std::vector<std::vector<int>> packages;
    int n_pp = -1;
};

struct Filter {
    bool enabled = false;
    BitMat rows;  // rows spanning C_perp in the frame of the first 2n columns
};

struct LevelResult {
    int g = 0;
    long long lower = 0, upper = 0;
    double seconds = 0;
    bool improved = false;
    int best_gamma = -1;
    unsigned long long best_rank = 0;
};

class Plan {
   public:
    Plan(std::vector<GammaIn> gammas, Mode mode, int pair_count, const Filter &filter, const sdb_run_options &opts);
    ~Plan();
    Plan(const Plan &) = delete;
    Plan &operator=(const Plan &) = delete;

    // Runs the generation loop from device-resident data; fills report/trace (trace_cap
    // entries) and, when best_out != nullptr, the best codeword in the Gamma frame.
    void run(sdb_report *report, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out,
             double *level_seconds);

    // One generation of a single-matrix plan folded into a bounds state (reference
    // enumerate_generation, engine.cpp:296-301): candidates with weight below `upper` (the
    // sentinel when 0) lower it; returns whether one did, the new upper, this generation's
    // candidate count and, when it improved, the first minimal codeword in the Gamma frame.
    bool run_level(int g, long long upper, long long *upper_out, unsigned long long *candidates,
                   uint64_t *best_out);

    double h2d_seconds = 0;
    unsigned long long upload_bytes = 0;
    int n_gammas() const { return G_; }
    int sentinel() const { return sentinel_; }

   private:
    // host-side launch description of one level, built the first time a run reaches it
    struct LevelHost {
        bool ready = false;
        bool sharded = false;         // split across ranks (else every rank runs it whole)
        int t = 0;                    // 0: walk kernel, else the tile kernel's tail size
        LevelLaunch walk{};
        TilePlan tile{};
        PkgLevel pkg{};
        PTilePlan ptile{};
        TcPlan tc{};                  // t == -3: tensor-core tile kernel
    };

    void upload();
    int launch_level(int g);  // the level's kernel(s) on the plan's stream; returns the launch count
    long long lower_bound(int g) const;
    unsigned early_bound(int g) const;
    void prepare_level(int g);
    bool prepare_ptile(int g, LevelHost &lv, int world, int rank);
    bool prepare_tc(int g, LevelHost &lv, int world, int rank);
    cudaEvent_t level_event(int i);

    std::vector<GammaIn> gammas_;
    Mode mode_;
    int pair_count_;
    sdb_run_options opts_;
    int G_ = 0, N_ = 0, W_ = 0, SW_ = 0, BK_ = 0, scale_ = 1, max_weight_ = 0, sentinel_ = 0;
    bool image_layout_ = false;
    std::vector<uint32_t> h_rows_;
    std::vector<uint32_t> h_prows_;  // [G][N][K_] the tile kernels' probe words
    int K_ = 1;
    bool single_level_ = false;  // run_level (the enumerate_generation seam): no early exit
    std::vector<uint64_t> h_syn_;
    std::vector<unsigned long long> h_binom_;
    int device_ = 0, num_sms_ = 148;
    cudaStream_t stream_ = nullptr;
    void *d_mem_ = nullptr;
    size_t d_bytes_ = 0;
    ProblemDev pd_{};
    std::vector<LevelHost> levels_;             // [N + 1]
    std::vector<cudaEvent_t> events_;           // 2 per level: before the level kernel, after its close
    unsigned long long *d_counters_ = nullptr;  // [N + 1] tile unit dispensers, one per level
    unsigned long long *d_counter_init_ = nullptr;
    unsigned long long *d_tables_ = nullptr;    // tile unit tables of all levels, back to back
    size_t table_cap_ = 0, table_used_ = 0;
    std::vector<unsigned long long> h_counter_init_;
    unsigned char *h_stage_ = nullptr;         // pinned staging image of the device block
    RunCtl *h_ctl_ = nullptr;                  // its ctl section: target of the level checks' D2H
    unsigned long long *h_pinned_ = nullptr;  // its unit-table section (table_cap_ entries)
    // tensor-core tile kernel: coordinate encoding of every Gamma (tcenc.hpp)
    bool tc_ok_ = false;
    TcEncoding tc_enc_;
    const uint32_t *d_tc_sign_ = nullptr;
    const short *d_tc_mask_ = nullptr;
    const TcGammaDev *d_tc_gam_ = nullptr;
    // package routes
    bool packaged_ = false;
    int P_ = 0;                                  // package slots per Gamma
    std::vector<int> np_;                        // packages of each Gamma
    std::vector<short> h_pk_rows_;               // [G][P][3]
    std::vector<unsigned char> h_pk_size_;       // [G][P]
    std::vector<unsigned long long> h_wsuf_;     // [G][P + 1][BK]
    PkgDev pk_{};
    // packaged tile kernel: expanded elements and weighted colex counts (PtileDev)
    int E_ = 0;
    std::vector<short> h_e_row_, h_e_pkg_, h_r_row_, h_r_pkg_, h_off_, h_r_off_;
    std::vector<unsigned long long> h_F_, h_FR_;
    PtileDev pt_{};
    unsigned long long F_at(int j, int x, int i) const { return h_F_[(size_t(j) * (E_ + 1) + x) * BK_ + i]; }
    unsigned long long FR_at(int j, int x, int i) const { return h_FR_[(size_t(j) * (E_ + 1) + x) * BK_ + i]; }
    unsigned long long level_candidates(int g) const;
    void unrank_best(int g, int j, unsigned long long r, std::vector<uint64_t> &acc) const;
};

// Host cost model for one level: 0 = lexicographic-walk kernel, else the tail size t of
// the head x tail tile kernel. Exposed for tests.
struct TileChoice {
    int t;       // 0: walk kernel
    int tchunk;  // tails per unit
};
TileChoice choose_tile(int G, int N, int g, int W, int K, unsigned long long per_gamma, int forced_kernel, int num_sms,
                       int world);
// levels with fewer candidates run whole on every rank (RunOptions.shard_min = 0)
constexpr unsigned long long kDefaultShardMin = 1ull << 26;
int choose_tile_t(int G, int N, int g, int W, unsigned long long per_gamma, int forced_kernel);

// Tensor-core levels: the head x tail units on tcgen05 (device.hpp: TcPlan). Levels with at
// least this many candidates take it when the plan's encoding allows (RunOptions.kernel 0);
// kernel 4 forces it on every level with g >= 2, kernel 2 forces the POPC tile kernel.
constexpr unsigned long long kTcMinCandidates = 1ull << 24;
struct TcChoice {
    int t;    // 0: not worth it / not possible
    int nbt;  // B tiles per unit
};
TcChoice choose_tc(int G, int N, int g, const std::vector<TcGammaDev> &gam, int kmax, int kw, int W, int BK,
                   int num_sms, int world);

// Per Gamma and 32-symbol block, swap the x- and z-words of every row so that the word the
// tile kernel's fast path folds (the first of the block) is the denser one. Weights are
// unchanged (popc(x|z) is symmetric).
struct ProbeChoice {
    std::vector<int> extra;  // per Gamma: the block whose partner word may join the probe
    bool use_extra = false;  // probe words per row = W + 1 (else W; 2 when W = 1)
    std::vector<int> fill;   // per Gamma: the block whose partner fills the last block's free bits
    uint32_t free_mask = 0;  // bit positions of the last block that hold no symbol
};
// bits: symbols per half (the last block holds bits - 32 (W - 1) of them)
ProbeChoice orient_probe_words(std::vector<uint32_t> &rows, int G, int N, int W, int bits);

// Saturating binomial table (N+1) x BK.
std::vector<unsigned long long> binom_table(int N, int BK);

// Compressed syndromes for all rows of all gammas (G*N rows), filter semantics of
// AdmissibilityFilter::for_rows; returns SW (0 when disabled).
int build_syndromes(const std::vector<GammaIn> &gammas, int n, const Filter &f, std::vector<uint64_t> &out);

void check_cuda(cudaError_t e, const char *what);

// brute_force_distance (distance.cpp:151-224) on the device; returns the minimum symplectic
// weight of the admissible combinations (throws InternalFailure when there is none).
int run_brute(const BitMat &a, const sdb_run_options &o, double *device_seconds);

// Batch of same-shape normalizers, one code per CTA.
void run_batch(const uint64_t *rows, int n_codes, int n_rows, int n_cols, int row_words, const sdb_run_options &o,
               int *distances, int *statuses, int *generations, sdb_trace_entry *traces, int *trace_lens,
               int trace_cap, double *device_seconds);

}  // namespace sdb
