/*
 * symdist_b200.h — C-ABI drop-in boundary for the symplectic Brouwer-Zimmermann
 * enumeration hot path on B200 (sm_100a).
 *
 * Plain pointers and sizes only (no torch, no C++ types). Every entry point is
 * synchronous, allocates nothing on the caller's behalf and returns an sdb_status.
 * Matrices are bit-packed rows: row r occupies `row_words` = ceil(n_cols/64)
 * little-endian uint64 words at rows + r*row_words, column c at bit c%64 of word
 * c/64, padding bits zero — the reference's BitVector layout
 * (proj/include/symdist/bitvec.hpp:12-38).
 *
 * Reference interfaces each entry point replaces (paths under /root/reference/proj):
 *   sdb_saved_isometry      symdist::saved_isometry      include/symdist/distance.hpp:68
 *                                                         (src/distance.cpp:135-149)
 *   sdb_compute_distance    symdist::compute_distance    include/symdist/distance.hpp:74-75
 *   sdb_run_bz              symdist::run_bz              include/symdist/engine.hpp:60-61
 *                                                         (src/engine.cpp:303-343), singleton
 *                                                         packages (information_sets / singleton_gamma)
 *   sdb_lower_bound         symdist::lower_bound         include/symdist/engine.hpp:47
 *   sdb_validate_normalizer symdist::validate_normalizer include/symdist/distance.hpp:57
 *   sdb_isometry_transform  symdist::isometry_transform  include/symdist/prep.hpp:69
 *   sdb_information_sets    symdist::information_sets    include/symdist/prep.hpp:75
 *   sdb_saved_1_gamma       symdist::saved_1_gamma       include/symdist/distance.hpp:60
 *                                                         (src/distance.cpp:95-113)
 *   sdb_saved_2_gamma       symdist::saved_2_gamma       include/symdist/distance.hpp:64
 *                                                         (src/distance.cpp:115-133)
 *   sdb_run_bz_packaged     symdist::run_bz              include/symdist/engine.hpp:60-61
 *                                                         with 1/3-packages (prep.hpp:13-35)
 *   sdb_prepare_packages    symdist::diagonalize_f2 / diagonalize_f4 + second_gamma
 *                                                         include/symdist/prep.hpp:48-64
 *   sdb_saved_isometry_batch  (no reference counterpart: a loop of saved_isometry
 *                              calls, one code per CTA on the GPU; BASELINE config 3)
 *   sdb_generate_code       (BASELINE.md §2 seeded config generator)
 *   sdb_random_stabilizer   symdist::random_stabilizer   include/symdist/distance.hpp:80
 *   sdb_parse_matrix_text   symdist::parse_matrix_text   include/symdist/matrix_io.hpp:13-14
 *   sdb_format_matrix       symdist::format_matrix       include/symdist/matrix_io.hpp:18
 *   sdb_comm_*              NCCL communicator for the per-level min-allreduce (multi-GPU;
 *                           the reference's in-process CAS-min, engine.cpp:178-181, across GPUs)
 *   sdb_plan_*              device-resident split of sdb_saved_isometry: prep + H2D once,
 *                           then the level loop from HBM (used to time the kernel path alone)
 *
 * Error mapping (the reference throws; proj/include/symdist/errors.hpp:7-20 and the CLI
 * exit codes proj/tools/symdist_main.cpp:197-209):
 *   SDB_ERR_PARSE            ParseError
 *   SDB_ERR_VALIDATION       ValidationError
 *   SDB_ERR_INTERNAL         InternalError
 *   SDB_ERR_DEVICE           CUDA / NCCL failure (no reference counterpart)
 *   SDB_ERR_INVALID_ARGUMENT std::invalid_argument
 * sdb_last_error() returns the message of the calling thread's last failure.
 */
#ifndef SYMDIST_B200_H
#define SYMDIST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDB_ABI_VERSION 2

typedef enum {
    SDB_OK = 0,
    SDB_ERR_PARSE = 1,
    SDB_ERR_VALIDATION = 2,
    SDB_ERR_INTERNAL = 3,
    SDB_ERR_DEVICE = 4,
    SDB_ERR_INVALID_ARGUMENT = 5
} sdb_status;

/* Algorithm ids follow symdist::Algorithm's declaration order (distance.hpp:23-29). */
typedef enum {
    SDB_ALG_AUTO = 0,
    SDB_ALG_SAVED_1_GAMMA = 1,
    SDB_ALG_SAVED_2_GAMMA = 2,
    SDB_ALG_SAVED_ISOMETRY = 3,
    SDB_ALG_BRUTE_FORCE = 4
} sdb_algorithm;

/* symdist::WeightMode (prep.hpp:11) */
typedef enum { SDB_MODE_SYMPLECTIC = 0, SDB_MODE_HAMMING = 1 } sdb_weight_mode;

/* symdist::BoundsTraceEntry (engine.hpp:35-39) */
typedef struct {
    int g;
    long long lower;
    long long upper;
} sdb_trace_entry;

/* Per-level exchange for multi-GPU sharding: elementwise min of `count` uint64 values
 * across all ranks, in place. Return 0 on success. Called once or twice per level with
 * count = 1. NULL when world == 1. */
typedef int (*sdb_allreduce_min_fn)(void *ctx, uint64_t *values, int count);

/* symdist::RunOptions (distance.hpp:33-37) plus device / sharding fields. */
typedef struct {
    int workers;            /* recorded in the report like the reference; the GPU path ignores it */
    int validate;           /* run validate_normalizer first (default 1) */
    int dual_filter;        /* C_perp \ C admissibility filter (default 1) */
    int device;             /* CUDA device ordinal for this process */
    int max_generation;     /* 0: run to termination. >0: stop after that level (partial trace,
                               report.complete = 0); used for config 5 parity at g <= 8 */
    int rank;               /* this process's shard of every level's rank space */
    int world;              /* number of shards (GPUs); 1 = single GPU */
    sdb_allreduce_min_fn allreduce_min;
    void *allreduce_ctx;
    int kernel;             /* 0 auto, 1 force the lexicographic-walk kernel (batch: row-major device
                               prep and every level on the per-thread walk, no meet-in-the-middle
                               lists), 2 force the POPC head x tail tile kernel, 3 batch only: run
                               the prep (validation, information sets) on the host, 4 force the
                               tensor-core tile kernel on every level g >= 2 (auto uses it on
                               levels of >= 2^24 candidates) */
    void *stream;           /* cudaStream_t to run on (NULL: a private non-blocking stream) */
    void *comm;             /* sdb_comm_create handle (NCCL): with world > 1 the level exchange is a
                               stream-ordered min-allreduce, no host round trip (else allreduce_min) */
    long long shard_min;    /* levels with fewer candidates run whole on every rank, no exchange
                               (0: default 2^26; 1: shard every level) */
    int reserved[4];
} sdb_run_options;

/* symdist::DistanceReport (distance.hpp:44-52) plus GPU-side measurements. */
typedef struct {
    int distance;
    int algorithm;                       /* sdb_algorithm */
    int generations;
    unsigned long long candidates_enumerated; /* level-complete count, = reference */
    double elapsed_seconds;              /* normalizer in host memory -> report */
    int workers;
    int trace_len;
    /* extras */
    int complete;                        /* terminated by L >= U or exhaustion */
    long long upper;                     /* final U in the engine's units (Hamming on isometry) */
    unsigned long long candidates_visited; /* what the kernels enumerated (this rank) */
    double prep_seconds;                 /* validation + isometry + information sets + H2D */
    double enum_seconds;                 /* sum of per-level device time (CUDA events) */
    int n_gammas;
    int kernel_launches;                 /* CUDA kernels launched by this call */
    int best_generation;                 /* level of the first minimal candidate (-1: none) */
    int best_gamma;                      /* its Gamma index */
    unsigned long long best_rank;        /* its lexicographic rank inside that level/Gamma */
    unsigned long long h2d_bytes;        /* host->device bytes this call moved */
    unsigned long long d2h_bytes;        /* device->host bytes this call moved */
    int last_level_kernel;               /* kernel of the last level run: 1 walk, 2 POPC tile,
                                            3 tensor-core tile, 4 package walk, 5 package tile */
    int reserved;
    unsigned long long candidates_skipped; /* left out by the mid-level early exit: once a level's
                                              minimum reaches L(g-1) it is the distance, and
                                              work whose keys all exceed the best key cannot
                                              change trace or best; visited + skipped =
                                              enumerated on a single rank */
} sdb_report;

void sdb_default_options(sdb_run_options *opts);
const char *sdb_last_error(void);
int sdb_abi_version(void);
/* 1 if a CUDA device is usable, else 0 (message in sdb_last_error). */
int sdb_device_available(void);

/* ---- distance API ---------------------------------------------------------------- */

/* Saved_isometry on an (n+k) x 2n normalizer. trace receives up to trace_cap entries
 * (report.trace_len is the full length). best_out, when non-NULL, receives the best
 * codeword in the Gamma frame (3n columns, ceil(3n/64) words), like BoundsState::best. */
sdb_status sdb_saved_isometry(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                              const sdb_run_options *opts, sdb_report *report,
                              sdb_trace_entry *trace, int trace_cap, uint64_t *best_out);

/* Saved_1_Gamma / Saved_2_Gamma: the package routes, symplectic units (distance = U). best_out
 * (2n columns, ceil(2n/64) words) is in the prepared frame (Saved_1_Gamma permutes pairs). */
sdb_status sdb_saved_1_gamma(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                             const sdb_run_options *opts, sdb_report *report,
                             sdb_trace_entry *trace, int trace_cap, uint64_t *best_out);
sdb_status sdb_saved_2_gamma(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                             const sdb_run_options *opts, sdb_report *report,
                             sdb_trace_entry *trace, int trace_cap, uint64_t *best_out);

/* compute_distance dispatch (distance.cpp:226-240): AUTO runs Saved_2_Gamma when k <= 2 and
 * the isometry route otherwise; SDB_ALG_BRUTE_FORCE is the Gray-code walk over all 2^(n+k)
 * combinations on the device (brute_force_distance, distance.cpp:151-224; n + k <= 28 like
 * the reference, SDB_ERR_INVALID_ARGUMENT beyond). */
sdb_status sdb_compute_distance(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                                int algorithm, const sdb_run_options *opts, sdb_report *report,
                                sdb_trace_entry *trace, int trace_cap);

/* One code per CTA: n_codes normalizers of identical shape, packed back to back
 * (code c at rows + c*n_rows*row_words). distances[c] is the code's distance or -1 with
 * statuses[c] != 0 on a per-code error; traces: n_codes x trace_cap entries. */
sdb_status sdb_saved_isometry_batch(const uint64_t *rows, int n_codes, int n_rows, int n_cols,
                                    int row_words, const sdb_run_options *opts, int *distances,
                                    int *statuses, int *generations, sdb_trace_entry *traces,
                                    int *trace_lens, int trace_cap, double *elapsed_seconds,
                                    double *device_seconds);

/* ---- engine API ------------------------------------------------------------------- */

/* run_bz over n_gammas singleton-package matrices sharing one frame (n_rows x n_cols
 * each, packed back to back). mode: SDB_MODE_*. pair_count: n (symplectic: n_cols/2;
 * hamming: n_cols/3 when divisible else 0). rank_deficits: per matrix (hamming lower
 * bound). filter_rows (may be NULL when filter_enabled == 0): filter_n_rows x 2n in the
 * same frame as the first 2n columns, with AdmissibilityFilter::for_rows(rows, k)
 * semantics (enabled iff filter_enabled && filter_k >= 1). */
sdb_status sdb_run_bz(const uint64_t *gammas, int n_gammas, int n_rows, int n_cols, int row_words,
                      int mode, int pair_count, const int *rank_deficits,
                      const uint64_t *filter_rows, int filter_n_rows, int filter_n_cols,
                      int filter_row_words, int filter_enabled, int filter_k,
                      const sdb_run_options *opts, sdb_report *report, sdb_trace_entry *trace,
                      int trace_cap, uint64_t *best_out);

/* run_bz over packaged matrices (1 or 3 rows per package; reference PackagedGamma). Matrix j
 * has gamma_rows[j] <= max_rows rows at gammas + j*max_rows*row_words. packages: for each
 * matrix in turn, n_packages[j] entries of [size, row_0, .., row_{size-1}]. n_pp (may be
 * NULL: all packages principal) feeds the two-matrix lower bound. */
sdb_status sdb_run_bz_packaged(const uint64_t *gammas, int n_gammas, const int *gamma_rows, int max_rows,
                               int n_cols, int row_words, int mode, int pair_count,
                               const int *rank_deficits, const int *n_packages, const int *n_pp,
                               const int *packages, const uint64_t *filter_rows, int filter_n_rows,
                               int filter_n_cols, int filter_row_words, int filter_enabled, int filter_k,
                               const sdb_run_options *opts, sdb_report *report, sdb_trace_entry *trace,
                               int trace_cap, uint64_t *best_out);

/* symdist::BoundsState's per-generation fields (engine.hpp:33-40). */
typedef struct {
    long long upper;                          /* in/out; 0 = unset: the sentinel first */
    unsigned long long candidates_enumerated; /* in/out: += the generation's candidate count */
    int improved;                             /* out: 1 when a candidate lowered upper */
} sdb_bounds_state;

/* enumerate_generation(gamma, g, state, filter, workers) (engine.hpp:53-54,
 * engine.cpp:296-301): every g-combination of ONE matrix (one member row per package; n_packages
 * = 0 means one package per row, else packages encoded as in sdb_run_bz_packaged) folded into
 * *state. Candidates below state->upper must pass the filter; the first minimal one (reference
 * visiting order) is written to best_out (row_words words, Gamma frame) when it improved upper.
 * Errors as the reference: g outside [1, n_p] or a filter frame other than 2n columns is
 * SDB_ERR_INVALID_ARGUMENT. The whole generation runs on opts->device (no sharding). */
sdb_status sdb_enumerate_generation(const uint64_t *gamma, int n_rows, int n_cols, int row_words, int mode,
                                    int pair_count, int n_packages, const int *packages, int g,
                                    const uint64_t *filter_rows, int filter_n_rows, int filter_n_cols,
                                    int filter_row_words, int filter_enabled, int filter_k,
                                    const sdb_run_options *opts, sdb_bounds_state *state, uint64_t *best_out);

/* lower_bound(g, gammas) for singleton Hamming / symplectic matrices. */
sdb_status sdb_lower_bound(int g, int mode, int n_gammas, const int *rank_deficits,
                           const int *n_packages, const int *n_pp, long long *out);

/* ---- host prep (no device needed) ------------------------------------------------- */

/* ok = 1 when valid, else 0 with the reference's message in msg. */
sdb_status sdb_validate_normalizer(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                                   int *ok, char *msg, int msg_len);
sdb_status sdb_isometry_transform(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                                  uint64_t *out, int out_row_words);
/* Up to max_gammas matrices (n_rows x n_cols each, out_row_words stride) into out;
 * deficits[j]; pivots[j*n_rows + i] (-1 for rows without a pivot). */
sdb_status sdb_information_sets(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                                int max_gammas, uint64_t *out, int out_row_words, int *deficits,
                                int *pivots, int *n_gammas);
/* The package routes' prepared matrices (algorithm SDB_ALG_SAVED_1_GAMMA: diagonalize_f2;
 * SDB_ALG_SAVED_2_GAMMA: diagonalize_f4 then second_gamma). Matrix j (gamma_rows[j] rows of
 * n_cols) at out + j*max_rows*out_row_words; packages encoded as in sdb_run_bz_packaged. */
sdb_status sdb_prepare_packages(const uint64_t *rows, int n_rows, int n_cols, int row_words, int algorithm,
                                int max_gammas, int max_rows, uint64_t *out, int out_row_words,
                                int *gamma_rows, int *n_packages, int *n_pp, int *packages,
                                int packages_cap, int *n_gammas);

/* Tensor-core tile kernel encoding (device.hpp TcPlan, csrc/tcenc.cpp), host only: runs the
 * isometry prep of an (n+k) x 2n normalizer (validation off) when isometry != 0 — else the
 * matrix itself (2n columns) is the one symplectic-mode Gamma — builds the per-Gamma ±1
 * coordinates, and checks S * popc(x|z) = C0 + c_h + sum head_k tail_k on `trials` random
 * head/tail splits per Gamma. *mismatches = failed checks (-1: the code needs more than 128
 * coordinates, no tensor-core path); k_per_gamma (may be NULL) receives up to max_gammas
 * coordinate counts, *n_gammas the matrix count. */
sdb_status sdb_tc_encoding_check(const uint64_t *rows, int n_rows, int n_cols, int row_words, int isometry,
                                 uint64_t seed, int trials, int *mismatches, int *k_per_gamma,
                                 int max_gammas, int *n_gammas);

/* BASELINE.md §2 generator: (n+k) x 2n normalizer from seed (xorshift64*), transvections
 * <= 0 means 4n. */
sdb_status sdb_generate_code(int n, int k, uint64_t seed, int transvections, uint64_t *out,
                             int out_row_words);

/* random_stabilizer (distance.cpp:242-294): the reference's mt19937_64 instance generator,
 * same draws; (n+k) x 2n into out. */
sdb_status sdb_random_stabilizer(int n, int k, uint64_t seed, uint64_t *out, int out_row_words);

/* Matrix text format (matrix_io.cpp:26-106, matrix_io.hpp:13-18): "K N" header then K rows of
 * N '0'/'1' characters. Parse failures return SDB_ERR_PARSE with the reference's
 * "origin:line: what" message. out may be NULL to query the shape. format_matrix writes the
 * inverse text (NUL-terminated) when buf is non-NULL; *len = its length. */
sdb_status sdb_parse_matrix_text(const char *text, const char *origin, uint64_t *out, int out_row_words,
                                 int max_rows, int *n_rows, int *n_cols);
sdb_status sdb_format_matrix(const uint64_t *rows, int n_rows, int n_cols, int row_words, char *buf, int cap,
                             int *len);

/* ---- multi-GPU: NCCL communicator for the per-level exchange ------------------------ */
/* Rank 0 makes the id and shares it out of band (bench.py: torch.distributed broadcast);
 * every rank then creates its communicator on its device. */
sdb_status sdb_comm_unique_id(unsigned char id[128]);
sdb_status sdb_comm_create(const unsigned char id[128], int rank, int world, int device, void **comm);
void sdb_comm_destroy(void *comm);
/* Synchronous elementwise min of count host uint64 values across the communicator (the
 * plumbing of the per-level exchange; usable as an sdb_allreduce_min_fn body). */
sdb_status sdb_comm_allreduce_min(void *comm, uint64_t *values, int count, int device);

/* ---- device-resident plan (prep + H2D once, levels from HBM) ---------------------- */
typedef struct sdb_plan sdb_plan;
sdb_status sdb_plan_create(const uint64_t *rows, int n_rows, int n_cols, int row_words,
                           const sdb_run_options *opts, sdb_plan **out);
sdb_status sdb_plan_run(sdb_plan *plan, sdb_report *report, sdb_trace_entry *trace,
                        int trace_cap, double *level_seconds);
void sdb_plan_destroy(sdb_plan *plan);

#ifdef __cplusplus
}
#endif

#endif /* SYMDIST_B200_H */
