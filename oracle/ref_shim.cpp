// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/src/*.cpp,
// compiled in place by oracle/Makefile into oracle/_ref/). It lets the Python tests,
// the golden-vector generator (tests/golden/make_golden.py) and bench.py's CPU arm call
// the reference's own public API:
//   symdist::saved_isometry / compute_distance   proj/include/symdist/distance.hpp:68,74
//   symdist::information_sets / isometry_transform proj/include/symdist/prep.hpp:69,75
//   symdist::run_bz / enumerate_generation / lower_bound proj/include/symdist/engine.hpp:47-61
//   symdist::random_stabilizer / brute_force_distance / validate_normalizer
// Matrices cross this boundary as row-major 0/1 bytes (rows x cols).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "symdist/distance.hpp"
#include "symdist/engine.hpp"
#include "symdist/errors.hpp"
#include "symdist/gf4.hpp"
#include "symdist/prep.hpp"

using namespace symdist;

extern "C" {
typedef struct {
    int g;
    long lower;
    long upper;
} ref_trace_entry;

typedef struct {
    int distance;
    int algorithm;
    int generations;
    unsigned long long candidates;
    double elapsed_seconds;
    int workers;
    int trace_len;
} ref_report;
}

namespace {

BitMatrix from_bytes(const uint8_t* bits, int rows, int cols) {
    BitMatrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
            if (bits[static_cast<std::size_t>(r) * cols + c]) m.set(r, c, true);
    return m;
}

void to_bytes(const BitMatrix& m, uint8_t* out) {
    for (std::size_t r = 0; r < m.n_rows(); ++r)
        for (std::size_t c = 0; c < m.n_cols(); ++c) out[r * m.n_cols() + c] = m.get(r, c) ? 1 : 0;
}

void set_err(char* err, int errlen, const char* what) {
    if (err && errlen > 0) {
        std::snprintf(err, static_cast<std::size_t>(errlen), "%s", what);
    }
}

// 0 ok, 1 parse, 2 validation, 3 internal, 5 invalid_argument, 6 other.
template <class F>
int guarded(char* err, int errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const ParseError& e) {
        set_err(err, errlen, e.what());
        return 1;
    } catch (const ValidationError& e) {
        set_err(err, errlen, e.what());
        return 2;
    } catch (const InternalError& e) {
        set_err(err, errlen, e.what());
        return 3;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return 5;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 6;
    }
}

void fill_report(const DistanceReport& rep, ref_report* out, ref_trace_entry* trace, int cap) {
    out->distance = rep.distance;
    out->algorithm = static_cast<int>(rep.algorithm);
    out->generations = rep.generations;
    out->candidates = rep.candidates_enumerated;
    out->elapsed_seconds = rep.elapsed_seconds;
    out->workers = rep.workers;
    out->trace_len = static_cast<int>(rep.bounds_trace.size());
    for (int i = 0; i < out->trace_len && i < cap; ++i) {
        trace[i].g = rep.bounds_trace[static_cast<std::size_t>(i)].g;
        trace[i].lower = rep.bounds_trace[static_cast<std::size_t>(i)].lower;
        trace[i].upper = rep.bounds_trace[static_cast<std::size_t>(i)].upper;
    }
}

}  // namespace

extern "C" {

// alg: 0 auto, 1 saved_1_gamma, 2 saved_2_gamma, 3 saved_isometry, 4 brute_force
int ref_compute_distance(const uint8_t* bits, int rows, int cols, int alg, int workers, int validate,
                         int dual_filter, ref_report* rep, ref_trace_entry* trace, int trace_cap,
                         char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const StabilizerInstance inst = StabilizerInstance::from_matrix(from_bytes(bits, rows, cols));
        RunOptions opts;
        opts.workers = workers;
        opts.validate = validate != 0;
        opts.dual_filter = dual_filter != 0;
        fill_report(compute_distance(inst, static_cast<Algorithm>(alg), opts), rep, trace, trace_cap);
    });
}

int ref_validate(const uint8_t* bits, int rows, int cols, int* ok, char* msg, int msglen) {
    return guarded(msg, msglen, [&] {
        const StabilizerInstance inst = StabilizerInstance::from_matrix(from_bytes(bits, rows, cols));
        const ValidationResult res = validate_normalizer(inst);
        *ok = res.ok ? 1 : 0;
        set_err(msg, msglen, res.message.c_str());
    });
}

int ref_random_stabilizer(int n, int k, unsigned long long seed, uint8_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] { to_bytes(random_stabilizer(n, k, seed).a, out); });
}

int ref_isometry_transform(const uint8_t* bits, int rows, int cols, uint8_t* out, char* err, int errlen) {
    return guarded(err, errlen, [&] { to_bytes(isometry_transform(from_bytes(bits, rows, cols)), out); });
}

// Gammas of the isometry route: out holds max_gammas blocks of rows x out_cols bytes.
int ref_information_sets(const uint8_t* bits, int rows, int cols, int max_gammas, uint8_t* out,
                         int* deficits, int* pivots, int* n_gammas, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const std::vector<PackagedGamma> gs = information_sets(from_bytes(bits, rows, cols));
        *n_gammas = static_cast<int>(gs.size());
        for (int j = 0; j < static_cast<int>(gs.size()) && j < max_gammas; ++j) {
            const PackagedGamma& g = gs[static_cast<std::size_t>(j)];
            to_bytes(g.matrix, out + static_cast<std::size_t>(j) * rows * cols);
            deficits[j] = g.rank_deficit;
            for (int p = 0; p < g.n_p(); ++p) pivots[j * rows + p] = g.packages[static_cast<std::size_t>(p)].pivot;
        }
    });
}

// saved_isometry's prep followed by run_bz's generation loop, stopped after g_max
// (g_max <= 0: no cap, identical to run_bz). Per-level wall time and candidate counts are
// recorded around the reference's own enumerate_generation calls.
int ref_isometry_levels(const uint8_t* bits, int rows, int cols, int workers, int validate,
                        int dual_filter, int g_max, ref_trace_entry* trace, double* level_seconds,
                        unsigned long long* level_candidates, int trace_cap, int* n_levels,
                        long* upper_out, double* prep_seconds, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        using Clock = std::chrono::steady_clock;
        const auto t0 = Clock::now();
        const StabilizerInstance inst = StabilizerInstance::from_matrix(from_bytes(bits, rows, cols));
        if (validate) {
            const ValidationResult res = validate_normalizer(inst);
            if (!res.ok) throw ValidationError(res.message);
        }
        const BitMatrix image = isometry_transform(inst.a);
        const std::vector<PackagedGamma> gammas = information_sets(image);
        const AdmissibilityFilter filter = dual_filter ? AdmissibilityFilter::for_rows(inst.a, inst.k)
                                                       : AdmissibilityFilter::disabled();
        *prep_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
        BoundsState state;
        state.upper = static_cast<long>(gammas[0].matrix.n_cols()) + 1;
        state.lower = 1;
        int g_limit = gammas[0].n_p();
        for (const PackagedGamma& gm : gammas) g_limit = std::min(g_limit, gm.n_p());
        if (g_max > 0) g_limit = std::min(g_limit, g_max);
        *n_levels = 0;
        for (int g = 1; g <= g_limit; ++g) {
            const auto tl = Clock::now();
            const std::uint64_t before = state.candidates_enumerated;
            for (const PackagedGamma& gm : gammas) enumerate_generation(gm, g, state, filter, workers);
            const double secs = std::chrono::duration<double>(Clock::now() - tl).count();
            state.generation = g;
            state.lower = lower_bound(g, gammas);
            if (*n_levels < trace_cap) {
                trace[*n_levels].g = g;
                trace[*n_levels].lower = state.lower;
                trace[*n_levels].upper = state.upper;
                level_seconds[*n_levels] = secs;
                level_candidates[*n_levels] = state.candidates_enumerated - before;
            }
            ++*n_levels;
            if (state.lower >= state.upper) break;
        }
        *upper_out = state.upper;
    });
}

// run_bz on one singleton_gamma view (mode 0 symplectic, 1 hamming) with an optional filter
// (filter_rows == 0: disabled). best receives the best codeword's bits (length best_cap).
int ref_run_bz_singleton(const uint8_t* bits, int rows, int cols, int mode, const uint8_t* filter_bits,
                         int filter_rows, int filter_cols, int filter_k, int workers,
                         ref_trace_entry* trace, int trace_cap, int* trace_len, long* upper,
                         int* generation, unsigned long long* candidates, uint8_t* best, int best_cap,
                         int* best_len, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const PackagedGamma gamma = singleton_gamma(from_bytes(bits, rows, cols),
                                                    mode ? WeightMode::hamming : WeightMode::symplectic);
        const AdmissibilityFilter filter =
            filter_rows > 0 ? AdmissibilityFilter::for_rows(from_bytes(filter_bits, filter_rows, filter_cols), filter_k)
                            : AdmissibilityFilter::disabled();
        const BoundsState st = run_bz({gamma}, filter, workers);
        *trace_len = static_cast<int>(st.trace.size());
        for (int i = 0; i < *trace_len && i < trace_cap; ++i) {
            trace[i].g = st.trace[static_cast<std::size_t>(i)].g;
            trace[i].lower = st.trace[static_cast<std::size_t>(i)].lower;
            trace[i].upper = st.trace[static_cast<std::size_t>(i)].upper;
        }
        *upper = st.upper;
        *generation = st.generation;
        *candidates = st.candidates_enumerated;
        *best_len = static_cast<int>(st.best.size());
        for (int i = 0; i < *best_len && i < best_cap; ++i) best[i] = st.best.get(static_cast<std::size_t>(i)) ? 1 : 0;
    });
}

// saved_isometry with best codeword: the reference's run_bz on information_sets(image).
int ref_isometry_best(const uint8_t* bits, int rows, int cols, int workers, uint8_t* best, int best_cap,
                      int* best_len, long* upper, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const StabilizerInstance inst = StabilizerInstance::from_matrix(from_bytes(bits, rows, cols));
        const std::vector<PackagedGamma> gammas = information_sets(isometry_transform(inst.a));
        const BoundsState st = run_bz(gammas, AdmissibilityFilter::for_rows(inst.a, inst.k), workers);
        *upper = st.upper;
        *best_len = static_cast<int>(st.best.size());
        for (int i = 0; i < *best_len && i < best_cap; ++i) best[i] = st.best.get(static_cast<std::size_t>(i)) ? 1 : 0;
    });
}

// The package routes' prep (alg 1: diagonalize_f2; 2: diagonalize_f4 + second_gamma): matrix j
// as gamma_rows[j] x cols bytes at out + j*max_rows*cols; packages encoded per matrix as
// [size, row...] runs (n_packages[j] of them).
int ref_prepare_packages(const uint8_t* bits, int rows, int cols, int alg, int max_rows, uint8_t* out,
                         int* gamma_rows, int* n_packages, int* n_pp, int* packages, int packages_cap,
                         int* n_gammas, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const BitMatrix a = from_bytes(bits, rows, cols);
        std::vector<PackagedGamma> gs;
        if (alg == 1) {
            gs.push_back(diagonalize_f2(a));
        } else {
            auto [b, pc] = diagonalize_f4(to_gf4(a));
            PackagedGamma d = second_gamma(to_gf4(b.matrix), pc);
            gs.push_back(std::move(b));
            gs.push_back(std::move(d));
        }
        *n_gammas = static_cast<int>(gs.size());
        int used = 0;
        for (int j = 0; j < *n_gammas; ++j) {
            const PackagedGamma& g = gs[static_cast<std::size_t>(j)];
            if (static_cast<int>(g.matrix.n_rows()) > max_rows) throw std::invalid_argument("max_rows too small");
            to_bytes(g.matrix, out + static_cast<std::size_t>(j) * max_rows * cols);
            gamma_rows[j] = static_cast<int>(g.matrix.n_rows());
            n_packages[j] = g.n_p();
            n_pp[j] = g.n_pp;
            for (const Package& pk : g.packages) {
                if (used + 1 + static_cast<int>(pk.rows.size()) > packages_cap)
                    throw std::invalid_argument("packages_cap too small");
                packages[used++] = static_cast<int>(pk.rows.size());
                for (int r : pk.rows) packages[used++] = r;
            }
        }
    });
}

// saved_1_gamma / saved_2_gamma run through the reference's own prep and run_bz, returning the
// bound state's best codeword (the single-worker BoundsState::best) and U.
int ref_package_best(const uint8_t* bits, int rows, int cols, int alg, int workers, uint8_t* best,
                     int best_cap, int* best_len, long* upper, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        const StabilizerInstance inst = StabilizerInstance::from_matrix(from_bytes(bits, rows, cols));
        std::vector<PackagedGamma> gs;
        BitMatrix frame(0, inst.a.n_cols());
        if (alg == 1) {
            PackagedGamma g = diagonalize_f2(inst.a);
            for (std::size_t r = 0; r < inst.a.n_rows(); ++r) frame.append_row(g.matrix.row(r));
            gs.push_back(std::move(g));
        } else {
            auto [b, pc] = diagonalize_f4(to_gf4(inst.a));
            PackagedGamma d = second_gamma(to_gf4(b.matrix), pc);
            gs.push_back(std::move(b));
            gs.push_back(std::move(d));
            frame = inst.a;
        }
        const BoundsState st = run_bz(gs, AdmissibilityFilter::for_rows(std::move(frame), inst.k), workers);
        *upper = st.upper;
        *best_len = static_cast<int>(st.best.size());
        for (int i = 0; i < *best_len && i < best_cap; ++i) best[i] = st.best.get(static_cast<std::size_t>(i)) ? 1 : 0;
    });
}

// enumerate_generation (engine.hpp:53-54) on one matrix: singleton_gamma(bits, mode) or, with
// n_packages > 0, packages encoded as [size, row...] runs; filter rows (filter_rows == 0:
// disabled); the bound state enters with upper_io (0 = unset) and no best.
int ref_enumerate_generation(const uint8_t* bits, int rows, int cols, int mode, int n_packages, const int* packages,
                             int g, const uint8_t* filter_bits, int filter_rows, int filter_cols, int filter_k,
                             int workers, long* upper_io, unsigned long long* candidates, uint8_t* best, int best_cap,
                             int* best_len, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        PackagedGamma gamma = singleton_gamma(from_bytes(bits, rows, cols),
                                              mode ? WeightMode::hamming : WeightMode::symplectic);
        if (n_packages > 0) {
            gamma.packages.clear();
            for (int q = 0, pos = 0; q < n_packages; ++q) {
                Package pk;
                const int sz = packages[pos++];
                for (int i = 0; i < sz; ++i) pk.rows.push_back(packages[pos++]);
                gamma.packages.push_back(std::move(pk));
            }
        }
        const AdmissibilityFilter filter =
            filter_rows > 0 ? AdmissibilityFilter::for_rows(from_bytes(filter_bits, filter_rows, filter_cols), filter_k)
                            : AdmissibilityFilter::disabled();
        BoundsState st;
        st.upper = *upper_io;
        enumerate_generation(gamma, g, st, filter, workers);
        *upper_io = st.upper;
        *candidates = st.candidates_enumerated;
        *best_len = static_cast<int>(st.best.size());
        for (int i = 0; i < *best_len && i < best_cap; ++i) best[i] = st.best.get(static_cast<std::size_t>(i)) ? 1 : 0;
    });
}

}  // extern "C"
