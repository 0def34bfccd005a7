// extern "C" boundary (include/symdist_b200.h). Every entry point catches and maps
// exceptions to sdb_status; the message is kept per thread for sdb_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/symdist_b200.h"
#include "comm.hpp"
#include "engine.hpp"
#include "tcenc.hpp"
#include "errors.hpp"
#include "gf2.hpp"
#include "packages.hpp"

namespace {

thread_local std::string g_last_error;

template <class F>
sdb_status guarded(F &&f) {
    try {
        f();
        g_last_error.clear();
        return SDB_OK;
    } catch (const sdb::ParseFailure &e) {
        g_last_error = e.what();
        return SDB_ERR_PARSE;
    } catch (const sdb::ValidationFailure &e) {
        g_last_error = e.what();
        return SDB_ERR_VALIDATION;
    } catch (const sdb::InternalFailure &e) {
        g_last_error = e.what();
        return SDB_ERR_INTERNAL;
    } catch (const sdb::DeviceFailure &e) {
        g_last_error = e.what();
        return SDB_ERR_DEVICE;
    } catch (const std::invalid_argument &e) {
        g_last_error = e.what();
        return SDB_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc &) {
        g_last_error = "host allocation failed";
        return SDB_ERR_INTERNAL;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return SDB_ERR_INTERNAL;
    }
}

void check_matrix_args(const uint64_t *rows, int n_rows, int n_cols, int row_words) {
    if (n_rows < 0 || n_cols < 0) throw sdb::InvalidArgument("negative matrix shape");
    if (n_rows > 0 && !rows) throw sdb::InvalidArgument("null matrix pointer");
    if (row_words < (n_cols + 63) / 64) throw sdb::InvalidArgument("row_words smaller than ceil(n_cols/64)");
}

sdb_run_options opts_or_default(const sdb_run_options *o) {
    sdb_run_options d;
    sdb_default_options(&d);
    return o ? *o : d;
}

void zero_report(sdb_report *r) {
    std::memset(r, 0, sizeof *r);
    r->best_generation = -1;
    r->best_gamma = -1;
}

// saved_isometry (distance.cpp:135-149): validate -> isometry -> information_sets ->
// filter from the original rows -> run_bz -> U/2
void saved_isometry_impl(const uint64_t *rows, int n_rows, int n_cols, int row_words, const sdb_run_options &o,
                         sdb_report *rep, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out) {
    const auto t0 = std::chrono::steady_clock::now();
    check_matrix_args(rows, n_rows, n_cols, row_words);
    if (n_cols == 0 || n_cols % 2 != 0)
        throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
    zero_report(rep);
    const sdb::BitMat a = sdb::BitMat::from_words(rows, n_rows, n_cols, row_words);
    const int n = n_cols / 2, k = n_rows - n;
    if (o.validate) {
        const sdb::Validation v = sdb::validate_normalizer(a);
        if (!v.ok) throw sdb::ValidationFailure(v.message);
    }
    std::vector<sdb::InfoSet> is = sdb::information_sets(sdb::isometry_transform(a));
    std::vector<sdb::GammaIn> gammas;
    for (sdb::InfoSet &s : is) gammas.push_back(sdb::GammaIn{std::move(s.matrix), s.rank_deficit});
    sdb::Filter f;
    f.enabled = o.dual_filter && k >= 1;
    if (f.enabled) f.rows = a;
    const auto tp = std::chrono::steady_clock::now();
    sdb::Plan plan(std::move(gammas), sdb::Mode::hamming, n, f, o);
    const auto tq = std::chrono::steady_clock::now();
    rep->h2d_bytes = plan.upload_bytes;
    plan.run(rep, trace, trace_cap, best_out, nullptr);
    rep->prep_seconds = std::chrono::duration<double>(tp - t0).count() + plan.h2d_seconds;
    if (std::getenv("SDB_TRACE_HOST"))
        std::fprintf(stderr, "[sdb] prep %.3f ms, plan %.3f ms, run %.3f ms (levels %.3f ms)\n",
                     1e3 * std::chrono::duration<double>(tp - t0).count(),
                     1e3 * std::chrono::duration<double>(tq - tp).count(),
                     1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - tq).count(),
                     1e3 * rep->enum_seconds);
    if (rep->complete && rep->upper % 2 != 0)
        throw sdb::InternalFailure("saved_isometry: image Hamming distance must be even");
    rep->distance = int(rep->upper / 2);
    rep->algorithm = SDB_ALG_SAVED_ISOMETRY;
    rep->workers = o.workers;
    rep->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

sdb::GammaIn to_gamma_in(sdb::Packaged &&p) {
    sdb::GammaIn g;
    g.matrix = std::move(p.matrix);
    g.rank_deficit = p.rank_deficit;
    g.packages = std::move(p.packages);
    g.n_pp = p.n_pp;
    return g;
}

// The package routes' prep (reference distance.cpp:95-133): Saved_1_Gamma diagonalizes over
// F2 and filters in the permuted frame (the first n+k prepared rows); Saved_2_Gamma runs the
// two F4 diagonalizations and filters in the input frame.
std::vector<sdb::GammaIn> package_gammas(const sdb::BitMat &a, int algorithm, sdb::BitMat *frame) {
    std::vector<sdb::GammaIn> gammas;
    if (algorithm == SDB_ALG_SAVED_1_GAMMA) {
        sdb::Packaged pg = sdb::diagonalize_f2(a);
        *frame = sdb::BitMat(a.rows, pg.matrix.cols);
        for (int r = 0; r < a.rows; r++) std::copy(pg.matrix.row(r), pg.matrix.row(r) + pg.matrix.stride, frame->row(r));
        gammas.push_back(to_gamma_in(std::move(pg)));
    } else {
        auto bp = sdb::diagonalize_f4(sdb::to_gf4(a));
        sdb::Packaged d = sdb::second_gamma(sdb::to_gf4(bp.first.matrix), bp.second);
        gammas.push_back(to_gamma_in(std::move(bp.first)));
        gammas.push_back(to_gamma_in(std::move(d)));
        *frame = a;
    }
    return gammas;
}

// saved_1_gamma / saved_2_gamma (distance.cpp:95-133): validate -> packages -> run_bz in
// symplectic mode -> distance = U
void package_route_impl(int algorithm, const uint64_t *rows, int n_rows, int n_cols, int row_words,
                        const sdb_run_options &o, sdb_report *rep, sdb_trace_entry *trace, int trace_cap,
                        uint64_t *best_out) {
    const auto t0 = std::chrono::steady_clock::now();
    check_matrix_args(rows, n_rows, n_cols, row_words);
    if (n_cols == 0 || n_cols % 2 != 0)
        throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
    zero_report(rep);
    const sdb::BitMat a = sdb::BitMat::from_words(rows, n_rows, n_cols, row_words);
    const int n = n_cols / 2, k = n_rows - n;
    if (o.validate) {
        const sdb::Validation v = sdb::validate_normalizer(a);
        if (!v.ok) throw sdb::ValidationFailure(v.message);
    }
    sdb::BitMat frame;
    std::vector<sdb::GammaIn> gammas = package_gammas(a, algorithm, &frame);
    sdb::Filter f;
    f.enabled = o.dual_filter && k >= 1;
    if (f.enabled) f.rows = std::move(frame);
    const auto tp = std::chrono::steady_clock::now();
    sdb::Plan plan(std::move(gammas), sdb::Mode::symplectic, n, f, o);
    rep->h2d_bytes = plan.upload_bytes;
    plan.run(rep, trace, trace_cap, best_out, nullptr);
    rep->prep_seconds = std::chrono::duration<double>(tp - t0).count() + plan.h2d_seconds;
    rep->distance = int(rep->upper);
    rep->algorithm = algorithm;
    rep->workers = o.workers;
    rep->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// brute_force_distance (distance.cpp:151-224): validate -> Gray walk on the device
void brute_force_impl(const uint64_t *rows, int n_rows, int n_cols, int row_words, const sdb_run_options &o,
                      sdb_report *rep) {
    const auto t0 = std::chrono::steady_clock::now();
    check_matrix_args(rows, n_rows, n_cols, row_words);
    if (n_cols == 0 || n_cols % 2 != 0)
        throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
    zero_report(rep);
    const sdb::BitMat a = sdb::BitMat::from_words(rows, n_rows, n_cols, row_words);
    if (o.validate) {
        const sdb::Validation v = sdb::validate_normalizer(a);
        if (!v.ok) throw sdb::ValidationFailure(v.message);
    }
    double dev = 0;
    rep->distance = sdb::run_brute(a, o, &dev);
    rep->upper = rep->distance;
    rep->algorithm = SDB_ALG_BRUTE_FORCE;
    rep->generations = 0;
    rep->candidates_enumerated = (1ull << n_rows) - 1;
    rep->candidates_visited = rep->candidates_enumerated;
    rep->enum_seconds = dev;
    rep->kernel_launches = 1;
    rep->complete = 1;
    rep->workers = 1;
    rep->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

struct sdb_plan {
    sdb::Plan *plan;
    int n;
    int algorithm;
    sdb_run_options opts;
    double prep_seconds;
};

extern "C" {

void sdb_default_options(sdb_run_options *o) {
    std::memset(o, 0, sizeof *o);
    o->workers = 1;
    o->validate = 1;
    o->dual_filter = 1;
    o->device = 0;
    o->max_generation = 0;
    o->rank = 0;
    o->world = 1;
}

const char *sdb_last_error(void) { return g_last_error.c_str(); }

int sdb_abi_version(void) { return SDB_ABI_VERSION; }

int sdb_device_available(void) {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        g_last_error = e != cudaSuccess ? cudaGetErrorString(e) : "no CUDA device";
        cudaGetLastError();
        return 0;
    }
    return 1;
}

sdb_status sdb_saved_isometry(const uint64_t *rows, int n_rows, int n_cols, int row_words, const sdb_run_options *opts,
                              sdb_report *report, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out) {
    return guarded([&] {
        if (!report) throw sdb::InvalidArgument("null report");
        saved_isometry_impl(rows, n_rows, n_cols, row_words, opts_or_default(opts), report, trace, trace_cap,
                            best_out);
    });
}

sdb_status sdb_saved_1_gamma(const uint64_t *rows, int n_rows, int n_cols, int row_words, const sdb_run_options *opts,
                             sdb_report *report, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out) {
    return guarded([&] {
        if (!report) throw sdb::InvalidArgument("null report");
        package_route_impl(SDB_ALG_SAVED_1_GAMMA, rows, n_rows, n_cols, row_words, opts_or_default(opts), report,
                           trace, trace_cap, best_out);
    });
}

sdb_status sdb_saved_2_gamma(const uint64_t *rows, int n_rows, int n_cols, int row_words, const sdb_run_options *opts,
                             sdb_report *report, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out) {
    return guarded([&] {
        if (!report) throw sdb::InvalidArgument("null report");
        package_route_impl(SDB_ALG_SAVED_2_GAMMA, rows, n_rows, n_cols, row_words, opts_or_default(opts), report,
                           trace, trace_cap, best_out);
    });
}

sdb_status sdb_prepare_packages(const uint64_t *rows, int n_rows, int n_cols, int row_words, int algorithm,
                                int max_gammas, int max_rows, uint64_t *out, int out_row_words, int *gamma_rows,
                                int *n_packages, int *n_pp, int *packages, int packages_cap, int *n_gammas) {
    return guarded([&] {
        check_matrix_args(rows, n_rows, n_cols, row_words);
        if (n_cols == 0 || n_cols % 2 != 0)
            throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
        if (algorithm != SDB_ALG_SAVED_1_GAMMA && algorithm != SDB_ALG_SAVED_2_GAMMA)
            throw sdb::InvalidArgument("prepare_packages: saved_1_gamma or saved_2_gamma");
        if (out_row_words < (n_cols + 63) / 64) throw sdb::InvalidArgument("out_row_words too small");
        const sdb::BitMat a = sdb::BitMat::from_words(rows, n_rows, n_cols, row_words);
        sdb::BitMat frame;
        const std::vector<sdb::GammaIn> gs = package_gammas(a, algorithm, &frame);
        if (n_gammas) *n_gammas = int(gs.size());
        int used = 0;
        for (int j = 0; j < int(gs.size()) && j < max_gammas; j++) {
            const sdb::GammaIn &g = gs[size_t(j)];
            if (g.matrix.rows > max_rows) throw sdb::InvalidArgument("prepare_packages: max_rows too small");
            g.matrix.to_words(out + size_t(j) * max_rows * out_row_words, out_row_words);
            gamma_rows[j] = g.matrix.rows;
            n_packages[j] = int(g.packages.size());
            n_pp[j] = g.n_pp;
            for (const std::vector<int> &pk : g.packages) {
                if (used + 1 + int(pk.size()) > packages_cap) throw sdb::InvalidArgument("packages_cap too small");
                packages[used++] = int(pk.size());
                for (int r : pk) packages[used++] = r;
            }
        }
    });
}

sdb_status sdb_compute_distance(const uint64_t *rows, int n_rows, int n_cols, int row_words, int algorithm,
                                const sdb_run_options *opts, sdb_report *report, sdb_trace_entry *trace,
                                int trace_cap) {
    return guarded([&] {
        if (!report) throw sdb::InvalidArgument("null report");
        const int k = n_rows - n_cols / 2;
        const sdb_run_options o = opts_or_default(opts);
        switch (algorithm) {
            case SDB_ALG_SAVED_ISOMETRY:
                saved_isometry_impl(rows, n_rows, n_cols, row_words, o, report, trace, trace_cap, nullptr);
                return;
            case SDB_ALG_AUTO:
                // distance.cpp:233-237: the two-matrix route when k <= 2, else the isometry
                if (k <= 2) {
                    package_route_impl(SDB_ALG_SAVED_2_GAMMA, rows, n_rows, n_cols, row_words, o, report, trace,
                                       trace_cap, nullptr);
                } else {
                    saved_isometry_impl(rows, n_rows, n_cols, row_words, o, report, trace, trace_cap, nullptr);
                }
                return;
            case SDB_ALG_SAVED_1_GAMMA:
            case SDB_ALG_SAVED_2_GAMMA:
                package_route_impl(algorithm, rows, n_rows, n_cols, row_words, o, report, trace, trace_cap, nullptr);
                return;
            case SDB_ALG_BRUTE_FORCE:
                brute_force_impl(rows, n_rows, n_cols, row_words, o, report);
                return;
            default:
                throw sdb::InvalidArgument("compute_distance: unknown algorithm");
        }
    });
}

sdb_status sdb_saved_isometry_batch(const uint64_t *rows, int n_codes, int n_rows, int n_cols, int row_words,
                                    const sdb_run_options *opts, int *distances, int *statuses, int *generations,
                                    sdb_trace_entry *traces, int *trace_lens, int trace_cap, double *elapsed_seconds,
                                    double *device_seconds) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (n_codes < 0) throw sdb::InvalidArgument("negative code count");
        check_matrix_args(rows, n_rows * std::max(n_codes, 0), n_cols, row_words);
        if (!distances || !statuses || !generations || !trace_lens || (trace_cap > 0 && !traces))
            throw sdb::InvalidArgument("null output array");
        sdb::run_batch(rows, n_codes, n_rows, n_cols, row_words, opts_or_default(opts), distances, statuses,
                       generations, traces, trace_lens, trace_cap, device_seconds);
        if (elapsed_seconds)
            *elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

sdb_status sdb_run_bz(const uint64_t *gammas, int n_gammas, int n_rows, int n_cols, int row_words, int mode,
                      int pair_count, const int *rank_deficits, const uint64_t *filter_rows, int filter_n_rows,
                      int filter_n_cols, int filter_row_words, int filter_enabled, int filter_k,
                      const sdb_run_options *opts, sdb_report *report, sdb_trace_entry *trace, int trace_cap,
                      uint64_t *best_out) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!report) throw sdb::InvalidArgument("null report");
        if (n_gammas <= 0) throw sdb::InvalidArgument("run_bz: need at least one generator matrix");
        check_matrix_args(gammas, n_rows * n_gammas, n_cols, row_words);
        if (mode != SDB_MODE_SYMPLECTIC && mode != SDB_MODE_HAMMING) throw sdb::InvalidArgument("unknown weight mode");
        zero_report(report);
        std::vector<sdb::GammaIn> gs;
        for (int j = 0; j < n_gammas; j++)
            gs.push_back(sdb::GammaIn{sdb::BitMat::from_words(gammas + size_t(j) * n_rows * row_words, n_rows, n_cols,
                                                              row_words),
                                      rank_deficits ? rank_deficits[j] : 0});
        sdb::Filter f;
        f.enabled = filter_enabled && filter_k >= 1;
        if (f.enabled) {
            check_matrix_args(filter_rows, filter_n_rows, filter_n_cols, filter_row_words);
            f.rows = sdb::BitMat::from_words(filter_rows, filter_n_rows, filter_n_cols, filter_row_words);
        }
        const sdb_run_options o = opts_or_default(opts);
        sdb::Plan plan(std::move(gs), mode == SDB_MODE_HAMMING ? sdb::Mode::hamming : sdb::Mode::symplectic,
                       pair_count, f, o);
        plan.run(report, trace, trace_cap, best_out, nullptr);
        report->distance = int(report->upper);
        report->workers = o.workers;
        report->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

sdb_status sdb_run_bz_packaged(const uint64_t *gammas, int n_gammas, const int *gamma_rows, int max_rows, int n_cols,
                               int row_words, int mode, int pair_count, const int *rank_deficits,
                               const int *n_packages, const int *n_pp, const int *packages,
                               const uint64_t *filter_rows, int filter_n_rows, int filter_n_cols,
                               int filter_row_words, int filter_enabled, int filter_k, const sdb_run_options *opts,
                               sdb_report *report, sdb_trace_entry *trace, int trace_cap, uint64_t *best_out) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (!report || !gamma_rows || !n_packages || !packages) throw sdb::InvalidArgument("null argument");
        if (n_gammas <= 0) throw sdb::InvalidArgument("run_bz: need at least one generator matrix");
        if (mode != SDB_MODE_SYMPLECTIC && mode != SDB_MODE_HAMMING) throw sdb::InvalidArgument("unknown weight mode");
        check_matrix_args(gammas, max_rows * n_gammas, n_cols, row_words);
        zero_report(report);
        std::vector<sdb::GammaIn> gs;
        int pos = 0;
        for (int j = 0; j < n_gammas; j++) {
            if (gamma_rows[j] < 0 || gamma_rows[j] > max_rows) throw sdb::InvalidArgument("gamma_rows out of range");
            sdb::GammaIn g;
            g.matrix = sdb::BitMat::from_words(gammas + size_t(j) * max_rows * row_words, gamma_rows[j], n_cols,
                                               row_words);
            g.rank_deficit = rank_deficits ? rank_deficits[j] : 0;
            g.n_pp = n_pp ? n_pp[j] : -1;
            for (int q = 0; q < n_packages[j]; q++) {
                const int sz = packages[pos++];
                if (sz < 1 || sz > 3) throw sdb::InvalidArgument("run_bz: packages hold one to three rows");
                g.packages.emplace_back(packages + pos, packages + pos + sz);
                pos += sz;
            }
            if (g.packages.empty()) throw sdb::InvalidArgument("run_bz: matrix with no packages");
            gs.push_back(std::move(g));
        }
        sdb::Filter f;
        f.enabled = filter_enabled && filter_k >= 1;
        if (f.enabled) {
            check_matrix_args(filter_rows, filter_n_rows, filter_n_cols, filter_row_words);
            f.rows = sdb::BitMat::from_words(filter_rows, filter_n_rows, filter_n_cols, filter_row_words);
        }
        const sdb_run_options o = opts_or_default(opts);
        sdb::Plan plan(std::move(gs), mode == SDB_MODE_HAMMING ? sdb::Mode::hamming : sdb::Mode::symplectic,
                       pair_count, f, o);
        plan.run(report, trace, trace_cap, best_out, nullptr);
        report->distance = int(report->upper);
        report->workers = o.workers;
        report->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

sdb_status sdb_enumerate_generation(const uint64_t *gamma, int n_rows, int n_cols, int row_words, int mode,
                                    int pair_count, int n_packages, const int *packages, int g,
                                    const uint64_t *filter_rows, int filter_n_rows, int filter_n_cols,
                                    int filter_row_words, int filter_enabled, int filter_k,
                                    const sdb_run_options *opts, sdb_bounds_state *state, uint64_t *best_out) {
    return guarded([&] {
        if (!state) throw sdb::InvalidArgument("null bounds state");
        if (mode != SDB_MODE_SYMPLECTIC && mode != SDB_MODE_HAMMING) throw sdb::InvalidArgument("unknown weight mode");
        if (n_packages < 0 || (n_packages > 0 && !packages)) throw sdb::InvalidArgument("null packages");
        check_matrix_args(gamma, n_rows, n_cols, row_words);
        state->improved = 0;
        sdb::GammaIn gm;
        gm.matrix = sdb::BitMat::from_words(gamma, n_rows, n_cols, row_words);
        for (int q = 0, pos = 0; q < n_packages; q++) {
            const int sz = packages[pos++];
            if (sz < 1 || sz > 3) throw sdb::InvalidArgument("enumerate_generation: packages hold one to three rows");
            gm.packages.emplace_back(packages + pos, packages + pos + sz);
            pos += sz;
        }
        const int np = n_packages > 0 ? n_packages : n_rows;
        if (g < 1 || g > np) throw sdb::InvalidArgument("enumerate_generation: generation out of range");
        sdb::Filter f;
        f.enabled = filter_enabled && filter_k >= 1;
        if (f.enabled) {
            check_matrix_args(filter_rows, filter_n_rows, filter_n_cols, filter_row_words);
            f.rows = sdb::BitMat::from_words(filter_rows, filter_n_rows, filter_n_cols, filter_row_words);
        }
        sdb_run_options o = opts_or_default(opts);
        o.rank = 0;  // the whole generation on this device
        o.world = 1;
        o.comm = nullptr;
        o.allreduce_min = nullptr;
        std::vector<sdb::GammaIn> gs;
        gs.push_back(std::move(gm));
        sdb::Plan plan(std::move(gs), mode == SDB_MODE_HAMMING ? sdb::Mode::hamming : sdb::Mode::symplectic,
                       pair_count, f, o);
        long long upper = state->upper;
        unsigned long long count = 0;
        const bool improved = plan.run_level(g, upper, &upper, &count, best_out);
        state->upper = upper;
        state->candidates_enumerated += count;
        state->improved = improved ? 1 : 0;
    });
}

sdb_status sdb_lower_bound(int g, int mode, int n_gammas, const int *rank_deficits, const int *n_packages,
                           const int *n_pp, long long *out) {
    return guarded([&] {
        if (n_gammas <= 0) throw sdb::InvalidArgument("lower_bound: no generator matrices");
        if (!out) throw sdb::InvalidArgument("null output");
        if (mode == SDB_MODE_HAMMING) {
            long long s = 0;
            for (int j = 0; j < n_gammas; j++) s += std::max(0LL, (long long)g + 1 - (rank_deficits ? rank_deficits[j] : 0));
            *out = s;
            return;
        }
        if (n_gammas == 1) {
            *out = (long long)g + 1;
            return;
        }
        if (n_gammas == 2) {
            const long long np = n_packages ? n_packages[1] : 0, npp = n_pp ? n_pp[1] : 0;
            *out = (long long)g + 1 + std::max(0LL, (long long)g + 1 + npp - np);
            return;
        }
        throw sdb::InvalidArgument("lower_bound: symplectic mode takes one or two matrices");
    });
}

sdb_status sdb_validate_normalizer(const uint64_t *rows, int n_rows, int n_cols, int row_words, int *ok, char *msg,
                                   int msg_len) {
    return guarded([&] {
        check_matrix_args(rows, n_rows, n_cols, row_words);
        if (n_cols == 0 || n_cols % 2 != 0)
            throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
        const sdb::Validation v = sdb::validate_normalizer(sdb::BitMat::from_words(rows, n_rows, n_cols, row_words));
        if (ok) *ok = v.ok ? 1 : 0;
        if (msg && msg_len > 0) {
            std::strncpy(msg, v.message.c_str(), size_t(msg_len) - 1);
            msg[msg_len - 1] = 0;
        }
    });
}

sdb_status sdb_isometry_transform(const uint64_t *rows, int n_rows, int n_cols, int row_words, uint64_t *out,
                                  int out_row_words) {
    return guarded([&] {
        check_matrix_args(rows, n_rows, n_cols, row_words);
        const sdb::BitMat img = sdb::isometry_transform(sdb::BitMat::from_words(rows, n_rows, n_cols, row_words));
        if (out_row_words < img.stride) throw sdb::InvalidArgument("out_row_words too small");
        img.to_words(out, out_row_words);
    });
}

sdb_status sdb_information_sets(const uint64_t *rows, int n_rows, int n_cols, int row_words, int max_gammas,
                                uint64_t *out, int out_row_words, int *deficits, int *pivots, int *n_gammas) {
    return guarded([&] {
        check_matrix_args(rows, n_rows, n_cols, row_words);
        if (out_row_words < (n_cols + 63) / 64) throw sdb::InvalidArgument("out_row_words too small");
        const std::vector<sdb::InfoSet> is =
            sdb::information_sets(sdb::BitMat::from_words(rows, n_rows, n_cols, row_words));
        if (n_gammas) *n_gammas = int(is.size());
        for (int j = 0; j < int(is.size()) && j < max_gammas; j++) {
            is[size_t(j)].matrix.to_words(out + size_t(j) * n_rows * out_row_words, out_row_words);
            if (deficits) deficits[j] = is[size_t(j)].rank_deficit;
            if (pivots)
                for (int i = 0; i < n_rows; i++) pivots[size_t(j) * n_rows + i] = is[size_t(j)].pivots[size_t(i)];
        }
    });
}

sdb_status sdb_tc_encoding_check(const uint64_t *rows, int n_rows, int n_cols, int row_words, int isometry,
                                 uint64_t seed, int trials, int *mismatches, int *k_per_gamma, int max_gammas,
                                 int *n_gammas) {
    return guarded([&] {
        check_matrix_args(rows, n_rows, n_cols, row_words);
        if (n_cols % 2) throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
        const int n = n_cols / 2;
        const sdb::BitMat a = sdb::BitMat::from_words(rows, n_rows, n_cols, row_words);
        std::vector<sdb::BitMat> ms;
        if (isometry) {
            for (sdb::InfoSet &is : sdb::information_sets(sdb::isometry_transform(a))) ms.push_back(std::move(is.matrix));
        } else {
            ms.push_back(a);
        }
        std::vector<const sdb::BitMat *> mp;
        for (const sdb::BitMat &m : ms) mp.push_back(&m);
        const sdb::TcEncoding enc = sdb::tc_encode(mp, n_rows, n, isometry != 0);
        if (n_gammas) *n_gammas = int(ms.size());
        for (int j = 0; k_per_gamma && j < int(enc.gam.size()) && j < max_gammas; j++) k_per_gamma[j] = enc.gam[size_t(j)].K;
        const int bad = enc.ok ? sdb::tc_selfcheck(enc, mp, n_rows, n, isometry != 0, seed, trials) : -1;
        if (mismatches) *mismatches = bad;
    });
}

sdb_status sdb_random_stabilizer(int n, int k, uint64_t seed, uint64_t *out, int out_row_words) {
    return guarded([&] {
        if (!out) throw sdb::InvalidArgument("null output");
        const sdb::BitMat a = sdb::random_stabilizer(n, k, seed);
        if (out_row_words < a.stride) throw sdb::InvalidArgument("out_row_words too small");
        a.to_words(out, out_row_words);
    });
}

sdb_status sdb_parse_matrix_text(const char *text, const char *origin, uint64_t *out, int out_row_words, int max_rows,
                                 int *n_rows, int *n_cols) {
    return guarded([&] {
        if (!text || !n_rows || !n_cols) throw sdb::InvalidArgument("null argument");
        const sdb::BitMat m = sdb::parse_matrix_text(text, origin ? origin : "<input>");
        *n_rows = m.rows;
        *n_cols = m.cols;
        if (out) {
            if (m.rows > max_rows || out_row_words < m.stride) throw sdb::InvalidArgument("output buffer too small");
            m.to_words(out, out_row_words);
        }
    });
}

sdb_status sdb_format_matrix(const uint64_t *rows, int n_rows, int n_cols, int row_words, char *buf, int cap,
                             int *len) {
    return guarded([&] {
        check_matrix_args(rows, n_rows, n_cols, row_words);
        const std::string s = sdb::format_matrix(sdb::BitMat::from_words(rows, n_rows, n_cols, row_words));
        if (len) *len = int(s.size());
        if (buf) {
            if (cap < int(s.size()) + 1) throw sdb::InvalidArgument("buffer too small");
            std::memcpy(buf, s.c_str(), s.size() + 1);
        }
    });
}

sdb_status sdb_generate_code(int n, int k, uint64_t seed, int transvections, uint64_t *out, int out_row_words) {
    return guarded([&] {
        if (!out) throw sdb::InvalidArgument("null output");
        const sdb::BitMat a = sdb::generate_code(n, k, seed, transvections);
        if (out_row_words < a.stride) throw sdb::InvalidArgument("out_row_words too small");
        a.to_words(out, out_row_words);
    });
}

sdb_status sdb_plan_create(const uint64_t *rows, int n_rows, int n_cols, int row_words, const sdb_run_options *opts,
                           sdb_plan **out) {
    return guarded([&] {
        if (!out) throw sdb::InvalidArgument("null plan output");
        *out = nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        check_matrix_args(rows, n_rows, n_cols, row_words);
        if (n_cols == 0 || n_cols % 2 != 0)
            throw sdb::InvalidArgument("StabilizerInstance: column count must be even and nonzero");
        const sdb_run_options o = opts_or_default(opts);
        const sdb::BitMat a = sdb::BitMat::from_words(rows, n_rows, n_cols, row_words);
        const int n = n_cols / 2, k = n_rows - n;
        if (o.validate) {
            const sdb::Validation v = sdb::validate_normalizer(a);
            if (!v.ok) throw sdb::ValidationFailure(v.message);
        }
        std::vector<sdb::InfoSet> is = sdb::information_sets(sdb::isometry_transform(a));
        std::vector<sdb::GammaIn> gammas;
        for (sdb::InfoSet &s : is) gammas.push_back(sdb::GammaIn{std::move(s.matrix), s.rank_deficit});
        sdb::Filter f;
        f.enabled = o.dual_filter && k >= 1;
        if (f.enabled) f.rows = a;
        auto *p = new sdb_plan{nullptr, n, SDB_ALG_SAVED_ISOMETRY, o, 0};
        try {
            p->plan = new sdb::Plan(std::move(gammas), sdb::Mode::hamming, n, f, o);
        } catch (...) {
            delete p;
            throw;
        }
        p->prep_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = p;
    });
}

sdb_status sdb_plan_run(sdb_plan *plan, sdb_report *report, sdb_trace_entry *trace, int trace_cap,
                        double *level_seconds) {
    return guarded([&] {
        if (!plan || !report) throw sdb::InvalidArgument("null plan or report");
        const auto t0 = std::chrono::steady_clock::now();
        zero_report(report);
        plan->plan->run(report, trace, trace_cap, nullptr, level_seconds);
        if (report->complete && report->upper % 2 != 0)
            throw sdb::InternalFailure("saved_isometry: image Hamming distance must be even");
        report->distance = int(report->upper / 2);
        report->algorithm = plan->algorithm;
        report->workers = plan->opts.workers;
        report->prep_seconds = plan->prep_seconds;
        report->elapsed_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

sdb_status sdb_comm_unique_id(unsigned char id[128]) {
    return guarded([&] {
        if (!id) throw sdb::InvalidArgument("null id");
        sdb::comm_unique_id(id);
    });
}

sdb_status sdb_comm_create(const unsigned char id[128], int rank, int world, int device, void **comm) {
    return guarded([&] {
        if (!id || !comm) throw sdb::InvalidArgument("null argument");
        *comm = sdb::comm_create(id, rank, world, device);
    });
}

sdb_status sdb_comm_allreduce_min(void *comm, uint64_t *values, int count, int device) {
    return guarded([&] {
        if (!comm || (!values && count > 0) || count < 0) throw sdb::InvalidArgument("null argument");
        sdb::check_cuda(cudaSetDevice(device), "cudaSetDevice");
        unsigned long long *d = nullptr;
        sdb::check_cuda(cudaMalloc(&d, size_t(std::max(count, 1)) * 8), "cudaMalloc");
        try {
            sdb::check_cuda(cudaMemcpy(d, values, size_t(count) * 8, cudaMemcpyHostToDevice), "H2D");
            sdb::comm_allreduce_min_u64(comm, d, size_t(count), nullptr);
            sdb::check_cuda(cudaMemcpy(values, d, size_t(count) * 8, cudaMemcpyDeviceToHost), "D2H");
        } catch (...) {
            cudaFree(d);
            throw;
        }
        cudaFree(d);
    });
}

void sdb_comm_destroy(void *comm) {
    try {
        sdb::comm_destroy(comm);
    } catch (...) {
    }
}

void sdb_plan_destroy(sdb_plan *plan) {
    if (!plan) return;
    delete plan->plan;
    delete plan;
}

}  // extern "C"
