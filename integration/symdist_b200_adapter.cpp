// Reference-side adapter: the file a maintainer adds to the reference tree so
// that symdist::saved_isometry / saved_1_gamma / saved_2_gamma / compute_distance run on the
// B200 through libsymdist_b200's C ABI (include/symdist_b200.h). It compiles against the
// reference's own headers (proj/include/symdist/*.hpp) and returns the reference's own
// DistanceReport type, so every caller (CLI, tests, bench) is unchanged.
//
//   symdist::saved_isometry  proj/include/symdist/distance.hpp:68   (proj/src/distance.cpp:135-149)
//   symdist::saved_1_gamma   proj/include/symdist/distance.hpp:60   (proj/src/distance.cpp:95-113)
//   symdist::saved_2_gamma   proj/include/symdist/distance.hpp:64   (proj/src/distance.cpp:115-133)
//   symdist::compute_distance proj/include/symdist/distance.hpp:74-75 (proj/src/distance.cpp:226-240)
//   error classes            proj/include/symdist/errors.hpp:7-20
#include "symdist_b200_adapter.hpp"

#include <stdexcept>
#include <string>
#include <vector>

#include "symdist/errors.hpp"
#include "symdist_b200.h"

namespace symdist {
namespace {

using RouteFn = sdb_status (*)(const uint64_t *, int, int, int, const sdb_run_options *, sdb_report *,
                               sdb_trace_entry *, int, uint64_t *);

// BitVector rows are little-endian 64-bit words (bitvec.hpp:12-14): the C ABI's row layout.
std::vector<uint64_t> pack(const BitMatrix &m, int &words) {
    words = int((m.n_cols() + 63) / 64);
    std::vector<uint64_t> out(m.n_rows() * size_t(words), 0);
    for (size_t r = 0; r < m.n_rows(); ++r) {
        const BitVector &v = m.row(r);
        for (size_t w = 0; w < v.word_count() && w < size_t(words); ++w) out[r * size_t(words) + w] = v.word_data()[w];
    }
    return out;
}

[[noreturn]] void rethrow(sdb_status st) {
    const std::string msg = sdb_last_error();
    switch (st) {
        case SDB_ERR_PARSE: throw ParseError(msg);
        case SDB_ERR_VALIDATION: throw ValidationError(msg);
        case SDB_ERR_INTERNAL: throw InternalError(msg);
        case SDB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        default: throw std::runtime_error("CUDA: " + msg);  // no reference counterpart
    }
}

sdb_run_options options(const RunOptions &opts) {
    sdb_run_options o;
    sdb_default_options(&o);
    o.workers = opts.workers;  // recorded in the report; the GPU path does not use host threads
    o.validate = opts.validate ? 1 : 0;
    o.dual_filter = opts.dual_filter ? 1 : 0;
    return o;
}

DistanceReport to_report(const sdb_report &rep, const std::vector<sdb_trace_entry> &tr, const RunOptions &opts) {
    DistanceReport out;
    out.distance = rep.distance;
    out.algorithm = static_cast<Algorithm>(rep.algorithm);  // same declaration order (distance.hpp:23-29)
    out.generations = rep.generations;
    out.candidates_enumerated = rep.candidates_enumerated;
    out.elapsed_seconds = rep.elapsed_seconds;
    out.workers = opts.workers;
    for (int i = 0; i < rep.trace_len && i < int(tr.size()); ++i)
        out.bounds_trace.push_back(BoundsTraceEntry{tr[size_t(i)].g, tr[size_t(i)].lower, tr[size_t(i)].upper});
    return out;
}

DistanceReport route(RouteFn fn, const StabilizerInstance &inst, const RunOptions &opts) {
    int words = 0;
    const std::vector<uint64_t> packed = pack(inst.a, words);
    const sdb_run_options o = options(opts);
    sdb_report rep{};
    std::vector<sdb_trace_entry> tr(512);
    const sdb_status st = fn(packed.data(), int(inst.a.n_rows()), int(inst.a.n_cols()), words, &o, &rep, tr.data(),
                             int(tr.size()), nullptr);
    if (st != SDB_OK) rethrow(st);
    return to_report(rep, tr, opts);
}

}  // namespace

DistanceReport saved_isometry_b200(const StabilizerInstance &inst, const RunOptions &opts) {
    return route(sdb_saved_isometry, inst, opts);
}

DistanceReport saved_1_gamma_b200(const StabilizerInstance &inst, const RunOptions &opts) {
    return route(sdb_saved_1_gamma, inst, opts);
}

DistanceReport saved_2_gamma_b200(const StabilizerInstance &inst, const RunOptions &opts) {
    return route(sdb_saved_2_gamma, inst, opts);
}

DistanceReport compute_distance_b200(const StabilizerInstance &inst, Algorithm alg, const RunOptions &opts) {
    int words = 0;
    const std::vector<uint64_t> packed = pack(inst.a, words);
    const sdb_run_options o = options(opts);
    sdb_report rep{};
    std::vector<sdb_trace_entry> tr(512);
    const sdb_status st = sdb_compute_distance(packed.data(), int(inst.a.n_rows()), int(inst.a.n_cols()), words,
                                               int(alg), &o, &rep, tr.data(), int(tr.size()));
    if (st != SDB_OK) rethrow(st);
    return to_report(rep, tr, opts);
}

}  // namespace symdist
