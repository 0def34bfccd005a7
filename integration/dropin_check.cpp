// Drop-in proof (test infrastructure): links the UNMODIFIED reference library
// (oracle/_ref/libsymdist_ref.so) and the adapter over libsymdist_b200.so into one program,
// parses each matrix file with the reference's own parser (matrix_io.hpp:13-15), runs the
// reference's entry point and the adapter's on the same StabilizerInstance and prints one JSON
// line per (file, algorithm) with both DistanceReports (distance.hpp:44-52) and whether every
// field the reference defines agrees (elapsed_seconds aside). Errors are compared by class.
//
//   dropin_check [--workers N] [--algs isometry,1g,2g,auto] FILE...
#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "symdist/distance.hpp"
#include "symdist/errors.hpp"
#include "symdist/matrix_io.hpp"
#include "symdist_b200_adapter.hpp"

using namespace symdist;

namespace {

struct Outcome {
    std::string error;  // exception class, empty on success
    std::string message;
    DistanceReport rep;
    double wall = 0;
};

Outcome run(const std::function<DistanceReport()> &fn) {
    Outcome o;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        o.rep = fn();
    } catch (const ParseError &e) {
        o.error = "ParseError", o.message = e.what();
    } catch (const ValidationError &e) {
        o.error = "ValidationError", o.message = e.what();
    } catch (const InternalError &e) {
        o.error = "InternalError", o.message = e.what();
    } catch (const std::invalid_argument &e) {
        o.error = "invalid_argument", o.message = e.what();
    } catch (const std::exception &e) {
        o.error = "other", o.message = e.what();
    }
    o.wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return o;
}

std::string esc(const std::string &s) {
    std::string out;
    for (char c : s) {
        if (c == '"' || c == '\\') out += '\\';
        if (c == '\n') { out += "\\n"; continue; }
        out += c;
    }
    return out;
}

std::string json(const Outcome &o) {
    std::ostringstream s;
    if (!o.error.empty()) {
        s << "{\"error\":\"" << o.error << "\",\"message\":\"" << esc(o.message) << "\",\"wall\":" << o.wall << "}";
        return s.str();
    }
    const DistanceReport &r = o.rep;
    s << "{\"distance\":" << r.distance << ",\"algorithm\":\"" << algorithm_name(r.algorithm)
      << "\",\"generations\":" << r.generations << ",\"candidates_enumerated\":" << r.candidates_enumerated
      << ",\"workers\":" << r.workers << ",\"elapsed_seconds\":" << r.elapsed_seconds << ",\"wall\":" << o.wall
      << ",\"trace\":[";
    for (size_t i = 0; i < r.bounds_trace.size(); ++i)
        s << (i ? "," : "") << "[" << r.bounds_trace[i].g << "," << r.bounds_trace[i].lower << ","
          << r.bounds_trace[i].upper << "]";
    s << "]}";
    return s.str();
}

bool same(const Outcome &a, const Outcome &b) {
    if (a.error != b.error) return false;
    if (!a.error.empty()) return true;
    const DistanceReport &x = a.rep, &y = b.rep;
    if (x.distance != y.distance || x.algorithm != y.algorithm || x.generations != y.generations ||
        x.candidates_enumerated != y.candidates_enumerated || x.workers != y.workers ||
        x.bounds_trace.size() != y.bounds_trace.size())
        return false;
    for (size_t i = 0; i < x.bounds_trace.size(); ++i)
        if (x.bounds_trace[i].g != y.bounds_trace[i].g || x.bounds_trace[i].lower != y.bounds_trace[i].lower ||
            x.bounds_trace[i].upper != y.bounds_trace[i].upper)
            return false;
    return true;
}

}  // namespace

int main(int argc, char **argv) {
    int workers = int(std::thread::hardware_concurrency());
    std::string algs = "isometry";
    std::vector<std::string> files;
    for (int i = 1; i < argc; ++i) {
        if (!std::strcmp(argv[i], "--workers") && i + 1 < argc) workers = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--algs") && i + 1 < argc) algs = argv[++i];
        else files.emplace_back(argv[i]);
    }
    if (workers < 1) workers = 1;
    RunOptions opts;
    opts.workers = workers;
    int mismatches = 0;
    for (const std::string &f : files) {
        Outcome parsed = run([&] { parse_matrix_file(f); return DistanceReport{}; });
        if (!parsed.error.empty()) {
            std::printf("{\"file\":\"%s\",\"parse_error\":\"%s\"}\n", esc(f).c_str(), esc(parsed.message).c_str());
            continue;
        }
        const StabilizerInstance inst = parse_matrix_file(f);
        std::stringstream ss(algs);
        std::string alg;
        while (std::getline(ss, alg, ',')) {
            Outcome ref, gpu;
            if (alg == "isometry") {
                ref = run([&] { return saved_isometry(inst, opts); });
                gpu = run([&] { return saved_isometry_b200(inst, opts); });
            } else if (alg == "1g") {
                ref = run([&] { return saved_1_gamma(inst, opts); });
                gpu = run([&] { return saved_1_gamma_b200(inst, opts); });
            } else if (alg == "2g") {
                ref = run([&] { return saved_2_gamma(inst, opts); });
                gpu = run([&] { return saved_2_gamma_b200(inst, opts); });
            } else if (alg == "auto") {
                ref = run([&] { return compute_distance(inst, Algorithm::auto_select, opts); });
                gpu = run([&] { return compute_distance_b200(inst, Algorithm::auto_select, opts); });
            } else {
                std::fprintf(stderr, "dropin_check: unknown algorithm %s\n", alg.c_str());
                return 2;
            }
            const bool eq = same(ref, gpu);
            mismatches += eq ? 0 : 1;
            std::printf("{\"file\":\"%s\",\"alg\":\"%s\",\"equal\":%s,\"reference\":%s,\"b200\":%s}\n", esc(f).c_str(),
                        alg.c_str(), eq ? "true" : "false", json(ref).c_str(), json(gpu).c_str());
            std::fflush(stdout);
        }
    }
    return mismatches ? 1 : 0;
}
