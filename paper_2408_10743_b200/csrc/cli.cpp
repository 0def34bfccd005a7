// symdist_b200: the reference CLI (proj/tools/symdist_main.cpp) over the C ABI
// (include/symdist_b200.h) — compute / verify / bench with the same flags, the same text
// output ("g= L= U=" trace lines, "distance d", the JSON report with the reference's keys) and
// the same exit codes (symdist_main.cpp:197-209: parse 1, validation / invalid argument 2,
// internal 3; CUDA failures 4). Every distance runs on the GPU.
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/symdist_b200.h"

namespace {

struct CliError : std::runtime_error {
    int code;
    CliError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void check(sdb_status st) {
    if (st == SDB_OK) return;
    const std::string msg = sdb_last_error();
    switch (st) {
        case SDB_ERR_PARSE: throw CliError(1, "error: " + msg);
        case SDB_ERR_VALIDATION:
        case SDB_ERR_INVALID_ARGUMENT: throw CliError(2, "error: " + msg);
        case SDB_ERR_INTERNAL: throw CliError(3, "internal error: " + msg);
        default: throw CliError(4, "device error: " + msg);
    }
}

struct Instance {
    int rows = 0, cols = 0, words = 0;
    std::vector<uint64_t> a;
    int n() const { return cols / 2; }
    int k() const { return rows - cols / 2; }
};

Instance parse_file(const std::string &path) {
    std::ifstream in(path);
    if (!in) throw CliError(1, "error: " + path + ": cannot open file");
    std::ostringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();
    Instance inst;
    check(sdb_parse_matrix_text(text.c_str(), path.c_str(), nullptr, 0, 0, &inst.rows, &inst.cols));
    inst.words = (inst.cols + 63) / 64;
    inst.a.assign(size_t(inst.rows) * inst.words, 0);
    check(sdb_parse_matrix_text(text.c_str(), path.c_str(), inst.a.data(), inst.words, inst.rows, &inst.rows,
                                &inst.cols));
    return inst;
}

int parse_algorithm(const std::string &name) {
    if (name == "auto") return SDB_ALG_AUTO;
    if (name == "1gamma") return SDB_ALG_SAVED_1_GAMMA;
    if (name == "2gamma") return SDB_ALG_SAVED_2_GAMMA;
    if (name == "isometry") return SDB_ALG_SAVED_ISOMETRY;
    if (name == "brute") return SDB_ALG_BRUTE_FORCE;
    throw CliError(2, "--alg: unknown algorithm '" + name + "'");
}

const char *algorithm_name(int alg) {
    switch (alg) {
        case SDB_ALG_AUTO: return "auto";
        case SDB_ALG_SAVED_1_GAMMA: return "saved_1_gamma";
        case SDB_ALG_SAVED_2_GAMMA: return "saved_2_gamma";
        case SDB_ALG_SAVED_ISOMETRY: return "saved_isometry";
        case SDB_ALG_BRUTE_FORCE: return "brute_force";
    }
    return "?";
}

struct Result {
    sdb_report rep{};
    std::vector<sdb_trace_entry> trace;
};

Result compute(const Instance &inst, int alg, const sdb_run_options &o) {
    Result r;
    r.trace.resize(1024);
    check(sdb_compute_distance(inst.a.data(), inst.rows, inst.cols, inst.words, alg, &o, &r.rep, r.trace.data(),
                               int(r.trace.size())));
    r.trace.resize(size_t(std::min(r.rep.trace_len, int(r.trace.size()))));
    return r;
}

// shortest decimal that reads back to the same double (what nlohmann::json prints)
std::string json_double(double x) {
    char buf[64];
    for (int prec = 1; prec <= 17; prec++) {
        std::snprintf(buf, sizeof buf, "%.*g", prec, x);
        if (std::strtod(buf, nullptr) == x) break;
    }
    std::string s = buf;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

// The reference's report_to_json (symdist_main.cpp:28-42) as nlohmann::json::dump(2) prints
// it: keys in sorted order, two-space indent.
std::string report_json(const Result &r, const Instance &inst) {
    std::ostringstream o;
    o << "{\n  \"algorithm\": \"" << algorithm_name(r.rep.algorithm) << "\",\n  \"bounds_trace\": [";
    for (size_t i = 0; i < r.trace.size(); i++) {
        o << (i ? "," : "") << "\n    {\n      \"L\": " << r.trace[i].lower << ",\n      \"U\": " << r.trace[i].upper
          << ",\n      \"g\": " << r.trace[i].g << "\n    }";
    }
    o << (r.trace.empty() ? "]" : "\n  ]") << ",\n  \"candidates_enumerated\": " << r.rep.candidates_enumerated
      << ",\n  \"distance\": " << r.rep.distance << ",\n  \"elapsed_seconds\": " << json_double(r.rep.elapsed_seconds)
      << ",\n  \"generations\": " << r.rep.generations << ",\n  \"k\": " << inst.k() << ",\n  \"n\": " << inst.n()
      << ",\n  \"workers\": " << r.rep.workers << "\n}";
    return o.str();
}

int cmd_compute(const std::string &file, const std::string &alg_name, int threads, bool emit_json, bool emit_trace,
                bool no_validate, bool no_dual_filter) {
    const Instance inst = parse_file(file);
    sdb_run_options o;
    sdb_default_options(&o);
    o.workers = threads;
    o.validate = no_validate ? 0 : 1;
    o.dual_filter = no_dual_filter ? 0 : 1;
    const Result r = compute(inst, parse_algorithm(alg_name), o);
    if (emit_trace)
        for (const sdb_trace_entry &e : r.trace) std::cout << "g=" << e.g << " L=" << e.lower << " U=" << e.upper << '\n';
    std::cout << "distance " << r.rep.distance << '\n';
    if (emit_json) std::cout << report_json(r, inst) << '\n';
    return 0;
}

int cmd_verify(const std::string &file, int threads) {
    const Instance inst = parse_file(file);
    sdb_run_options o;
    sdb_default_options(&o);
    o.workers = threads;
    std::vector<std::pair<int, int>> results;
    for (int alg : {SDB_ALG_SAVED_1_GAMMA, SDB_ALG_SAVED_2_GAMMA, SDB_ALG_SAVED_ISOMETRY})
        results.emplace_back(alg, compute(inst, alg, o).rep.distance);
    if (inst.rows <= 28)
        results.emplace_back(SDB_ALG_BRUTE_FORCE, compute(inst, SDB_ALG_BRUTE_FORCE, o).rep.distance);
    else
        std::cout << "note: n+k > 28, oracle skipped\n";
    const int d = results.front().second;
    if (std::all_of(results.begin(), results.end(), [d](const auto &r) { return r.second == d; })) {
        std::cout << "AGREE d=" << d << '\n';
        return 0;
    }
    std::cout << "DISAGREE\n";
    for (const auto &[alg, dist] : results) std::cout << "  " << algorithm_name(alg) << ": " << dist << '\n';
    throw CliError(3, "internal error: algorithms disagree on the distance");
}

double median_of(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t m = v.size() / 2;
    return v.size() % 2 ? v[m] : 0.5 * (v[m - 1] + v[m]);
}

int cmd_bench(int n, int k, int count, uint64_t seed, int threads) {
    sdb_run_options o;
    sdb_default_options(&o);
    o.workers = threads;
    o.validate = 0;  // instances are valid by construction
    const int algs[3] = {SDB_ALG_SAVED_1_GAMMA, SDB_ALG_SAVED_2_GAMMA, SDB_ALG_SAVED_ISOMETRY};
    std::vector<std::vector<double>> times(3);
    std::printf("instance  n  k  distance");
    for (int alg : algs) std::printf("  %14s_s", algorithm_name(alg));
    std::printf("\n");
    for (int i = 0; i < count; ++i) {
        Instance inst;
        inst.rows = n + k;
        inst.cols = 2 * n;
        inst.words = (inst.cols + 63) / 64;
        inst.a.assign(size_t(inst.rows) * inst.words, 0);
        check(sdb_random_stabilizer(n, k, seed + uint64_t(i), inst.a.data(), inst.words));
        std::printf("%8d %2d %2d", i, inst.n(), inst.k());
        int distance = -1;
        std::vector<double> row;
        for (int a = 0; a < 3; ++a) {
            const Result r = compute(inst, algs[a], o);
            if (distance < 0) {
                distance = r.rep.distance;
                std::printf("  %8d", distance);
            } else if (r.rep.distance != distance) {
                throw CliError(3, "internal error: bench: algorithms disagree on instance " + std::to_string(i));
            }
            times[size_t(a)].push_back(r.rep.elapsed_seconds);
            row.push_back(r.rep.elapsed_seconds);
        }
        for (double t : row) std::printf("  %16.6f", t);
        std::printf("\n");
    }
    std::printf("\nalgorithm         runs    median_s      mean_s       min_s       max_s\n");
    for (int a = 0; a < 3; ++a) {
        const std::vector<double> &t = times[size_t(a)];
        double sum = 0;
        for (double x : t) sum += x;
        std::printf("%-16s %5zu  %10.6f  %10.6f  %10.6f  %10.6f\n", algorithm_name(algs[a]), t.size(), median_of(t),
                    t.empty() ? 0.0 : sum / double(t.size()), *std::min_element(t.begin(), t.end()),
                    *std::max_element(t.begin(), t.end()));
    }
    return 0;
}

void usage() {
    std::cerr << "symplectic minimum distance of qubit stabilizer codes (B200)\n"
                 "usage: symdist_b200 compute FILE [--alg auto|1gamma|2gamma|isometry|brute] [--threads T]\n"
                 "                                 [--json] [--trace] [--no-validate] [--no-dual-filter]\n"
                 "       symdist_b200 verify FILE [--threads T]\n"
                 "       symdist_b200 bench [--n N] [--k K] [--count C] [--seed S] [--threads T]\n";
}

}  // namespace

int main(int argc, char **argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    if (args.empty()) {
        usage();
        return 106;  // CLI11: a required subcommand is missing
    }
    const std::string cmd = args[0];
    std::string file, alg = "auto";
    int threads = 1, bench_n = 10, bench_k = 2, bench_count = 5;
    uint64_t bench_seed = 1;
    bool emit_json = false, emit_trace = false, no_validate = false, no_dual_filter = false;
    try {
        auto value = [&](size_t &i) -> std::string {
            if (i + 1 >= args.size()) throw CliError(2, args[i] + ": expected a value");
            return args[++i];
        };
        for (size_t i = 1; i < args.size(); i++) {
            const std::string &a = args[i];
            if (a == "--alg") alg = value(i);
            else if (a == "--threads") threads = std::stoi(value(i));
            else if (a == "--json") emit_json = true;
            else if (a == "--trace") emit_trace = true;
            else if (a == "--no-validate") no_validate = true;
            else if (a == "--no-dual-filter") no_dual_filter = true;
            else if (a == "--n") bench_n = std::stoi(value(i));
            else if (a == "--k") bench_k = std::stoi(value(i));
            else if (a == "--count") bench_count = std::stoi(value(i));
            else if (a == "--seed") bench_seed = std::stoull(value(i));
            else if (!a.empty() && a[0] != '-' && file.empty()) file = a;
            else throw CliError(2, "unexpected argument '" + a + "'");
        }
        if (cmd == "compute") {
            if (file.empty()) throw CliError(2, "compute: FILE is required");
            return cmd_compute(file, alg, threads, emit_json, emit_trace, no_validate, no_dual_filter);
        }
        if (cmd == "verify") {
            if (file.empty()) throw CliError(2, "verify: FILE is required");
            return cmd_verify(file, threads);
        }
        if (cmd == "bench") return cmd_bench(bench_n, bench_k, bench_count, bench_seed, threads);
        usage();
        return 109;  // CLI11: unknown subcommand
    } catch (const CliError &e) {
        std::cout.flush();
        std::cerr << e.what() << '\n';
        return e.code;
    } catch (const std::exception &e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
