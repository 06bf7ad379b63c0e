// parsa_main.cpp — the `parsa` command-line driver on the B200 engines.
//
// Same subcommands, flags and output text as the reference CLI
// (tools/parsa_main.cpp:1-217): list-functions, run, compare, trace.  The
// reference parses with CLI11, which is not vendored; this driver has its
// own small parser for exactly the flags the reference declares
// (`--flag value` and `--flag=value`).
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "parsa/harness.hpp"

namespace {

using namespace parsa;

struct Flags {
    std::string config, function_id, engine = "v2", chains, start, precision;
    double t0 = -1, tmin = -1, rho = -1;
    int chain_length = -1, reps = -1, workers = -1;
    std::uint64_t seed = 0;
    bool seed_set = false;
    std::string out_csv, summary_json, trace_csv;
    std::vector<std::string> engines{"v1", "v2"}; // compare
    std::string compare_out;
};

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::vector<std::string> split_commas(const std::string& s) {
    std::vector<std::string> parts;
    std::string cur;
    for (char ch : s) {
        if (ch == ',') {
            parts.push_back(cur);
            cur.clear();
        } else {
            cur += ch;
        }
    }
    parts.push_back(cur);
    return parts;
}

double to_double(const std::string& flag, const std::string& v) {
    try {
        std::size_t used = 0;
        const double d = std::stod(v, &used);
        if (used == v.size()) return d;
    } catch (const std::exception&) {
    }
    throw UsageError(flag + ": Value " + v + " could not be converted");
}

long long to_integer(const std::string& flag, const std::string& v) {
    try {
        std::size_t used = 0;
        const long long d = std::stoll(v, &used);
        if (used == v.size()) return d;
    } catch (const std::exception&) {
    }
    throw UsageError(flag + ": Value " + v + " could not be converted");
}

// Parses argv[first..] for subcommand `cmd` into f.
void parse_flags(const std::string& cmd, int argc, char** argv, int first, Flags& f) {
    const bool sched = cmd == "run" || cmd == "compare" || cmd == "trace";
    for (int i = first; i < argc; ++i) {
        std::string name = argv[i], value;
        bool inline_value = false;
        if (name.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + name);
        if (const auto eq = name.find('='); eq != std::string::npos) {
            value = name.substr(eq + 1);
            name = name.substr(0, eq);
            inline_value = true;
        }
        const auto next = [&]() -> std::string {
            if (inline_value) return value;
            if (i + 1 >= argc) throw UsageError(name + ": 1 required argument(s) missing");
            return argv[++i];
        };
        if (!sched) throw UsageError("The following argument was not expected: " + name);
        if (name == "--config") f.config = next();
        else if (name == "--function") f.function_id = next();
        else if (name == "--t0") f.t0 = to_double(name, next());
        else if (name == "--tmin") f.tmin = to_double(name, next());
        else if (name == "--rho") f.rho = to_double(name, next());
        else if (name == "--chain-length") f.chain_length = static_cast<int>(to_integer(name, next()));
        else if (name == "--chains") f.chains = next();
        else if (name == "--start") f.start = next();
        else if (name == "--seed") {
            f.seed = static_cast<std::uint64_t>(to_integer(name, next()));
            f.seed_set = true;
        } else if (name == "--reps") f.reps = static_cast<int>(to_integer(name, next()));
        else if (name == "--precision") f.precision = next();
        else if (name == "--workers") f.workers = static_cast<int>(to_integer(name, next()));
        else if (name == "--engine" && cmd != "compare") f.engine = next();
        else if (name == "--engines" && cmd == "compare") f.engines = split_commas(next());
        else if (name == "--out" && cmd == "run") f.out_csv = next();
        else if (name == "--out" && cmd == "compare") f.compare_out = next();
        else if (name == "--out" && cmd == "trace") f.trace_csv = next();
        else if (name == "--summary" && cmd == "run") f.summary_json = next();
        else if (name == "--trace" && cmd == "run") f.trace_csv = next();
        else throw UsageError("The following argument was not expected: " + name);
    }
}

// flags over the optional JSON config (parsa_main.cpp:50-85)
RunSpec spec_from(const Flags& f) {
    RunSpec spec;
    spec.replications = 1;
    if (!f.config.empty()) spec = run_spec_from_json_file(f.config);
    if (!f.function_id.empty()) spec.function_id = f.function_id;
    if (!f.engine.empty()) spec.engine = parse_engine(f.engine);
    if (f.t0 > 0) spec.schedule.t0 = f.t0;
    if (f.tmin > 0) spec.schedule.t_min = f.tmin;
    if (f.rho > 0) spec.schedule.rho = f.rho;
    if (f.chain_length > 0) spec.schedule.sweep_length = f.chain_length;
    if (!f.chains.empty()) spec.n_chains = parse_chain_count(f.chains);
    if (!f.start.empty()) {
        if (f.start == "shared") spec.start_mode = StartMode::shared_point;
        else if (f.start == "random") spec.start_mode = StartMode::random_per_chain;
        else throw std::invalid_argument("--start: expected shared|random");
    }
    if (f.seed_set) spec.seed = f.seed;
    if (f.reps > 0) spec.replications = f.reps;
    if (!f.precision.empty()) {
        if (f.precision == "double") spec.precision = Precision::f64;
        else if (f.precision == "single") spec.precision = Precision::f32;
        else throw std::invalid_argument("--precision: expected double|single");
    }
    if (f.workers >= 0) spec.workers = f.workers;
    if (!f.out_csv.empty()) spec.out_csv = f.out_csv;
    if (!f.summary_json.empty()) spec.summary_json = f.summary_json;
    if (!f.trace_csv.empty()) spec.trace_csv = f.trace_csv;
    return spec;
}

// "[lo,hi]^n" when every coordinate shares the box, else the product
std::string box_text(const BoxDomain& b) {
    bool same = true;
    for (int k = 1; k < b.dim(); ++k) same = same && b.lower[k] == b.lower[0] && b.upper[k] == b.upper[0];
    if (same)
        return "[" + format_double(b.lower[0]) + "," + format_double(b.upper[0]) + "]^" + std::to_string(b.dim());
    std::string t;
    for (int k = 0; k < b.dim(); ++k) {
        if (k) t += "x";
        t += "[" + format_double(b.lower[k]) + "," + format_double(b.upper[k]) + "]";
    }
    return t;
}

int list_functions() {
    std::printf("%-6s %-26s %5s %-18s %s\n", "id", "name", "n", "domain", "f_star");
    for (const ObjectiveFunction& f : registry())
        std::printf("%-6s %-26s %5d %-18s %s\n", f.id.c_str(), f.name.c_str(), f.dim, box_text(f.domain).c_str(),
                    format_double(f.reference.f_star).c_str());
    return 0;
}

int run(const Flags& f) {
    const RunSpec spec = spec_from(f);
    const ReplicationReport rep = run_spec(spec);
    std::cout << "function " << spec.function_id << ", engine " << engine_name(spec.engine) << ", "
              << rep.rows.size() << " replication(s), " << rep.evaluations << " evaluations each\n";
    std::cout << "value_error median " << format_double(rep.value_error.median) << " (mean "
              << format_double(rep.value_error.mean) << ", min " << format_double(rep.value_error.min) << ", max "
              << format_double(rep.value_error.max) << ")\n";
    if (rep.location_error) std::cout << "location_error median " << format_double(rep.location_error->median) << "\n";
    else std::cout << "location_error -\n";
    std::cout << "wall_time_s median " << format_double(rep.wall_time_s.median) << "\n";
    return 0;
}

int compare(const Flags& f) {
    std::vector<RunSpec> specs;
    for (const std::string& e : f.engines) {
        Flags one = f;
        one.engine = e;
        specs.push_back(spec_from(one));
    }
    const ComparisonTable t = compare_engines(specs);
    std::cout << t.to_text();
    if (!f.compare_out.empty()) {
        std::ofstream out(f.compare_out);
        if (!out) throw std::runtime_error("cannot open output file: " + f.compare_out);
        out << "engine,median_value_error,median_location_error,median_wall_time_s,time_ratio_vs_first\n";
        for (const ComparisonRow& r : t.rows)
            out << r.engine << ',' << format_double(r.median_value_error) << ','
                << (r.median_location_error ? format_double(*r.median_location_error) : std::string("-")) << ','
                << format_double(r.median_wall_time_s) << ',' << format_double(r.time_ratio_vs_first) << '\n';
    }
    return 0;
}

int trace(const Flags& f) {
    RunSpec spec = spec_from(f);
    spec.replications = 1;
    if (spec.trace_csv.empty()) throw std::invalid_argument("--out: trace needs an output path");
    (void)run_spec(spec);
    std::cout << "trace written to " << spec.trace_csv << "\n";
    return 0;
}

const char* kUsage =
    "parallel simulated annealing benchmark driver (B200)\n"
    "Usage: parsa SUBCOMMAND [OPTIONS]\n"
    "Subcommands:\n"
    "  list-functions   print the benchmark registry\n"
    "  run              run a replicated experiment\n"
    "  compare          engines side by side at equal budget\n"
    "  trace            single run, write the convergence trace\n";

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "A subcommand is required\n" << kUsage;
        return 106;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        std::cout << kUsage;
        return 0;
    }
    if (cmd != "list-functions" && cmd != "run" && cmd != "compare" && cmd != "trace") {
        std::cerr << "The following argument was not expected: " << cmd << "\n" << kUsage;
        return 109;
    }
    Flags flags;
    try {
        parse_flags(cmd, argc, argv, 2, flags);
        if (cmd == "trace" && flags.trace_csv.empty()) throw UsageError("--out is required");
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\n" << kUsage;
        return 109;
    }
    try {
        if (cmd == "list-functions") return list_functions();
        if (cmd == "run") return run(flags);
        if (cmd == "compare") return compare(flags);
        return trace(flags);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
