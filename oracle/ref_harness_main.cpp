// ref_harness_main.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the UNMODIFIED reference harness (harness.cpp, compiled from
// /root/reference/proj/src by oracle/Makefile, namespace renamed to
// parsa_ref) on a JSON run config, so tests/golden/make_harness_golden.py can
// record the reference's own report files (rows CSV, summary JSON, traces)
// as byte-exact fixtures for the B200 harness and CLI.
//
//   ref_harness run <config.json>
#include <cstdio>
#include <exception>
#include <string>

#include "parsa/harness.hpp"

int main(int argc, char** argv) {
    if (argc != 3 || std::string(argv[1]) != "run") {
        std::fprintf(stderr, "usage: ref_harness run <config.json>\n");
        return 2;
    }
    try {
        const parsa_ref::RunSpec spec = parsa_ref::run_spec_from_json_file(argv[2]);
        const auto rep = parsa_ref::run_spec(spec);
        std::printf("%zu rows, %llu evaluations\n", rep.rows.size(),
                    static_cast<unsigned long long>(rep.evaluations));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
