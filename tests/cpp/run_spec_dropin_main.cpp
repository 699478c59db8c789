// Drop-in check of the C++ solver interface: the reference CLI's run_spec
// (bjgmres_cli.cpp:112-168) and its helpers, extracted unmodified at build
// time into oracle/_ref/run_spec_extract.inc (oracle/extract_run_spec.py;
// the reference text is never committed), compiled against this repo's
// include/bjgmres/*.hpp and run on libhpbj.so. Only the CLI11 front end and
// the nlohmann::json report of the reference are left out; this main parses
// a few options and prints the result as one JSON line, writing x to a file.
//
// usage: run_spec_dropin MATRIX.mtx BLOCKS RESTART TOL MAX_RESTARTS PRECISION RHS X_OUT
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "bjgmres/gmres.hpp"
#include "bjgmres/graph.hpp"
#include "bjgmres/matrix_market.hpp"
#include "bjgmres/partition.hpp"
#include "bjgmres/preconditioner.hpp"
#include "bjgmres/spmv.hpp"

using namespace bjgmres;

namespace {
#include "run_spec_extract.inc"
}  // namespace

int main(int argc, char** argv) {
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s MATRIX BLOCKS RESTART TOL MAX_RESTARTS PRECISION RHS X_OUT\n", argv[0]);
        return 1;
    }
    RunSpec spec;
    spec.matrix_path = argv[1];
    spec.blocks = std::stoll(argv[2]);
    spec.restart_m = std::stoll(argv[3]);
    spec.tol = std::stod(argv[4]);
    spec.max_restarts = std::stoll(argv[5]);
    spec.precision = argv[6];
    spec.rhs_mode = argv[7];
    try {
        const RunResult r = run_spec(spec);
        std::ofstream xo(argv[8], std::ios::binary);
        xo.write(reinterpret_cast<const char*>(r.x.data()), static_cast<std::streamsize>(sizeof(double) * r.x.size()));
        index_t pert = 0;
        double cond_max = 0.0;
        for (const auto& st : r.block_stats) {
            pert += st.perturbation_count;
            cond_max = std::max(cond_max, st.cond_estimate);
        }
        std::printf("{\"name\": \"%s\", \"n\": %lld, \"nnz\": %lld, \"converged\": %s, \"iterations\": %lld, "
                    "\"restarts\": %lld, \"final_residual\": %.17g, \"history\": %zu, \"blocks\": %zu, "
                    "\"perturbations\": %lld, \"cond_max\": %.6g, \"setup_ms\": %.3f, \"solve_ms\": %.3f}\n",
                    r.matrix_name.c_str(), (long long)r.n, (long long)r.nnz, r.report.converged ? "true" : "false",
                    (long long)r.report.total_iterations, (long long)r.report.restarts, r.report.final_residual,
                    r.report.residual_history.size(), r.block_stats.size(), (long long)pert, cond_max, r.setup_ms,
                    r.solve_ms);
        return r.report.converged ? 0 : 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
