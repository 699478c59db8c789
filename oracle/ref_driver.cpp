// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// C-ABI harness over the UNMODIFIED reference library (arXiv 2509.09139
// artifact, /root/reference/proj). oracle/Makefile compiles the reference
// sources in place (proj/src/*.cpp, with the reference's own flags
// -std=c++20 -O2 -fopenmp -ffp-contract=off, proj/CMakeLists.txt:3,12-16)
// together with this file into oracle/_ref/libbjref.so. Nothing from the
// reference is copied into this repository; this file only *calls* its
// public API exactly the way the reference CLI does (bjgmres_cli.cpp:112-168).
//
// Users: tests/ (parity checks), tests/golden/make_golden.py (fixtures) and
// bench.py --impl reference / cpu_baseline (the reference CPU arm).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "bjgmres/gmres.hpp"
#include "bjgmres/graph.hpp"
#include "bjgmres/lu.hpp"
#include "bjgmres/matrix_market.hpp"
#include "bjgmres/partition.hpp"
#include "bjgmres/preconditioner.hpp"
#include "bjgmres/sparse_matrix.hpp"
#include "bjgmres/spmv.hpp"

using namespace bjgmres;

namespace {

thread_local std::string g_err;

SparseMatrix make_matrix(int64_t n, const int64_t* rp, const int64_t* ci,
                         const double* v) {
    std::vector<index_t> starts(rp, rp + n + 1);
    const int64_t nnz = rp[n];
    std::vector<index_t> cols(ci, ci + nnz);
    std::vector<double> vals(v, v + nnz);
    return SparseMatrix(n, n, std::move(starts), std::move(cols), std::move(vals));
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
        .count();
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const SingularBlockError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

}  // namespace

extern "C" {

struct bjref_report {
    int64_t converged;
    int64_t total_iterations;
    int64_t restarts;
    double final_residual;
    int64_t breakdown;
    int64_t ls_rank_deficient;
    int64_t hist_len;
    int64_t cyc_len;
    double ms_graph;
    double ms_partition;
    double ms_block_jacobi;
    double ms_setup;  // materialize_low + graph + partition + block_jacobi (cli:125-151)
    double ms_solve;  // hybrid_restart_gmres (cli:162-164)
    int64_t perturbations;
};

const char* bjref_last_error(void) { return g_err.c_str(); }

// read_matrix_market_file; rp == nullptr: only report the sizes (nrows,
// ncols, nnz), else fill rp[nrows+1], ci[nnz], v[nnz].
int bjref_mm_read(const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz, int64_t* rp, int64_t* ci,
                  double* v) {
    return guarded([&] {
        const SparseMatrix a = read_matrix_market_file(path);
        *nrows = a.rows();
        *ncols = a.cols();
        *nnz = a.nnz();
        if (!rp) return;
        const auto st = a.row_starts();
        const auto cl = a.col_indices();
        const auto vl = a.values();
        std::copy(st.begin(), st.end(), rp);
        std::copy(cl.begin(), cl.end(), ci);
        std::copy(vl.begin(), vl.end(), v);
    });
}

// write_matrix_market_file
int bjref_mm_write(const char* path, int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
    return guarded([&] { write_matrix_market_file(path, make_matrix(n, rp, ci, v)); });
}

int bjref_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
               const double* x, double* y, int fp32) {
    return guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        if (fp32) {
            a.materialize_low();
            std::vector<float> xf(x, x + n), yf(n);
            spmv<float>(a, xf, yf);
            for (int64_t i = 0; i < n; ++i) y[i] = yf[i];
        } else {
            spmv<double>(a, std::span<const double>(x, n), std::span<double>(y, n));
        }
    });
}

/// Adjacency of graph_from_matrix as CSR: starts[n+1], nbr[], w[].
int bjref_graph(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                int64_t* starts, int64_t* nbr, double* w, int64_t cap) {
    return guarded([&] {
        const WeightedGraph g = graph_from_matrix(make_matrix(n, rp, ci, v));
        int64_t k = 0;
        starts[0] = 0;
        for (int64_t u = 0; u < n; ++u) {
            for (const WeightedEdge& e : g.adjacency[u]) {
                if (k >= cap) throw std::runtime_error("bjref_graph: capacity");
                nbr[k] = e.neighbor;
                w[k] = e.weight;
                ++k;
            }
            starts[u + 1] = k;
        }
    });
}

int bjref_partition(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    int64_t s, double tol, int64_t* assignment, int64_t* perm,
                    int64_t* block_starts, double* ms_graph, double* ms_part) {
    return guarded([&] {
        const SparseMatrix a = make_matrix(n, rp, ci, v);
        auto t0 = std::chrono::steady_clock::now();
        const WeightedGraph g = graph_from_matrix(a);
        if (ms_graph) *ms_graph = ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        const Partition p = partition_graph(g, s, tol);
        if (ms_part) *ms_part = ms_since(t0);
        std::memcpy(assignment, p.assignment.data(), sizeof(int64_t) * n);
        std::memcpy(perm, p.perm.data(), sizeof(int64_t) * n);
        std::memcpy(block_starts, p.block_starts.data(), sizeof(int64_t) * (s + 1));
    });
}

/// Partition of an explicit graph (CSR adjacency) — pins partition_graph on
/// hand-built graphs such as the reference tests' path graphs.
int bjref_partition_graph(int64_t n, const int64_t* starts, const int64_t* nbr,
                          const double* w, int64_t s, double tol, int64_t* assignment) {
    return guarded([&] {
        WeightedGraph g;
        g.num_nodes = n;
        g.adjacency.resize(n);
        for (int64_t u = 0; u < n; ++u)
            for (int64_t k = starts[u]; k < starts[u + 1]; ++k)
                g.adjacency[u].push_back({nbr[k], w[k]});
        const Partition p = partition_graph(g, s, tol);
        std::memcpy(assignment, p.assignment.data(), sizeof(int64_t) * n);
    });
}

int bjref_permute(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  const int64_t* perm, int64_t* rp_out, int64_t* ci_out, double* v_out) {
    return guarded([&] {
        const SparseMatrix b =
            permute_symmetric(make_matrix(n, rp, ci, v), std::span<const index_t>(perm, n));
        std::memcpy(rp_out, b.row_starts().data(), sizeof(int64_t) * (n + 1));
        std::memcpy(ci_out, b.col_indices().data(), sizeof(int64_t) * b.nnz());
        std::memcpy(v_out, b.values().data(), sizeof(double) * b.nnz());
    });
}

/// Block factors of Preconditioner::block_jacobi, densified per block as
/// F = L_strict + U in pivot order, row-major d x d, concatenated over blocks
/// in block order (offset of block b = sum_{c<b} d_c^2). F32 holds the
/// values_low() cast (preconditioner.cpp:140), F64 the binary64 masters.
// PreconditionerStats with the condition estimates (with_cond_estimates =
// true, the reference default): cond_estimate, error_bound, block_nnz per block.
int bjref_block_stats(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
                      const int64_t* assignment, double eps, double* cond, double* ebound, int64_t* block_nnz) {
    return guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        a.materialize_low();
        BlockJacobiOptions opts;
        opts.eps_pivot = eps;
        opts.policy.mode = PrecisionMode::Hybrid;
        opts.with_cond_estimates = true;
        const Preconditioner p = Preconditioner::block_jacobi(
            a, partition_from_assignment(std::vector<index_t>(assignment, assignment + n), s), opts);
        const BlockJacobiData* d = p.block_jacobi_data();
        for (int64_t b = 0; b < s; ++b) {
            cond[b] = d->stats[b].cond_estimate;
            ebound[b] = d->stats[b].error_bound;
            block_nnz[b] = d->stats[b].block_nnz;
        }
    });
}

int bjref_factors(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  int64_t s, const int64_t* assignment, double eps, float* f32,
                  double* f64, int64_t* pivot_rows, int64_t* pert_count,
                  int64_t* sing_col) {
    *sing_col = -1;
    int rc = guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        a.materialize_low();
        BlockJacobiOptions opts;
        opts.eps_pivot = eps;
        opts.policy.mode = PrecisionMode::Hybrid;
        opts.with_cond_estimates = false;
        const Preconditioner p = Preconditioner::block_jacobi(
            a, partition_from_assignment(std::vector<index_t>(assignment, assignment + n), s),
            opts);
        const BlockJacobiData* d = p.block_jacobi_data();
        int64_t off = 0;
        for (int64_t b = 0; b < s; ++b) {
            const LUFactors& f = d->factors[b];
            const int64_t dim = f.n;
            const int64_t base = d->partition.block_starts[b];
            if (f32) std::memset(f32 + off, 0, sizeof(float) * dim * dim);
            if (f64) std::memset(f64 + off, 0, sizeof(double) * dim * dim);
            const auto put = [&](const SparseMatrix& m) {
                const auto st = m.row_starts();
                const auto cs = m.col_indices();
                const auto vs = m.values();
                const auto vl = m.values_low();
                for (int64_t i = 0; i < dim; ++i)
                    for (int64_t k = st[i]; k < st[i + 1]; ++k) {
                        if (f32) f32[off + i * dim + cs[k]] = vl[k];
                        if (f64) f64[off + i * dim + cs[k]] = vs[k];
                    }
            };
            put(f.lower);
            put(f.upper);
            for (int64_t k = 0; k < dim; ++k) pivot_rows[base + k] = f.pivot_rows[k];
            pert_count[b] = d->stats[b].perturbation_count;
            off += dim * dim;
        }
    });
    return rc;
}

/// Preconditioner::apply<T> (preconditioner.cpp:159-198) in the original
/// ordering; mode 0 = binary64 factors, 1 = binary32 (Hybrid) factors.
int bjref_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                int64_t s, const int64_t* assignment, double eps, int mode,
                const double* vin, double* zout) {
    return guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        a.materialize_low();
        BlockJacobiOptions opts;
        opts.eps_pivot = eps;
        opts.policy.mode = PrecisionMode::Hybrid;
        opts.with_cond_estimates = false;
        const Preconditioner p = Preconditioner::block_jacobi(
            a, partition_from_assignment(std::vector<index_t>(assignment, assignment + n), s),
            opts);
        if (mode == 1) {
            std::vector<float> vf(vin, vin + n), zf(n);
            p.apply<float>(vf, zf);
            for (int64_t i = 0; i < n; ++i) zout[i] = zf[i];
        } else {
            p.apply<double>(std::span<const double>(vin, n), std::span<double>(zout, n));
        }
    });
}

/// Preconditioner::apply_neumann<T> (preconditioner.cpp:200-220), original
/// ordering; built with BlockJacobiOptions::neumann_order = order; mode 0 =
/// binary64, 1 = binary32 (Hybrid factors and a binary32 SpMV).
int bjref_apply_neumann(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        int64_t s, const int64_t* assignment, double eps, int order, int k, int mode,
                        const double* vin, double* zout) {
    return guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        a.materialize_low();
        BlockJacobiOptions opts;
        opts.eps_pivot = eps;
        opts.neumann_order = order;
        opts.policy.mode = PrecisionMode::Hybrid;
        opts.with_cond_estimates = false;
        const Preconditioner p = Preconditioner::block_jacobi(
            a, partition_from_assignment(std::vector<index_t>(assignment, assignment + n), s),
            opts);
        if (mode == 1) {
            const std::vector<float> vf(vin, vin + n);
            const std::vector<float> zf = p.apply_neumann<float>(a, vf, k);
            for (int64_t i = 0; i < n; ++i) zout[i] = zf[i];
        } else {
            const std::vector<double> z = p.apply_neumann<double>(a, std::span<const double>(vin, n), k);
            std::memcpy(zout, z.data(), sizeof(double) * n);
        }
    });
}

static int g_neumann_order = 0;  // BlockJacobiOptions::neumann_order for bjref_solve

void bjref_set_neumann_order(int order) { g_neumann_order = order; }

/// Full reference path exactly as run_spec (bjgmres_cli.cpp:112-168):
/// materialize_low, graph_from_matrix, partition_graph(s, 0.1) (or the given
/// assignment), block_jacobi, hybrid_restart_gmres. hist is (cycle, iter,
/// rel) triples.
int bjref_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                int64_t s, const int64_t* assignment, const double* b, int64_t m,
                double tol, int64_t max_restarts, int hybrid, int absolute_tol,
                double eps, int cond_estimates, double* x, bjref_report* rep,
                double* hist, int64_t hist_cap, double* cycres, int64_t cyc_cap) {
    std::memset(rep, 0, sizeof(*rep));
    return guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        const auto t_setup = std::chrono::steady_clock::now();
        if (hybrid) a.materialize_low();
        Partition part;
        if (assignment) {
            part = partition_from_assignment(
                std::vector<index_t>(assignment, assignment + n), s);
        } else {
            auto t0 = std::chrono::steady_clock::now();
            const WeightedGraph g = graph_from_matrix(a);
            rep->ms_graph = ms_since(t0);
            t0 = std::chrono::steady_clock::now();
            part = partition_graph(g, s, 0.1);
            rep->ms_partition = ms_since(t0);
        }
        BlockJacobiOptions opts;
        opts.eps_pivot = eps;
        opts.policy.mode = hybrid ? PrecisionMode::Hybrid : PrecisionMode::DoubleOnly;
        opts.with_cond_estimates = cond_estimates != 0;
        opts.neumann_order = g_neumann_order;
        auto t0 = std::chrono::steady_clock::now();
        const Preconditioner p = Preconditioner::block_jacobi(a, std::move(part), opts);
        rep->ms_block_jacobi = ms_since(t0);
        rep->ms_setup = ms_since(t_setup);
        for (const auto& st : p.block_jacobi_data()->stats)
            rep->perturbations += st.perturbation_count;

        GmresConfig cfg;
        cfg.restart_m = m;
        cfg.tol = tol;
        cfg.max_restarts = max_restarts;
        cfg.absolute_tol = absolute_tol != 0;
        cfg.policy.mode = hybrid ? PrecisionMode::Hybrid : PrecisionMode::DoubleOnly;
        const auto t_solve = std::chrono::steady_clock::now();
        const SolveResult sr = hybrid_restart_gmres(a, p, std::span<const double>(b, n), cfg);
        rep->ms_solve = ms_since(t_solve);

        std::memcpy(x, sr.x.data(), sizeof(double) * n);
        const SolveReport& r = sr.report;
        rep->converged = r.converged;
        rep->total_iterations = r.total_iterations;
        rep->restarts = r.restarts;
        rep->final_residual = r.final_residual;
        rep->breakdown = r.breakdown;
        rep->ls_rank_deficient = r.ls_rank_deficient;
        rep->hist_len = static_cast<int64_t>(r.residual_history.size());
        rep->cyc_len = static_cast<int64_t>(r.cycle_residuals.size());
        for (int64_t k = 0; k < rep->hist_len && k < hist_cap; ++k) {
            hist[3 * k + 0] = static_cast<double>(r.residual_history[k].cycle);
            hist[3 * k + 1] = static_cast<double>(r.residual_history[k].iteration);
            hist[3 * k + 2] = r.residual_history[k].relative_residual;
        }
        for (int64_t k = 0; k < rep->cyc_len && k < cyc_cap; ++k) cycres[k] = r.cycle_residuals[k];
    });
}

/// ilu0 (lu.cpp:227-312): the factored values in A's pattern — per row the
/// LUFactors lower row then the upper row (diagonal first), which is A's own
/// column order.
int bjref_ilu0_values(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, double* out) {
    return guarded([&] {
        const SparseMatrix a = make_matrix(n, rp, ci, v);
        const LUFactors f = ilu0(a);
        const auto ls = f.lower.row_starts();
        const auto us = f.upper.row_starts();
        const auto lv = f.lower.values();
        const auto uv = f.upper.values();
        int64_t q = 0;
        for (int64_t i = 0; i < n; ++i) {
            for (index_t k = ls[i]; k < ls[i + 1]; ++k) out[q++] = lv[k];
            for (index_t k = us[i]; k < us[i + 1]; ++k) out[q++] = uv[k];
        }
    });
}

/// Preconditioner::from_ilu0(a).apply<double> (preconditioner.cpp:168-170).
int bjref_ilu0_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* vin,
                     double* zout) {
    return guarded([&] {
        const SparseMatrix a = make_matrix(n, rp, ci, v);
        const Preconditioner p = Preconditioner::from_ilu0(a);
        p.apply<double>(std::span<const double>(vin, n), std::span<double>(zout, n));
    });
}

static int g_alt_precond = 0;  // bjref_solve_identity: 0 = identity, 1 = ILU(0) (run_spec, cli:128-131)

void bjref_set_alt_precond(int kind) { g_alt_precond = kind; }

/// Identity-preconditioned solve (Preconditioner::identity) for the
/// reference's unpreconditioned Krylov known-answer tests; with
/// bjref_set_alt_precond(1) the ILU(0) preconditioner instead.
int bjref_solve_identity(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                         const double* b, int64_t m, double tol, int64_t max_restarts,
                         int hybrid, double* x, bjref_report* rep, double* hist,
                         int64_t hist_cap, double* cycres, int64_t cyc_cap) {
    std::memset(rep, 0, sizeof(*rep));
    return guarded([&] {
        SparseMatrix a = make_matrix(n, rp, ci, v);
        if (hybrid) a.materialize_low();
        GmresConfig cfg;
        cfg.restart_m = m;
        cfg.tol = tol;
        cfg.max_restarts = max_restarts;
        cfg.policy.mode = hybrid ? PrecisionMode::Hybrid : PrecisionMode::DoubleOnly;
        const Preconditioner p =
            g_alt_precond == 1 ? Preconditioner::from_ilu0(a) : Preconditioner::identity(n);
        const SolveResult sr = hybrid_restart_gmres(a, p, std::span<const double>(b, n), cfg);
        std::memcpy(x, sr.x.data(), sizeof(double) * n);
        const SolveReport& r = sr.report;
        rep->converged = r.converged;
        rep->total_iterations = r.total_iterations;
        rep->restarts = r.restarts;
        rep->final_residual = r.final_residual;
        rep->breakdown = r.breakdown;
        rep->ls_rank_deficient = r.ls_rank_deficient;
        rep->hist_len = static_cast<int64_t>(r.residual_history.size());
        rep->cyc_len = static_cast<int64_t>(r.cycle_residuals.size());
        for (int64_t k = 0; k < rep->hist_len && k < hist_cap; ++k) {
            hist[3 * k + 0] = static_cast<double>(r.residual_history[k].cycle);
            hist[3 * k + 1] = static_cast<double>(r.residual_history[k].iteration);
            hist[3 * k + 2] = r.residual_history[k].relative_residual;
        }
        for (int64_t k = 0; k < rep->cyc_len && k < cyc_cap; ++k) cycres[k] = r.cycle_residuals[k];
    });
}

}  // extern "C"
