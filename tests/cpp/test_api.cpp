// C++ drop-in check: the reference's own test scenarios (proj/tests/
// test_krylov.cpp, test_preconditioners.cpp, test_graph_partition.cpp),
// restated against the reference API as include/bjgmres/*.hpp provides it
// (namespace bjgmres over libhpbj.so). Exit code 0 = all pass. Run by
// tests/test_cpp_api.py on a B200.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <vector>

#include "bjgmres/gmres.hpp"
#include "bjgmres/graph.hpp"
#include "bjgmres/partition.hpp"
#include "bjgmres/preconditioner.hpp"
#include "bjgmres/sparse_matrix.hpp"
#include "bjgmres/spmv.hpp"

using namespace bjgmres;

static int failures = 0;
#define EXPECT(cond)                                                  \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)

static SparseMatrix laplacian_2d(index_t nx, index_t ny) {  // fixtures.hpp:44-58
    std::vector<index_t> rs{0}, ci;
    std::vector<double> v;
    for (index_t iy = 0; iy < ny; ++iy)
        for (index_t ix = 0; ix < nx; ++ix) {
            const index_t c = iy * nx + ix;
            auto put = [&](index_t j, double x) { ci.push_back(j), v.push_back(x); };
            if (iy > 0) put(c - nx, -1.0);
            if (ix > 0) put(c - 1, -1.0);
            put(c, 4.0);
            if (ix + 1 < nx) put(c + 1, -1.0);
            if (iy + 1 < ny) put(c + nx, -1.0);
            rs.push_back(static_cast<index_t>(ci.size()));
        }
    return SparseMatrix(nx * ny, nx * ny, rs, ci, v);
}

static std::vector<double> matvec(const SparseMatrix& a, const std::vector<double>& x) {
    std::vector<double> y(a.rows(), 0.0);
    for (index_t i = 0; i < a.rows(); ++i)
        for (index_t k = a.row_starts()[i]; k < a.row_starts()[i + 1]; ++k) y[i] += a.values()[k] * x[a.col_indices()[k]];
    return y;
}

int main() {
    {  // test_krylov.cpp:308-329 ManufacturedSolutionOnLaplacian
        SparseMatrix a = laplacian_2d(32, 32);
        a.materialize_low();
        const std::vector<double> b = matvec(a, std::vector<double>(a.rows(), 1.0));
        BlockJacobiOptions o;
        o.policy.mode = PrecisionMode::Hybrid;
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_graph(graph_from_matrix(a), 16, 0.1), o);
        GmresConfig cfg;
        cfg.policy.mode = PrecisionMode::Hybrid;
        cfg.restart_m = 30;
        cfg.tol = 1e-8;
        const SolveResult r = hybrid_restart_gmres(a, p, b, cfg);
        EXPECT(r.report.converged);
        EXPECT(r.report.final_residual <= 1e-8);
        double err = 0.0;
        for (double xi : r.x) err = std::max(err, std::abs(xi - 1.0));
        EXPECT(err <= 1e-6);
        EXPECT(static_cast<index_t>(r.report.residual_history.size()) == r.report.total_iterations + 1);
    }
    {  // test_preconditioners.cpp:83-91 DiagonalMatrixDividesEntrywise (FP32 apply)
        const SparseMatrix a(4, 4, {0, 1, 2, 3, 4}, {0, 1, 2, 3}, {2.0, 5.0, 0.25, -4.0});
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_from_assignment({0, 0, 1, 1}, 2));
        const std::vector<double> v{1.0, 2.0, 3.0, 4.0};
        const std::vector<double> z = p.apply<double>(v);
        const double d[4] = {2.0, 5.0, 0.25, -4.0};
        for (int i = 0; i < 4; ++i) EXPECT(z[i] == static_cast<double>(static_cast<float>(v[i] / d[i])));
    }
    {  // test_preconditioners.cpp:196-211 SingularBlockFailsOnlyWithZeroEps
        const SparseMatrix a(4, 4, {0, 2, 4, 5, 6}, {0, 1, 0, 1, 2, 3}, {1.0, 1.0, 1.0, 1.0, 3.0, 4.0});
        bool thrown = false;
        try {
            BlockJacobiOptions strict;
            strict.eps_pivot = 0.0;
            Preconditioner::block_jacobi(a, partition_from_assignment({0, 0, 1, 1}, 2), strict);
        } catch (const SingularBlockError& e) {
            thrown = e.column() == 1;
        }
        EXPECT(thrown);
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_from_assignment({0, 0, 1, 1}, 2));
        const auto& st = p.block_jacobi_data()->stats;
        EXPECT(st[0].perturbation_count == 1 && st[1].perturbation_count == 0);
        EXPECT(st[0].block_nnz == 4 && st[1].block_nnz == 2 && st[0].block_dim == 2);
    }
    {  // test_graph_partition.cpp:212-216 stable gather; argument errors
        const Partition p = partition_from_assignment({1, 0, 1, 0}, 2);
        EXPECT((p.perm == std::vector<index_t>{2, 0, 3, 1}));
        bool thrown = false;
        try {
            partition_from_assignment({0, 0, 0, 0}, 2);
        } catch (const std::invalid_argument&) {
            thrown = true;
        }
        EXPECT(thrown);
    }
    {  // invalid config -> std::invalid_argument (gmres.cpp:203-207)
        SparseMatrix a = laplacian_2d(4, 4);
        a.materialize_low();
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_graph(graph_from_matrix(a), 2, 0.1));
        GmresConfig bad;
        bad.restart_m = 0;
        bool thrown = false;
        try {
            hybrid_restart_gmres(a, p, std::vector<double>(16, 1.0), bad);
        } catch (const std::invalid_argument&) {
            thrown = true;
        }
        EXPECT(thrown);
    }
    {  // test_preconditioners.cpp:238-249 ApplyNeumann FirstOrderSeriesExample
        const SparseMatrix a(2, 2, {0, 2, 4}, {0, 1, 0, 1}, {2.0, 1.0, 1.0, 2.0});
        BlockJacobiOptions opts;
        opts.neumann_order = 1;
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_from_assignment({0, 1}, 2), opts);
        const std::vector<double> v{1.0, 0.0};
        const std::vector<double> z = p.apply_neumann<double>(a, v, 1);
        EXPECT(z[0] == 0.5 && z[1] == -0.25);
        bool thrown = false;
        try {
            p.apply_neumann<double>(a, v, 2);
        } catch (const std::invalid_argument&) {
            thrown = true;
        }
        EXPECT(thrown);
    }
    {  // block diagnostics: cond >= 1 and the bound formula (preconditioner.cpp:13-15)
        const SparseMatrix a = laplacian_2d(8, 8);
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_graph(graph_from_matrix(a), 4, 0.1));
        for (const auto& st : p.block_jacobi_data()->stats) {
            EXPECT(st.cond_estimate >= 1.0);
            EXPECT(std::abs(st.error_bound - (st.cond_estimate * 0x1p-53 + 0x1p-24) * st.cond_estimate) <=
                   1e-12 * st.error_bound);
        }
    }
    {  // ILU(0) and identity behind the same solve (DoubleOnly), Hybrid ILU(0) throws like the reference
        SparseMatrix a = laplacian_2d(16, 16);
        const std::vector<double> b = matvec(a, std::vector<double>(a.rows(), 1.0));
        GmresConfig cfg;
        cfg.restart_m = 30;
        cfg.tol = 1e-10;
        cfg.policy.mode = PrecisionMode::DoubleOnly;
        a.materialize_low();
        const Preconditioner ilu = Preconditioner::from_ilu0(a);
        const SolveResult r = hybrid_restart_gmres(a, ilu, b, cfg);
        EXPECT(r.report.converged && r.report.final_residual <= 1e-10);
        const SolveResult r0 = hybrid_restart_gmres(a, Preconditioner::identity(a.rows()), b, cfg);
        EXPECT(r0.report.converged && r0.report.total_iterations > r.report.total_iterations);
        GmresConfig hyb = cfg;
        hyb.policy.mode = PrecisionMode::Hybrid;
        bool thrown = false;
        try {
            hybrid_restart_gmres(a, ilu, b, hyb);
        } catch (const std::logic_error&) {
            thrown = true;
        }
        EXPECT(thrown);
        const std::vector<double> z = ilu.apply<double>(b);
        EXPECT(z.size() == b.size());
        const LUFactors* f = ilu.ilu_factors();
        EXPECT(f && f->kind == FactorKind::Ilu0 && f->n == a.rows());
        EXPECT(f->lower.nnz() + f->upper.nnz() == a.nnz());
    }
    {  // graph_from_matrix weights (graph.cpp:17-51) read through the lists == the lazy CSR path
        const SparseMatrix a = SparseMatrix::from_triplets(
            std::vector<Triplet>{{0, 0, 4.0}, {0, 1, -1.0}, {1, 0, -3.0}, {1, 1, 4.0}, {1, 2, 2.0}, {2, 2, 1.0},
                                 {2, 3, 0.5}, {3, 3, 2.0}, {3, 3, 1.0}},
            4, 4);
        EXPECT(a.nnz() == 8 && a.value_at(3, 3) == 3.0);
        const WeightedGraph g = graph_from_matrix(a);
        EXPECT(g.num_nodes == 4 && g.degree(0) == 1 && g.num_edges() == 3);
        EXPECT(g.adjacency[0][0].neighbor == 1 && g.adjacency[0][0].weight == 2.0);
        EXPECT(g.adjacency[2][0].neighbor == 1 && g.adjacency[2][0].weight == 1.0);
        WeightedGraph h;  // an explicit graph takes the adjacency path
        h.num_nodes = 4;
        h.adjacency.resize(4);
        for (index_t u = 0; u < 4; ++u)
            for (const auto& e : g.adjacency[u]) h.adjacency[u].push_back(e);
        const Partition p1 = partition_graph(graph_from_matrix(a), 2, 0.1), p2 = partition_graph(h, 2, 0.1);
        EXPECT(p1.assignment == p2.assignment && p1.perm == p2.perm);
        std::stringstream io;
        export_partition(io, p1);
        const Partition p3 = import_partition(io, 4, 2);
        EXPECT(p3.assignment == p1.assignment && p3.block_starts == p1.block_starts);
    }
    {  // a preconditioner outlives the matrix object it was built from; a lagged
       // preconditioner solves a new matrix with the same pattern; a rebuilt one
       // reuses the pooled context and equals a fresh build
        auto make = [](double shift) {
            SparseMatrix a = laplacian_2d(24, 24);
            std::vector<double> v(a.values().begin(), a.values().end());
            for (index_t i = 0; i < a.rows(); ++i)
                for (index_t k = a.row_starts()[i]; k < a.row_starts()[i + 1]; ++k)
                    if (a.col_indices()[k] == i) v[k] += shift;
            SparseMatrix out(a.rows(), a.cols(), std::vector<index_t>(a.row_starts().begin(), a.row_starts().end()),
                             std::vector<index_t>(a.col_indices().begin(), a.col_indices().end()), std::move(v));
            out.materialize_low();
            return out;
        };
        GmresConfig cfg;
        cfg.restart_m = 30;
        cfg.tol = 1e-10;
        Preconditioner p = Preconditioner::identity(1);
        Partition part;
        {
            const SparseMatrix a0 = make(0.0);
            part = partition_graph(graph_from_matrix(a0), 9, 0.1);
            p = Preconditioner::block_jacobi(a0, part);
        }  // a0 gone: p keeps what it needs
        const SparseMatrix a1 = make(0.5);
        const std::vector<double> b = matvec(a1, std::vector<double>(a1.rows(), 1.0));
        const SolveResult lag = hybrid_restart_gmres(a1, p, b, cfg);
        EXPECT(lag.report.converged && lag.report.final_residual <= 1e-10);
        const Preconditioner p1 = Preconditioner::block_jacobi(a1, part);  // pooled context, refactor
        const SolveResult r1 = hybrid_restart_gmres(a1, p1, b, cfg);
        std::vector<double> z1 = p1.apply<double>(b);
        Preconditioner fresh = Preconditioner::identity(1);
        {
            std::vector<Preconditioner> hold;  // drain the pool: the next build gets a new context
            for (int k = 0; k < 6; ++k) hold.push_back(Preconditioner::block_jacobi(make(1.0 + k), part));
            fresh = Preconditioner::block_jacobi(a1, part);
        }
        const SolveResult r2 = hybrid_restart_gmres(a1, fresh, b, cfg);
        EXPECT(r1.report.total_iterations == r2.report.total_iterations && r1.x == r2.x);
        EXPECT(z1 == fresh.apply<double>(b));
        const BlockJacobiData* d = p1.block_jacobi_data();
        EXPECT(d && d->factors.size() == 9 && d->blocks.size() == 9);
        EXPECT(d->factors[0].n == d->stats[0].block_dim && d->blocks[0].rows() == d->stats[0].block_dim);
        EXPECT(d->blocks[0].nnz() == d->stats[0].block_nnz);
        const std::vector<double> ax = spmv<double>(a1, std::vector<double>(a1.rows(), 1.0));
        double e = 0.0;
        for (index_t i = 0; i < a1.rows(); ++i) e = std::max(e, std::abs(ax[i] - b[i]));
        EXPECT(e <= 1e-12);
        const SparseMatrix other = laplacian_2d(24, 23);
        bool thrown = false;
        try {
            hybrid_restart_gmres(other, p1, std::vector<double>(other.rows(), 1.0), cfg);
        } catch (const std::invalid_argument&) {
            thrown = true;
        }
        EXPECT(thrown);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
