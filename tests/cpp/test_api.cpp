// C++ drop-in check: the reference's own test scenarios (proj/tests/
// test_krylov.cpp, test_preconditioners.cpp, test_graph_partition.cpp),
// restated against include/bjgmres_b200.hpp (C++ API over libhpbj.so).
// Exit code 0 = all pass. Run by tests/test_cpp_api.py on a B200.
#include <cmath>
#include <cstdio>
#include <vector>

#include "bjgmres_b200.hpp"

using namespace bjgmres_b200;

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
        const SparseMatrix a = laplacian_2d(32, 32);
        const std::vector<double> b = matvec(a, std::vector<double>(a.rows(), 1.0));
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_graph(a, 16, 0.1));
        GmresConfig cfg;
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
        const std::vector<double> z = p.apply(v);
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
        EXPECT(p.stats()[0].perturbation_count == 1 && p.stats()[1].perturbation_count == 0);
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
        const SparseMatrix a = laplacian_2d(4, 4);
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_graph(a, 2, 0.1));
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
        const std::vector<double> z = p.apply_neumann(std::vector<double>{1.0, 0.0}, 1);
        EXPECT(z[0] == 0.5 && z[1] == -0.25);
        bool thrown = false;
        try {
            p.apply_neumann(std::vector<double>{1.0, 0.0}, 2);
        } catch (const std::invalid_argument&) {
            thrown = true;
        }
        EXPECT(thrown);
    }
    {  // block diagnostics: cond >= 1 and the bound formula (preconditioner.cpp:13-15)
        const SparseMatrix a = laplacian_2d(8, 8);
        const Preconditioner p = Preconditioner::block_jacobi(a, partition_graph(a, 4, 0.1));
        for (const auto& st : p.stats()) {
            EXPECT(st.cond_estimate >= 1.0);
            EXPECT(std::abs(st.error_bound - (st.cond_estimate * 0x1p-53 + 0x1p-24) * st.cond_estimate) <=
                   1e-12 * st.error_bound);
        }
    }
    {  // ILU(0) and identity behind the same solve (DoubleOnly), Hybrid ILU(0) throws like the reference
        const SparseMatrix a = laplacian_2d(16, 16);
        const std::vector<double> b = matvec(a, std::vector<double>(a.rows(), 1.0));
        GmresConfig cfg;
        cfg.restart_m = 30;
        cfg.tol = 1e-10;
        cfg.policy.mode = PrecisionMode::DoubleOnly;
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
        const std::vector<double> z = ilu.apply(b);
        EXPECT(z.size() == b.size());
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
