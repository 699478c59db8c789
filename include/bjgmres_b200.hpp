// bjgmres_b200.hpp — header-only C++ mirror of the reference solver API
// (/root/reference/proj/include/bjgmres) on top of the hpbj C ABI
// (include/hpbj.h, libhpbj.so). A caller of the reference — e.g. run_spec in
// bjgmres_cli.cpp:112-168 — switches by including this header instead of
// bjgmres/{sparse_matrix,graph,partition,preconditioner,gmres}.hpp and
// linking libhpbj.so: names, argument meaning and exception types match.
//
// Differences a caller can observe: the block-Jacobi
// preconditioner is the Hybrid (FP32) one and lives on a GPU, so
// GmresConfig::policy defaults to Hybrid here (DoubleOnly serves the FP64
// ILU(0) and identity preconditioners); the matrix passed to
// hybrid_restart_gmres must be the one the preconditioner was built from (it
// is device-resident).
#pragma once

#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hpbj.h"

namespace bjgmres_b200 {

using index_t = std::int64_t;

class SingularBlockError : public std::runtime_error {  // lu.hpp:52-60
public:
    SingularBlockError(const std::string& what, index_t column) : std::runtime_error(what), column_(column) {}
    index_t column() const { return column_; }

private:
    index_t column_;
};

namespace detail {
// The message is fetched only after the call has returned (rc is an argument,
// so it is evaluated before check runs): ctx == nullptr selects the calling
// thread's last context-free error.
inline void check(int rc, const hpbj_ctx* ctx, index_t column = -1) {
    if (rc == HPBJ_OK) return;
    const std::string m = hpbj_last_error(ctx);
    const char* msg = m.c_str();
    switch (rc) {
        case HPBJ_OK: return;
        case HPBJ_EINVAL: throw std::invalid_argument(msg);
        case HPBJ_ELOGIC: throw std::logic_error(msg);
        case HPBJ_ERANGE: throw std::out_of_range(msg);
        case HPBJ_ESINGULAR: throw SingularBlockError(msg, column);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace detail

// SparseMatrix (sparse_matrix.hpp:23-62): host CSR, FP64 master values.
class SparseMatrix {
public:
    SparseMatrix() = default;
    SparseMatrix(index_t nrows, index_t ncols, std::vector<index_t> row_starts, std::vector<index_t> col_indices,
                 std::vector<double> values)
        : n_(nrows), rs_(std::move(row_starts)), ci_(std::move(col_indices)), v_(std::move(values)) {
        if (nrows != ncols) throw std::invalid_argument("sparse matrix: must be square for this solver");
    }
    index_t rows() const { return n_; }
    index_t cols() const { return n_; }
    index_t nnz() const { return static_cast<index_t>(v_.size()); }
    std::span<const index_t> row_starts() const { return rs_; }
    std::span<const index_t> col_indices() const { return ci_; }
    std::span<const double> values() const { return v_; }
    void materialize_low() {}  // factors/values are cast on the device

private:
    index_t n_ = 0;
    std::vector<index_t> rs_{0}, ci_;
    std::vector<double> v_;
};

// Partition (partition.hpp:14-28)
struct Partition {
    index_t num_blocks = 0;
    std::vector<index_t> assignment, perm, block_starts;
    index_t num_nodes() const { return static_cast<index_t>(assignment.size()); }
    index_t block_size(index_t b) const { return block_starts[b + 1] - block_starts[b]; }
};

// graph_from_matrix + partition_graph (graph.hpp:30, partition.hpp:38-39),
// fused: the host partitioner works on the CSR directly.
inline Partition partition_graph(const SparseMatrix& a, index_t s, double imbalance_tol = 0.1) {
    Partition p;
    p.num_blocks = s;
    p.assignment.resize(a.rows());
    p.perm.resize(a.rows());
    p.block_starts.resize(s + 1);
    detail::check(hpbj_partition_graph(a.rows(), a.row_starts().data(), a.col_indices().data(), a.values().data(), s,
                                       imbalance_tol, p.assignment.data(), p.perm.data(), p.block_starts.data()),
                  nullptr);
    return p;
}

inline Partition partition_from_assignment(std::vector<index_t> assignment, index_t s) {
    Partition p;
    p.num_blocks = s;
    p.perm.resize(assignment.size());
    p.block_starts.resize(s + 1);
    detail::check(hpbj_partition_from_assignment(static_cast<index_t>(assignment.size()), assignment.data(), s,
                                                 p.perm.data(), p.block_starts.data()),
                  nullptr);
    p.assignment = std::move(assignment);
    return p;
}

struct BlockJacobiOptions {  // preconditioner.hpp:32-38 (Hybrid policy)
    double eps_pivot = 1e-10;
    int neumann_order = 0;  // 0 = direct block solves (preconditioner.hpp:34)
};

struct PreconditionerStats {  // preconditioner.hpp:14-20 (block_nnz: see measure_block_nnz)
    index_t block_dim = 0;
    index_t perturbation_count = 0;
    double cond_estimate = 0.0;  // cond_estimate_block (computed on the device when requested)
    double error_bound = 0.0;    // block_error_bound(cond, 2^-24, 2^-53)
};

// Preconditioner (preconditioner.hpp:50-98): cheap copyable handle to an
// immutable device-resident factorisation.
class Preconditioner {
public:
    enum class Kind { Identity, Ilu0, BlockJacobi };  // preconditioner.hpp:55

    static Preconditioner identity(index_t n) {  // bound to the matrix by the solve
        Preconditioner p;
        p.kind_ = Kind::Identity;
        p.n_ = n;
        return p;
    }
    // Preconditioner::from_ilu0 (preconditioner.cpp:94-98): FP64 ILU(0) factors on the device
    static Preconditioner from_ilu0(const SparseMatrix& a, int device = 0) {
        Preconditioner p;
        hpbj_ctx* raw = nullptr;
        detail::check(hpbj_create(&raw, device), nullptr);
        p.ctx_ = std::shared_ptr<hpbj_ctx>(raw, hpbj_destroy);
        detail::check(hpbj_set_matrix(raw, a.rows(), a.row_starts().data(), a.col_indices().data(), a.values().data()),
                      raw);
        detail::check(hpbj_ilu0_setup(raw, nullptr), raw);
        p.kind_ = Kind::Ilu0;
        p.n_ = a.rows();
        p.matrix_ = &a;
        return p;
    }
    Kind kind() const { return kind_; }

    static Preconditioner block_jacobi(const SparseMatrix& a, Partition partition,
                                       const BlockJacobiOptions& opts = {}, int device = 0) {
        if (partition.num_nodes() != a.rows())
            throw std::invalid_argument("block_jacobi: partition does not cover the matrix");
        Preconditioner p;
        hpbj_ctx* raw = nullptr;
        detail::check(hpbj_create(&raw, device), nullptr);
        p.ctx_ = std::shared_ptr<hpbj_ctx>(raw, hpbj_destroy);
        detail::check(hpbj_bj_set_neumann_order(raw, opts.neumann_order), raw);
        detail::check(hpbj_set_matrix(raw, a.rows(), a.row_starts().data(), a.col_indices().data(), a.values().data()),
                      raw);
        hpbj_setup_info info{};
        const int rc = hpbj_bj_setup(raw, partition.num_blocks, partition.perm.data(), partition.block_starts.data(),
                                     opts.eps_pivot, &info);
        detail::check(rc, raw, info.singular_column);
        p.n_ = a.rows();
        p.neumann_ = opts.neumann_order;
        p.matrix_ = &a;
        p.partition_ = std::make_shared<const Partition>(std::move(partition));
        return p;
    }
    index_t dim() const { return n_; }
    const Partition& partition() const { return *partition_; }

    // apply (preconditioner.hpp:69-70): z with M z = v — apply<float> for
    // block Jacobi, apply<double> for ILU(0) and the identity
    std::vector<double> apply(std::span<const double> v) const {
        if (static_cast<index_t>(v.size()) != n_)
            throw std::invalid_argument("preconditioner apply: dimension mismatch");
        if (kind_ == Kind::Identity) return std::vector<double>(v.begin(), v.end());
        std::vector<double> z(n_);
        detail::check(hpbj_precond_apply(ctx_.get(), v.data(), z.data()), ctx_.get());
        return z;
    }
    int neumann_order() const { return neumann_; }
    // apply_neumann<float> (preconditioner.hpp:79-83) on the matrix the
    // preconditioner was built from: z = sum_{i<=k} (I - Phi^-1 A)^i Phi^-1 v
    std::vector<double> apply_neumann(std::span<const double> v, int k) const {
        if (static_cast<index_t>(v.size()) != n_)
            throw std::invalid_argument("preconditioner apply: dimension mismatch");
        std::vector<double> z(n_);
        detail::check(hpbj_bj_apply_neumann(ctx_.get(), v.data(), z.data(), k), ctx_.get());
        return z;
    }
    std::vector<PreconditionerStats> stats(bool with_cond_estimates = true) const {
        if (kind_ != Kind::BlockJacobi) throw std::logic_error("stats: block-Jacobi preconditioner not set up");
        const size_t s = static_cast<size_t>(partition_->num_blocks);
        std::vector<index_t> d(s), pc(s);
        std::vector<double> cond(s, 0.0), eb(s, 0.0);
        detail::check(hpbj_get_block_stats(ctx_.get(), d.data(), pc.data()), ctx_.get());
        if (with_cond_estimates)
            detail::check(hpbj_get_block_diagnostics(ctx_.get(), cond.data(), eb.data()), ctx_.get());
        std::vector<PreconditionerStats> out(s);
        for (size_t b = 0; b < s; ++b) out[b] = {d[b], pc[b], cond[b], eb[b]};
        return out;
    }
    hpbj_ctx* context() const { return ctx_.get(); }
    const SparseMatrix* matrix() const { return matrix_; }

private:
    std::shared_ptr<hpbj_ctx> ctx_;
    std::shared_ptr<const Partition> partition_;
    const SparseMatrix* matrix_ = nullptr;
    index_t n_ = 0;
    int neumann_ = 0;
    Kind kind_ = Kind::BlockJacobi;
};

enum class PrecisionMode { DoubleOnly, Hybrid };  // types.hpp:15-26
struct PrecisionPolicy {
    PrecisionMode mode = PrecisionMode::Hybrid;  // the reference defaults to DoubleOnly (see the header note)
    bool hybrid() const { return mode == PrecisionMode::Hybrid; }
    double working_roundoff() const { return hybrid() ? 0x1p-24 : 0x1p-53; }
};

struct GmresConfig {  // gmres.hpp:89-97
    index_t restart_m = 50;
    double tol = 1e-8;
    index_t max_restarts = 40;
    bool absolute_tol = false;
    PrecisionPolicy policy{};
    double breakdown_tol_factor = 1e2;
};

struct HistoryPoint {  // gmres.hpp:99-103
    index_t cycle;
    index_t iteration;
    double relative_residual;
};

struct SolveReport {  // gmres.hpp:105-117
    bool converged = false;
    index_t total_iterations = 0;
    index_t restarts = 0;
    std::vector<HistoryPoint> residual_history;
    std::vector<double> cycle_residuals;
    double final_residual = 0.0;
    bool breakdown = false;
    bool ls_rank_deficient = false;
    double setup_seconds = 0.0;
    double iterate_seconds = 0.0;
};

struct SolveResult {
    std::vector<double> x;
    SolveReport report;
};

// hybrid_restart_gmres (gmres.hpp:145-147)
inline SolveResult hybrid_restart_gmres(const SparseMatrix& a, const Preconditioner& p, std::span<const double> b,
                                        const GmresConfig& config) {
    if (static_cast<index_t>(b.size()) != a.rows()) throw std::invalid_argument("gmres: rhs dimension mismatch");
    if (config.restart_m < 1 || config.tol <= 0.0 || config.max_restarts < 1)
        throw std::invalid_argument("gmres: invalid config");
    hpbj_ctx* ctx = p.context();
    std::shared_ptr<hpbj_ctx> bound;
    if (p.kind() == Preconditioner::Kind::Identity) {  // identity: a context for this matrix
        hpbj_ctx* raw = nullptr;
        detail::check(hpbj_create(&raw, 0), nullptr);
        bound = std::shared_ptr<hpbj_ctx>(raw, hpbj_destroy);
        detail::check(hpbj_set_matrix(raw, a.rows(), a.row_starts().data(), a.col_indices().data(), a.values().data()),
                      raw);
        detail::check(hpbj_identity_setup(raw), raw);
        ctx = raw;
    } else if (p.matrix() != &a) {
        throw std::invalid_argument("gmres: preconditioner was built from another matrix");
    }
    if (p.kind() == Preconditioner::Kind::Ilu0 && config.policy.hybrid())  // lu_solve<float> on FP64-only factors
        throw std::logic_error("values_low requested before materialize_low()");
    if (p.kind() == Preconditioner::Kind::BlockJacobi && !config.policy.hybrid())
        throw std::invalid_argument("gmres: DoubleOnly block Jacobi is not implemented on the GPU path");
    hpbj_gmres_opts o;
    hpbj_gmres_default_opts(&o);
    o.restart_m = config.restart_m;
    o.tol = config.tol;
    o.max_restarts = config.max_restarts;
    o.absolute_tol = config.absolute_tol ? 1 : 0;
    o.breakdown_tol_factor = config.breakdown_tol_factor;
    o.floor_roundoff = config.policy.working_roundoff();
    SolveResult out;
    out.x.resize(a.rows());
    std::vector<hpbj_history_point> hist(config.restart_m * config.max_restarts + 2);
    std::vector<double> cyc(config.max_restarts + 1);
    hpbj_report rep{};
    detail::check(hpbj_gmres(ctx, b.data(), out.x.data(), &o, &rep, hist.data(), static_cast<int64_t>(hist.size()),
                             cyc.data(), static_cast<int64_t>(cyc.size())),
                  ctx);
    SolveReport& r = out.report;
    r.converged = rep.converged != 0;
    r.total_iterations = rep.total_iterations;
    r.restarts = rep.restarts;
    r.final_residual = rep.final_residual;
    r.breakdown = rep.breakdown != 0;
    r.ls_rank_deficient = rep.ls_rank_deficient != 0;
    r.iterate_seconds = rep.ms_solve * 1e-3;
    for (int64_t k = 0; k < rep.history_len && k < static_cast<int64_t>(hist.size()); ++k)
        r.residual_history.push_back({hist[k].cycle, hist[k].iteration, hist[k].relative_residual});
    r.cycle_residuals.assign(cyc.begin(), cyc.begin() + std::min<int64_t>(rep.cycles, cyc.size()));
    return out;
}

}  // namespace bjgmres_b200
