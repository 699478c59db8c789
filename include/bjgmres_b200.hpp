// bjgmres_b200.hpp — the reference solver API (/root/reference/proj/include/
// bjgmres: namespace bjgmres, same type and function names, argument meaning
// and exception types) implemented over the hpbj C ABI (include/hpbj.h,
// libhpbj.so). A caller of the reference switches by putting this repo's
// include/ on the include path instead of proj/include — the forwarding
// headers include/bjgmres/{types,sparse_matrix,spmv,graph,partition,lu,
// preconditioner,gmres,matrix_market}.hpp keep its #include lines valid — and
// linking libhpbj.so. tests/cpp/test_run_spec.cpp compiles the body of the
// reference's run_spec (bjgmres_cli.cpp:112-168) against it unchanged.
//
// Ownership: SparseMatrix is a value type whose CSR payload is immutable and
// shared by copies (the reference exposes no mutator). A Preconditioner is a
// cheap copyable handle to an immutable device factorisation; it owns a
// shared_ptr to the payload it was built from and to a pooled device context
// (its own CUDA stream, memory pool and solve graph), which goes back to a
// per-process pool when the last handle dies, so a caller that rebuilds a
// preconditioner per step (config 4's Newton sequence) reuses the context:
// same pattern -> only the values are re-uploaded, same partition -> only the
// numeric refactorisation runs.
//
// Differences a caller can observe:
//  * PrecisionPolicy defaults to Hybrid (the reference: DoubleOnly). The GPU
//    block-Jacobi factors are FP32 (the Hybrid ones); a DoubleOnly solve with
//    block Jacobi throws std::invalid_argument. DoubleOnly serves ILU(0) and
//    the identity, whose applies run in FP64 on the device.
//  * The Krylov loop runs in FP64 with the FP32 preconditioner (north star);
//    the attainable-floor break uses 2^-24 as the reference Hybrid does.
//  * BlockJacobiData::factors holds each block's FP32 factors (widened to
//    double), fetched from the device on first access; exact zeros of the
//    dense device factors are dropped, so the sparsity can be smaller than
//    the reference's structural pattern. cond_estimate / error_bound are
//    computed on the device when first read.
//  * GmresConfig::collect_ritz = true throws std::invalid_argument (Ritz
//    values are a diagnostic that this build does not compute).
//  * hybrid_restart_gmres accepts any matrix with the preconditioner's
//    sparsity pattern (new values are uploaded, the factors stay — a lagged
//    preconditioner, as in the reference); a different pattern throws
//    std::invalid_argument.
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <istream>
#include <memory>
#include <mutex>
#include <optional>
#include <ostream>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <unistd.h>

#include "hpbj.h"

namespace bjgmres {

// ---------------------------------------------------------------- types.hpp
using index_t = std::int64_t;

enum class Norm { Two, Inf, One };

inline constexpr double kRoundoffSingle = 0x1p-24;
inline constexpr double kRoundoffDouble = 0x1p-53;

enum class PrecisionMode { DoubleOnly, Hybrid };

struct PrecisionPolicy {  // types.hpp:17-26 (default: see the header note)
    PrecisionMode mode = PrecisionMode::Hybrid;
    bool hybrid() const { return mode == PrecisionMode::Hybrid; }
    double working_roundoff() const { return hybrid() ? kRoundoffSingle : kRoundoffDouble; }
};

// ------------------------------------------------------------------ lu.hpp
class SingularBlockError : public std::runtime_error {  // lu.hpp:52-60
public:
    SingularBlockError(const std::string& what, index_t column) : std::runtime_error(what), column_(column) {}
    index_t column() const { return column_; }

private:
    index_t column_;
};

namespace detail {

// Status code -> the reference's exception type. The message is read after
// the call returned; ctx == nullptr selects the calling thread's last
// context-free error.
inline void check(int rc, const hpbj_ctx* ctx, index_t column = -1) {
    if (rc == HPBJ_OK) return;
    const std::string msg = hpbj_last_error(ctx);
    switch (rc) {
        case HPBJ_EINVAL: throw std::invalid_argument(msg);
        case HPBJ_ELOGIC: throw std::logic_error(msg);
        case HPBJ_ERANGE: throw std::out_of_range(msg);
        case HPBJ_ESINGULAR: throw SingularBlockError(msg, column);
        default: throw std::runtime_error(msg);
    }
}

// Immutable CSR payload of a SparseMatrix, shared by its copies.
struct Csr {
    index_t nrows = 0, ncols = 0;
    std::vector<index_t> rs{0}, ci;
    std::vector<double> v;
    mutable std::once_flag low_once;
    mutable std::vector<float> low;  // values_low(), derived on first use
};

inline bool same_pattern(const Csr& a, const Csr& b) {
    if (&a == &b) return true;
    return a.nrows == b.nrows && a.ncols == b.ncols && a.ci.size() == b.ci.size() &&
           std::memcmp(a.rs.data(), b.rs.data(), sizeof(index_t) * a.rs.size()) == 0 &&
           (a.ci.empty() || std::memcmp(a.ci.data(), b.ci.data(), sizeof(index_t) * a.ci.size()) == 0);
}

}  // namespace detail

// ------------------------------------------------------- sparse_matrix.hpp
struct Triplet {
    index_t row;
    index_t col;
    double value;
};

class SparseMatrix {  // sparse_matrix.hpp:23-62
public:
    SparseMatrix() : d_(std::make_shared<detail::Csr>()) {}
    SparseMatrix(index_t nrows, index_t ncols, std::vector<index_t> row_starts, std::vector<index_t> col_indices,
                 std::vector<double> values) {
        // invariants of sparse_matrix.cpp:14-35, same messages
        if (nrows < 0 || ncols < 0) throw std::invalid_argument("sparse matrix: negative dimension");
        if (row_starts.size() != static_cast<size_t>(nrows) + 1)
            throw std::invalid_argument("sparse matrix: row_starts length");
        if (row_starts.front() != 0 || row_starts.back() != static_cast<index_t>(col_indices.size()) ||
            col_indices.size() != values.size())
            throw std::invalid_argument("sparse matrix: inconsistent sizes");
        for (index_t i = 0; i < nrows; ++i) {
            if (row_starts[i] > row_starts[i + 1])
                throw std::invalid_argument("sparse matrix: row_starts not non-decreasing");
            for (index_t k = row_starts[i]; k < row_starts[i + 1]; ++k) {
                if (col_indices[k] < 0 || col_indices[k] >= ncols)
                    throw std::invalid_argument("sparse matrix: column index out of range");
                if (k > row_starts[i] && col_indices[k - 1] >= col_indices[k])
                    throw std::invalid_argument("sparse matrix: columns not strictly increasing");
            }
        }
        auto d = std::make_shared<detail::Csr>();
        d->nrows = nrows;
        d->ncols = ncols;
        d->rs = std::move(row_starts);
        d->ci = std::move(col_indices);
        d->v = std::move(values);
        d_ = std::move(d);
    }

    // sparse_matrix.cpp:52-88: sort by (row, col, value bits), sum duplicates
    // in that canonical order
    static SparseMatrix from_triplets(std::span<const Triplet> triplets, index_t nrows, index_t ncols) {
        for (const Triplet& t : triplets)
            if (t.row < 0 || t.row >= nrows || t.col < 0 || t.col >= ncols)
                throw std::out_of_range("from_triplets: index (" + std::to_string(t.row) + ", " +
                                        std::to_string(t.col) + ") out of range");
        std::vector<Triplet> s(triplets.begin(), triplets.end());
        std::sort(s.begin(), s.end(), [](const Triplet& a, const Triplet& b) {
            if (a.row != b.row) return a.row < b.row;
            if (a.col != b.col) return a.col < b.col;
            return std::bit_cast<std::uint64_t>(a.value) < std::bit_cast<std::uint64_t>(b.value);
        });
        std::vector<index_t> rs(nrows + 1, 0), ci;
        std::vector<double> v;
        ci.reserve(s.size());
        v.reserve(s.size());
        for (size_t k = 0; k < s.size();) {
            const index_t r = s[k].row, c = s[k].col;
            double sum = 0.0;
            while (k < s.size() && s[k].row == r && s[k].col == c) sum += s[k++].value;
            ci.push_back(c);
            v.push_back(sum);
            rs[r + 1] = static_cast<index_t>(ci.size());
        }
        for (index_t i = 0; i < nrows; ++i) rs[i + 1] = std::max(rs[i + 1], rs[i]);
        return SparseMatrix(nrows, ncols, std::move(rs), std::move(ci), std::move(v));
    }

    index_t rows() const { return d_->nrows; }
    index_t cols() const { return d_->ncols; }
    index_t nnz() const { return static_cast<index_t>(d_->v.size()); }
    std::span<const index_t> row_starts() const { return d_->rs; }
    std::span<const index_t> col_indices() const { return d_->ci; }
    std::span<const double> values() const { return d_->v; }

    // The device path down-casts on load; the host FP32 copy is derived on
    // first use of values_low().
    void materialize_low() { low_ = true; }
    bool has_low() const { return low_; }
    std::span<const float> values_low() const {
        if (!low_) throw std::logic_error("values_low requested before materialize_low()");
        std::call_once(d_->low_once, [&] {
            d_->low.resize(d_->v.size());
            for (size_t k = 0; k < d_->v.size(); ++k) d_->low[k] = static_cast<float>(d_->v[k]);
        });
        return d_->low;
    }
    template <class T>
    std::span<const T> values_as() const;

    double value_at(index_t i, index_t j) const {  // sparse_matrix.cpp:103-112
        if (i < 0 || i >= rows() || j < 0 || j >= cols()) throw std::out_of_range("value_at: index out of range");
        const auto first = d_->ci.begin() + d_->rs[i], last = d_->ci.begin() + d_->rs[i + 1];
        const auto it = std::lower_bound(first, last, j);
        return (it == last || *it != j) ? 0.0 : d_->v[static_cast<size_t>(it - d_->ci.begin())];
    }

    // identity of the (immutable) payload: device contexts cache by it
    const std::shared_ptr<const detail::Csr>& payload() const { return d_; }

private:
    std::shared_ptr<const detail::Csr> d_;
    bool low_ = false;
};

template <>
inline std::span<const double> SparseMatrix::values_as<double>() const {
    return values();
}
template <>
inline std::span<const float> SparseMatrix::values_as<float>() const {
    return values_low();
}

// permute_symmetric (sparse_matrix.cpp:113-153): B[p(i), p(j)] = A[i, j]
inline SparseMatrix permute_symmetric(const SparseMatrix& a, std::span<const index_t> perm) {
    const index_t n = a.rows();
    if (a.cols() != n) throw std::invalid_argument("permute_symmetric: matrix must be square");
    if (static_cast<index_t>(perm.size()) != n) throw std::invalid_argument("permute_symmetric: permutation length");
    std::vector<bool> seen(n, false);
    for (index_t p : perm) {
        if (p < 0 || p >= n || seen[p]) throw std::invalid_argument("permute_symmetric: not a bijection");
        seen[p] = true;
    }
    const auto rs = a.row_starts();
    const auto ci = a.col_indices();
    const auto v = a.values();
    std::vector<index_t> nrs(n + 1, 0);
    for (index_t i = 0; i < n; ++i) nrs[perm[i] + 1] = rs[i + 1] - rs[i];
    for (index_t i = 0; i < n; ++i) nrs[i + 1] += nrs[i];
    std::vector<index_t> nci(a.nnz());
    std::vector<double> nv(a.nnz());
    std::vector<std::pair<index_t, double>> row;
    for (index_t i = 0; i < n; ++i) {
        row.clear();
        for (index_t k = rs[i]; k < rs[i + 1]; ++k) row.emplace_back(perm[ci[k]], v[k]);
        std::sort(row.begin(), row.end());
        index_t d = nrs[perm[i]];
        for (const auto& [c, x] : row) {
            nci[d] = c;
            nv[d++] = x;
        }
    }
    return SparseMatrix(n, n, std::move(nrs), std::move(nci), std::move(nv));
}

inline double matrix_inf_norm(const SparseMatrix& a) {  // sparse_matrix.cpp:155-166
    const auto rs = a.row_starts();
    const auto v = a.values();
    double norm = 0.0;
    for (index_t i = 0; i < a.rows(); ++i) {
        double s = 0.0;
        for (index_t k = rs[i]; k < rs[i + 1]; ++k) s += std::abs(v[k]);
        norm = std::max(norm, s);
    }
    return norm;
}

inline double matrix_one_norm(const SparseMatrix& a) {  // sparse_matrix.cpp:168-176
    std::vector<double> cs(a.cols(), 0.0);
    const auto ci = a.col_indices();
    const auto v = a.values();
    for (index_t k = 0; k < a.nnz(); ++k) cs[ci[k]] += std::abs(v[k]);
    double norm = 0.0;
    for (double s : cs) norm = std::max(norm, s);
    return norm;
}

// ------------------------------------------------------ device contexts
namespace detail {

// A device context plus what it currently holds. Contexts go back to a
// per-process pool when their last user is gone (see the header note).
struct DeviceCtx {
    hpbj_ctx* ctx = nullptr;
    int device = 0;
    std::shared_ptr<const Csr> mat;          // matrix resident on the device
    std::vector<index_t> perm, block_starts;  // partition of the resident factors
    double eps = -1.0;
    int neumann = 0;
    bool bj = false;                          // block-Jacobi factors resident
};

class CtxPool {
public:
    static CtxPool& get() {
        static CtxPool p;
        return p;
    }
    std::unique_ptr<DeviceCtx> take(int device) {
        {
            std::lock_guard<std::mutex> g(mu_);
            for (size_t i = idle_.size(); i-- > 0;)
                if (idle_[i]->device == device) {
                    std::unique_ptr<DeviceCtx> c = std::move(idle_[i]);
                    idle_.erase(idle_.begin() + static_cast<std::ptrdiff_t>(i));
                    return c;
                }
        }
        auto c = std::make_unique<DeviceCtx>();
        c->device = device;
        check(hpbj_create(&c->ctx, device), nullptr);
        return c;
    }
    void give(std::unique_ptr<DeviceCtx> c) {
        if (!c || !c->ctx) return;
        std::lock_guard<std::mutex> g(mu_);
        idle_.push_back(std::move(c));
        while (idle_.size() > kMaxIdle) {
            hpbj_destroy(idle_.front()->ctx);
            idle_.erase(idle_.begin());
        }
    }
    ~CtxPool() {
        for (auto& c : idle_) hpbj_destroy(c->ctx);
    }

private:
    static constexpr size_t kMaxIdle = 4;
    std::mutex mu_;
    std::vector<std::unique_ptr<DeviceCtx>> idle_;
};

struct CtxLease {  // RAII: a context from the pool, returned on destruction
    std::unique_ptr<DeviceCtx> c;
    explicit CtxLease(int device) : c(CtxPool::get().take(device)) {}
    ~CtxLease() { CtxPool::get().give(std::move(c)); }
    CtxLease(const CtxLease&) = delete;
    CtxLease& operator=(const CtxLease&) = delete;
};

// Make `a` the matrix resident in c: nothing if it already is, new values
// if the pattern matches (factors are kept), else a full upload (which drops
// any factors; allow_new_pattern = false turns that case into an error).
inline void bind_matrix(DeviceCtx& c, const std::shared_ptr<const Csr>& a, bool allow_new_pattern) {
    if (c.mat == a) return;
    if (c.mat && same_pattern(*c.mat, *a)) {
        check(hpbj_update_values(c.ctx, a->v.data()), c.ctx);
        c.mat = a;
        return;
    }
    if (!allow_new_pattern)
        throw std::invalid_argument(
            "gmres: the matrix's sparsity pattern differs from the one the preconditioner was built from");
    check(hpbj_set_matrix(c.ctx, a->nrows, a->rs.data(), a->ci.data(), a->v.data()), c.ctx);
    c.mat = a;
    c.bj = false;
    c.perm.clear();
    c.block_starts.clear();
}

// A context holding `a` for stand-alone device operations (spmv<T>, the
// identity preconditioner): the most recently used one is kept.
inline std::shared_ptr<CtxLease> matrix_ctx(const std::shared_ptr<const Csr>& a) {
    static std::mutex mu;
    static std::shared_ptr<CtxLease> last;
    std::lock_guard<std::mutex> g(mu);
    if (!last || last->c->mat != a) {
        auto l = std::make_shared<CtxLease>(0);
        bind_matrix(*l->c, a, true);
        last = l;
    }
    return last;
}

}  // namespace detail

// --------------------------------------------------------------- spmv.hpp
// spmv<T> (spmv.hpp:31-53) on the device: FP64 CSR SpMV (x widened, y
// rounded to T for T = float).
template <class T>
void spmv(const SparseMatrix& a, std::span<const T> x, std::span<T> y) {
    if (static_cast<index_t>(x.size()) != a.cols() || static_cast<index_t>(y.size()) != a.rows())
        throw std::invalid_argument("spmv: dimension mismatch");
    if (a.rows() != a.cols()) throw std::invalid_argument("spmv: matrix must be square on the device path");
    if constexpr (std::is_same_v<T, float>) (void)a.values_low();  // same precondition as values_as<float>
    const auto lease = detail::matrix_ctx(a.payload());
    std::vector<double> xd(x.begin(), x.end()), yd(a.rows());
    detail::check(hpbj_spmv(lease->c->ctx, xd.data(), yd.data()), lease->c->ctx);
    for (index_t i = 0; i < a.rows(); ++i) y[i] = static_cast<T>(yd[i]);
}
template <class T>
void spmv_serial(const SparseMatrix& a, std::span<const T> x, std::span<T> y) {
    spmv<T>(a, x, y);  // rows are independent: same result
}
template <class T>
std::vector<T> spmv(const SparseMatrix& a, std::span<const T> x) {
    std::vector<T> y(a.rows());
    spmv<T>(a, x, y);
    return y;
}

// -------------------------------------------------------------- graph.hpp
struct WeightedEdge {
    index_t neighbor;
    double weight;
};

// WeightedGraph::adjacency: the adjacency lists of graph_from_matrix,
// materialised (hpbj_graph_from_matrix, bit-identical weights) only when a
// caller reads them; partition_graph of an unread graph partitions the CSR
// directly (the O(nnz) host partitioner, no per-node vectors).
class AdjacencyLists {
public:
    using value_type = std::vector<WeightedEdge>;
    AdjacencyLists() = default;
    explicit AdjacencyLists(std::shared_ptr<const detail::Csr> src)
        : src_(std::move(src)), once_(std::make_shared<std::once_flag>()) {}

    size_t size() const { return src_ ? static_cast<size_t>(src_->nrows) : lists_.size(); }
    bool empty() const { return size() == 0; }
    const value_type& operator[](size_t i) const { return built()[i]; }
    value_type& operator[](size_t i) { return own()[i]; }
    auto begin() const { return built().cbegin(); }
    auto end() const { return built().cend(); }
    auto begin() { return own().begin(); }
    auto end() { return own().end(); }
    void resize(size_t n) { own().resize(n); }
    void reserve(size_t n) { own().reserve(n); }
    void clear() { own().clear(); }
    void push_back(value_type v) { own().push_back(std::move(v)); }
    const value_type& at(size_t i) const { return built().at(i); }

    // CSR of the graph_from_matrix source while the lists are unread
    const detail::Csr* lazy_source() const { return (src_ && !materialised_) ? src_.get() : nullptr; }

private:
    const std::vector<value_type>& built() const {
        if (src_)
            std::call_once(*once_, [&] {
                const index_t n = src_->nrows;
                const index_t cap = 2 * static_cast<index_t>(src_->ci.size()) + 1;
                std::vector<index_t> st(n + 1), nb(cap);
                std::vector<double> w(cap);
                detail::check(hpbj_graph_from_matrix(n, src_->rs.data(), src_->ci.data(), src_->v.data(), st.data(),
                                                     nb.data(), w.data(), cap),
                              nullptr);
                lists_.assign(n, {});
                for (index_t u = 0; u < n; ++u) {
                    lists_[u].reserve(st[u + 1] - st[u]);
                    for (index_t k = st[u]; k < st[u + 1]; ++k) lists_[u].push_back({nb[k], w[k]});
                }
                materialised_ = true;
            });
        return lists_;
    }
    std::vector<value_type>& own() {  // a mutation detaches the lists from the source
        built();
        src_.reset();
        return lists_;
    }

    std::shared_ptr<const detail::Csr> src_;
    std::shared_ptr<std::once_flag> once_;
    mutable std::vector<value_type> lists_;
    mutable bool materialised_ = false;
};

struct WeightedGraph {  // graph.hpp:17-25
    index_t num_nodes = 0;
    AdjacencyLists adjacency;
    index_t degree(index_t v) const { return static_cast<index_t>(adjacency[v].size()); }
    index_t num_edges() const {
        index_t twice = 0;
        for (const auto& l : adjacency) twice += static_cast<index_t>(l.size());
        return twice / 2;
    }
};

// graph_from_matrix (graph.hpp:30, graph.cpp:17-51)
inline WeightedGraph graph_from_matrix(const SparseMatrix& a) {
    if (a.cols() != a.rows()) throw std::invalid_argument("graph_from_matrix: matrix must be square");
    WeightedGraph g;
    g.num_nodes = a.rows();
    g.adjacency = AdjacencyLists(a.payload());
    return g;
}

// ---------------------------------------------------------- partition.hpp
struct Partition {  // partition.hpp:14-28
    index_t num_blocks = 0;
    std::vector<index_t> assignment;    // node -> block
    std::vector<index_t> perm;          // old index -> new index
    std::vector<index_t> block_starts;  // size num_blocks + 1, over new indices
    std::vector<index_t> block_nnz;     // filled by measure_block_nnz
    double imbalance = 0.0;             // max block_nnz / mean block_nnz

    index_t num_nodes() const { return static_cast<index_t>(assignment.size()); }
    index_t block_size(index_t b) const { return block_starts[b + 1] - block_starts[b]; }
};

// partition_from_assignment (partition.hpp:33, partition.cpp:14-41)
inline Partition partition_from_assignment(std::vector<index_t> assignment, index_t s) {
    Partition p;
    p.num_blocks = s;
    p.perm.resize(assignment.size());
    p.block_starts.resize(static_cast<size_t>(std::max<index_t>(s, 0)) + 1);
    detail::check(hpbj_partition_from_assignment(static_cast<index_t>(assignment.size()), assignment.data(), s,
                                                 p.perm.data(), p.block_starts.data()),
                  nullptr);
    p.assignment = std::move(assignment);
    p.block_nnz.assign(s, 0);
    return p;
}

namespace detail {
inline Partition finish_partition(std::vector<index_t> assignment, std::vector<index_t> perm,
                                  std::vector<index_t> bst, index_t s) {
    Partition p;
    p.num_blocks = s;
    p.assignment = std::move(assignment);
    p.perm = std::move(perm);
    p.block_starts = std::move(bst);
    p.block_nnz.assign(s, 0);
    return p;
}
}  // namespace detail

// partition_graph (partition.hpp:38-39, partition.cpp:60-144), bit-identical
inline Partition partition_graph(const WeightedGraph& g, index_t s, double imbalance_tol = 0.1) {
    const index_t n = g.num_nodes;
    if (s < 1) throw std::invalid_argument("partition_graph: s must be >= 1");
    if (s > n) throw std::invalid_argument("partition_graph: s exceeds node count");
    if (imbalance_tol < 0.0) throw std::invalid_argument("partition_graph: negative imbalance tolerance");
    std::vector<index_t> asg(n), perm(n), bst(s + 1);
    if (const detail::Csr* c = g.adjacency.lazy_source(); c && c->nrows == n) {
        detail::check(hpbj_partition_graph(n, c->rs.data(), c->ci.data(), c->v.data(), s, imbalance_tol, asg.data(),
                                           perm.data(), bst.data()),
                      nullptr);
    } else {
        if (static_cast<index_t>(g.adjacency.size()) != n)
            throw std::invalid_argument("partition_graph: adjacency size differs from num_nodes");
        std::vector<index_t> st(n + 1, 0), nb;
        std::vector<double> w;
        for (index_t u = 0; u < n; ++u) {
            for (const WeightedEdge& e : g.adjacency[u]) {
                nb.push_back(e.neighbor);
                w.push_back(e.weight);
            }
            st[u + 1] = static_cast<index_t>(nb.size());
        }
        detail::check(hpbj_partition_adjacency(n, st.data(), nb.data(), w.data(), s, imbalance_tol, asg.data(),
                                               perm.data(), bst.data()),
                      nullptr);
    }
    return detail::finish_partition(std::move(asg), std::move(perm), std::move(bst), s);
}

// Extension: the fused graph + partition on a matrix (what partition_graph(
// graph_from_matrix(a), ...) does for an unread graph).
inline Partition partition_graph(const SparseMatrix& a, index_t s, double imbalance_tol = 0.1) {
    return partition_graph(graph_from_matrix(a), s, imbalance_tol);
}

// import_partition / export_partition (partition.cpp:146-174)
inline Partition import_partition(std::istream& in, index_t n, index_t s) {
    std::vector<index_t> assignment;
    assignment.reserve(static_cast<size_t>(std::max<index_t>(n, 0)));
    std::string line;
    long line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        std::istringstream ls(line);
        index_t b;
        if (!(ls >> b)) {
            if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
            throw std::runtime_error("partition file: line " + std::to_string(line_no) + ": malformed");
        }
        if (b < 0 || b >= s)
            throw std::out_of_range("partition file: line " + std::to_string(line_no) + ": block index " +
                                    std::to_string(b) + " out of range");
        assignment.push_back(b);
    }
    if (static_cast<index_t>(assignment.size()) != n)
        throw std::runtime_error("partition file: expected " + std::to_string(n) + " lines, got " +
                                 std::to_string(assignment.size()));
    return partition_from_assignment(std::move(assignment), s);
}

inline void export_partition(std::ostream& out, const Partition& p) {
    for (index_t b : p.assignment) out << b << "\n";
}

// measure_block_nnz (partition.cpp:176-194)
inline void measure_block_nnz(Partition& p, const SparseMatrix& a) {
    if (a.rows() != p.num_nodes()) throw std::invalid_argument("measure_block_nnz: dimension mismatch");
    p.block_nnz.assign(p.num_blocks, 0);
    const auto rs = a.row_starts();
    const auto ci = a.col_indices();
    for (index_t i = 0; i < a.rows(); ++i) {
        const index_t b = p.assignment[i];
        for (index_t k = rs[i]; k < rs[i + 1]; ++k)
            if (p.assignment[ci[k]] == b) ++p.block_nnz[b];
    }
    index_t total = 0, mx = 0;
    for (index_t c : p.block_nnz) {
        total += c;
        mx = std::max(mx, c);
    }
    const double mean = static_cast<double>(total) / static_cast<double>(p.num_blocks);
    p.imbalance = mean > 0.0 ? static_cast<double>(mx) / mean : 0.0;
}

// cut_weight (partition.cpp:196-203)
inline double cut_weight(const WeightedGraph& g, const Partition& p) {
    double cut = 0.0;
    for (index_t u = 0; u < g.num_nodes; ++u)
        for (const WeightedEdge& e : g.adjacency[u])
            if (u < e.neighbor && p.assignment[u] != p.assignment[e.neighbor]) cut += e.weight;
    return cut;
}

// ------------------------------------------------------------------ lu.hpp
enum class FactorKind { Exact, Ilu0 };

struct PerturbationRecord {  // lu.hpp:13-17
    index_t pivot_index;
    double original_value;
    double replaced_value;
};

struct LUFactors {  // lu.hpp:37-50
    index_t n = 0;
    SparseMatrix lower;  // strictly lower, unit diagonal implied
    SparseMatrix upper;  // diagonal first in each row
    std::vector<index_t> pivot_rows;
    std::vector<PerturbationRecord> perturbations;
    FactorKind kind = FactorKind::Exact;
    void materialize_low() {
        lower.materialize_low();
        upper.materialize_low();
    }
};

namespace detail {
// Reference layout (lu.hpp:37-50) from a row-major F = L_strict + U in pivot
// order; exact zeros dropped.
inline LUFactors lu_from_dense(index_t d, const std::vector<double>& f, std::vector<index_t> piv) {
    std::vector<index_t> lrs{0}, lci, urs{0}, uci;
    std::vector<double> lv, uv;
    for (index_t r = 0; r < d; ++r) {
        for (index_t c = 0; c < r; ++c)
            if (f[r * d + c] != 0.0) {
                lci.push_back(c);
                lv.push_back(f[r * d + c]);
            }
        lrs.push_back(static_cast<index_t>(lci.size()));
        uci.push_back(r);  // the diagonal, even if zero (regularised pivots never are)
        uv.push_back(f[r * d + r]);
        for (index_t c = r + 1; c < d; ++c)
            if (f[r * d + c] != 0.0) {
                uci.push_back(c);
                uv.push_back(f[r * d + c]);
            }
        urs.push_back(static_cast<index_t>(uci.size()));
    }
    LUFactors out;
    out.n = d;
    out.lower = SparseMatrix(d, d, std::move(lrs), std::move(lci), std::move(lv));
    // diagonal first: rows are not column-sorted in the reference's upper
    // factor, so it is built without the sorted-columns check
    out.upper = SparseMatrix(d, d, std::move(urs), std::move(uci), std::move(uv));
    out.pivot_rows = std::move(piv);
    return out;
}

// Read-only vector whose elements are produced on first access.
template <class T>
class LazyVector {
public:
    LazyVector() = default;
    LazyVector(size_t n, std::function<T(size_t)> load)
        : load_(std::move(load)), slots_(std::make_shared<std::vector<std::optional<T>>>(n)),
          mu_(std::make_shared<std::mutex>()) {}
    size_t size() const { return slots_ ? slots_->size() : 0; }
    bool empty() const { return size() == 0; }
    const T& operator[](size_t i) const {
        std::lock_guard<std::mutex> g(*mu_);
        auto& s = (*slots_)[i];
        if (!s) s = load_(i);
        return *s;
    }
    const T& at(size_t i) const {
        if (i >= size()) throw std::out_of_range("LazyVector::at");
        return (*this)[i];
    }

private:
    std::function<T(size_t)> load_;
    std::shared_ptr<std::vector<std::optional<T>>> slots_;
    std::shared_ptr<std::mutex> mu_;
};
}  // namespace detail

// ------------------------------------------------------ preconditioner.hpp
struct PreconditionerStats {  // preconditioner.hpp:14-20
    index_t block_dim = 0;
    index_t block_nnz = 0;
    index_t perturbation_count = 0;
    double cond_estimate = 0.0;
    double error_bound = 0.0;
};

// block_error_bound (preconditioner.cpp:13-15)
inline double block_error_bound(double cond_estimate, double eps_low, double eps_high) {
    return (cond_estimate * eps_high + eps_low) * cond_estimate;
}

struct BlockJacobiOptions {  // preconditioner.hpp:32-38
    double eps_pivot = 1e-10;
    int neumann_order = 0;  // 0 = direct block solves
    PrecisionPolicy policy{};
    bool parallel_build = true;       // the device build is always batched
    bool with_cond_estimates = true;  // computed on the device on first read of stats
};

struct BlockJacobiData {  // preconditioner.hpp:40-46
    Partition partition;
    detail::LazyVector<SparseMatrix> blocks;  // diagonal blocks of Q A Q^T (sliced on first access)
    detail::LazyVector<LUFactors> factors;    // FP32 device factors, widened (fetched on first access)
    std::vector<PreconditionerStats> stats;
    int neumann_order = 0;
};

namespace detail {
struct PcAccess;
struct PcState {
    std::unique_ptr<CtxLease> dev;        // factors (block Jacobi / ILU(0)) live here
    std::shared_ptr<const Csr> built;     // the matrix they were built from
    BlockJacobiOptions opts;
    bool low = true;                      // FP32 factor copies "materialised" (opts.policy Hybrid)
    mutable std::once_flag bj_once, ilu_once;
    mutable std::shared_ptr<BlockJacobiData> bj;
    mutable std::shared_ptr<LUFactors> ilu;
    mutable std::mutex mu;                // one device call at a time per context
};
}  // namespace detail

class Preconditioner {  // preconditioner.hpp:50-98
public:
    enum class Kind { Identity, Ilu0, BlockJacobi };

    static Preconditioner identity(index_t n) { return Preconditioner(Kind::Identity, n); }

    // Preconditioner::from_ilu0 (preconditioner.cpp:94-98): FP64 ILU(0) on the device
    static Preconditioner from_ilu0(const SparseMatrix& a, int device = 0) {
        Preconditioner p(Kind::Ilu0, a.rows());
        p.st_->dev = std::make_unique<detail::CtxLease>(device);
        detail::DeviceCtx& c = *p.st_->dev->c;
        detail::bind_matrix(c, a.payload(), true);
        c.bj = false;
        detail::check(hpbj_ilu0_setup(c.ctx, nullptr), c.ctx);
        p.st_->built = a.payload();
        p.st_->low = false;  // ilu0 keeps binary64 factors only (lu.cpp:227-312)
        return p;
    }

    // Preconditioner::block_jacobi (preconditioner.cpp:100-153): Q A Q^T,
    // batched FP32 LU of the diagonal blocks on the device
    static Preconditioner block_jacobi(const SparseMatrix& a, Partition partition, const BlockJacobiOptions& opts = {},
                                       int device = 0) {
        if (a.rows() != a.cols()) throw std::invalid_argument("block_jacobi: matrix must be square");
        if (partition.num_nodes() != a.rows())
            throw std::invalid_argument("block_jacobi: partition does not cover the matrix");
        Preconditioner p(Kind::BlockJacobi, a.rows());
        detail::PcState& st = *p.st_;
        st.dev = std::make_unique<detail::CtxLease>(device);
        detail::DeviceCtx& c = *st.dev->c;
        detail::bind_matrix(c, a.payload(), true);
        detail::check(hpbj_bj_set_neumann_order(c.ctx, opts.neumann_order), c.ctx);
        hpbj_setup_info info{};
        int rc;
        if (c.bj && c.eps == opts.eps_pivot && c.perm == partition.perm && c.block_starts == partition.block_starts)
            rc = hpbj_bj_refactor(c.ctx, &info);  // same pattern and partition: numeric refactorisation only
        else
            rc = hpbj_bj_setup(c.ctx, partition.num_blocks, partition.perm.data(), partition.block_starts.data(),
                               opts.eps_pivot, &info);
        c.bj = false;
        detail::check(rc, c.ctx, info.singular_column);
        c.bj = true;
        c.eps = opts.eps_pivot;
        c.perm = partition.perm;
        c.block_starts = partition.block_starts;
        st.built = a.payload();
        st.opts = opts;
        st.low = opts.policy.hybrid();
        auto data = std::make_shared<BlockJacobiData>();
        data->partition = std::move(partition);
        data->neumann_order = opts.neumann_order;
        st.bj = std::move(data);
        return p;
    }

    index_t dim() const { return n_; }
    Kind kind() const { return kind_; }
    int neumann_order() const { return kind_ == Kind::BlockJacobi ? st_->opts.neumann_order : 0; }

    // apply (preconditioner.cpp:159-198): z with M z = v, original ordering.
    // Block Jacobi runs the FP32 factors (v rounded to FP32 on load), ILU(0)
    // its FP64 factors; T only sets the vector type.
    template <class T>
    void apply(std::span<const T> v, std::span<T> z) const {
        if (static_cast<index_t>(v.size()) != n_ || static_cast<index_t>(z.size()) != n_)
            throw std::invalid_argument("preconditioner apply: dimension mismatch");
        if (kind_ == Kind::Identity) {
            std::copy(v.begin(), v.end(), z.begin());
            return;
        }
        if constexpr (std::is_same_v<T, float>)
            if (!st_->low) throw std::logic_error("values_low requested before materialize_low()");
        std::vector<double> vd(v.begin(), v.end()), zd(n_);
        {
            std::lock_guard<std::mutex> g(st_->mu);
            detail::DeviceCtx& c = *st_->dev->c;
            detail::check(hpbj_precond_apply(c.ctx, vd.data(), zd.data()), c.ctx);
        }
        for (index_t i = 0; i < n_; ++i) z[i] = static_cast<T>(zd[i]);
    }
    template <class T>
    void apply_serial(std::span<const T> v, std::span<T> z) const {
        apply<T>(v, z);  // blocks are independent: same result
    }
    template <class T>
    std::vector<T> apply(std::span<const T> v) const {
        std::vector<T> z(v.size());
        apply<T>(v, z);
        return z;
    }

    // apply_neumann (preconditioner.cpp:200-220), FP32 series on the device
    template <class T>
    std::vector<T> apply_neumann(const SparseMatrix& a, std::span<const T> v, int k) const {
        if (kind_ != Kind::BlockJacobi) throw std::logic_error("apply_neumann: block factors not available");
        if (k < 0 || k > st_->opts.neumann_order)
            throw std::invalid_argument("apply_neumann: order exceeds the one the preconditioner was built with");
        if (static_cast<index_t>(v.size()) != n_)
            throw std::invalid_argument("preconditioner apply: dimension mismatch");
        std::vector<double> vd(v.begin(), v.end()), zd(n_);
        {
            std::lock_guard<std::mutex> g(st_->mu);
            detail::DeviceCtx& c = *st_->dev->c;
            detail::bind_matrix(c, a.payload(), false);
            detail::check(hpbj_bj_apply_neumann(c.ctx, vd.data(), zd.data(), k), c.ctx);
        }
        return std::vector<T>(zd.begin(), zd.end());
    }

    const BlockJacobiData* block_jacobi_data() const {
        if (kind_ != Kind::BlockJacobi) return nullptr;
        std::call_once(st_->bj_once, [&] { fill_bj_data(); });
        return st_->bj.get();
    }
    const LUFactors* ilu_factors() const {
        if (kind_ != Kind::Ilu0) return nullptr;
        std::call_once(st_->ilu_once, [&] { fill_ilu(); });
        return st_->ilu.get();
    }

    // extensions
    hpbj_ctx* context() const { return st_->dev ? st_->dev->c->ctx : nullptr; }
    const Partition& partition() const { return st_->bj->partition; }

private:
    friend struct detail::PcAccess;
    Preconditioner(Kind kind, index_t n) : kind_(kind), n_(n), st_(std::make_shared<detail::PcState>()) {}

    void fill_bj_data() const {
        detail::PcState& st = *st_;
        BlockJacobiData& d = *st.bj;
        {  // measure_block_nnz (partition.cpp:176-194) on the payload itself
            const detail::Csr& A = *st.built;
            Partition& p = d.partition;
            p.block_nnz.assign(p.num_blocks, 0);
            for (index_t i = 0; i < A.nrows; ++i)
                for (index_t k = A.rs[i]; k < A.rs[i + 1]; ++k)
                    if (p.assignment[A.ci[k]] == p.assignment[i]) ++p.block_nnz[p.assignment[i]];
            index_t total = 0, mx = 0;
            for (index_t c : p.block_nnz) {
                total += c;
                mx = std::max(mx, c);
            }
            const double mean = static_cast<double>(total) / static_cast<double>(p.num_blocks);
            p.imbalance = mean > 0.0 ? static_cast<double>(mx) / mean : 0.0;
        }
        const size_t s = static_cast<size_t>(d.partition.num_blocks);
        std::vector<index_t> dims(s), pc(s);
        std::vector<double> cond(s, 0.0), eb(s, 0.0);
        {
            std::lock_guard<std::mutex> g(st.mu);
            hpbj_ctx* ctx = st.dev->c->ctx;
            detail::check(hpbj_get_block_stats(ctx, dims.data(), pc.data()), ctx);
            if (st.opts.with_cond_estimates) detail::check(hpbj_get_block_diagnostics(ctx, cond.data(), eb.data()), ctx);
        }
        d.stats.resize(s);
        for (size_t b = 0; b < s; ++b) {
            PreconditionerStats& x = d.stats[b];
            x.block_dim = dims[b];
            x.block_nnz = d.partition.block_nnz[b];
            x.perturbation_count = pc[b];
            if (st.opts.with_cond_estimates) {
                x.cond_estimate = cond[b];
                x.error_bound = block_error_bound(cond[b], st.low ? kRoundoffSingle : kRoundoffDouble, kRoundoffDouble);
            }
        }
        auto keep = st_;  // the lazy members hold the state alive
        d.factors = detail::LazyVector<LUFactors>(s, [keep](size_t b) {
            std::lock_guard<std::mutex> g(keep->mu);
            hpbj_ctx* ctx = keep->dev->c->ctx;
            const index_t d0 = keep->bj->partition.block_size(static_cast<index_t>(b));
            std::vector<float> f(static_cast<size_t>(d0 * d0));
            std::vector<index_t> piv(d0);
            index_t dim = 0;
            detail::check(hpbj_get_block_factors(ctx, static_cast<index_t>(b), &dim, f.data(), piv.data()), ctx);
            LUFactors out = detail::lu_from_dense(dim, std::vector<double>(f.begin(), f.end()), std::move(piv));
            if (keep->low) out.materialize_low();
            return out;
        });
        d.blocks = detail::LazyVector<SparseMatrix>(s, [keep](size_t b) {  // slice_diag_block, preconditioner.cpp:20-40
            const Partition& part = keep->bj->partition;
            const detail::Csr& A = *keep->built;
            const index_t b0 = part.block_starts[b], d0 = part.block_size(static_cast<index_t>(b));
            std::vector<index_t> rows(d0);
            for (index_t i = 0; i < A.nrows; ++i)
                if (part.assignment[i] == static_cast<index_t>(b)) rows[part.perm[i] - b0] = i;
            std::vector<index_t> rs{0}, ci;
            std::vector<double> v;
            std::vector<std::pair<index_t, double>> row;
            for (index_t r = 0; r < d0; ++r) {
                const index_t i = rows[r];
                row.clear();
                for (index_t k = A.rs[i]; k < A.rs[i + 1]; ++k)
                    if (part.assignment[A.ci[k]] == static_cast<index_t>(b))
                        row.emplace_back(part.perm[A.ci[k]] - b0, A.v[k]);
                std::sort(row.begin(), row.end());
                for (const auto& [c, x] : row) {
                    ci.push_back(c);
                    v.push_back(x);
                }
                rs.push_back(static_cast<index_t>(ci.size()));
            }
            return SparseMatrix(d0, d0, std::move(rs), std::move(ci), std::move(v));
        });
    }
    void fill_ilu() const {
        detail::PcState& st = *st_;
        const detail::Csr& A = *st.built;
        std::vector<double> lu(A.v.size());
        {
            std::lock_guard<std::mutex> g(st.mu);
            detail::check(hpbj_get_ilu0_values(st.dev->c->ctx, lu.data()), st.dev->c->ctx);
        }
        // lu.cpp:273-298: row i -> L (columns < i), U (diagonal first, then columns > i)
        std::vector<index_t> lrs{0}, lci, urs{0}, uci;
        std::vector<double> lv, uv;
        for (index_t i = 0; i < A.nrows; ++i) {
            index_t dpos = -1;
            for (index_t k = A.rs[i]; k < A.rs[i + 1]; ++k) {
                if (A.ci[k] < i) {
                    lci.push_back(A.ci[k]);
                    lv.push_back(lu[k]);
                } else if (A.ci[k] == i) {
                    dpos = k;
                }
            }
            lrs.push_back(static_cast<index_t>(lci.size()));
            uci.push_back(i);
            uv.push_back(dpos >= 0 ? lu[dpos] : 0.0);
            for (index_t k = A.rs[i]; k < A.rs[i + 1]; ++k)
                if (A.ci[k] > i) {
                    uci.push_back(A.ci[k]);
                    uv.push_back(lu[k]);
                }
            urs.push_back(static_cast<index_t>(uci.size()));
        }
        auto f = std::make_shared<LUFactors>();
        f->n = A.nrows;
        f->lower = SparseMatrix(A.nrows, A.nrows, std::move(lrs), std::move(lci), std::move(lv));
        f->upper = SparseMatrix(A.nrows, A.nrows, std::move(urs), std::move(uci), std::move(uv));
        f->pivot_rows.resize(A.nrows);
        for (index_t i = 0; i < A.nrows; ++i) f->pivot_rows[i] = i;
        f->kind = FactorKind::Ilu0;
        st.ilu = std::move(f);
    }

    Kind kind_ = Kind::Identity;
    index_t n_ = 0;
    std::shared_ptr<detail::PcState> st_;
};

namespace detail {
struct PcAccess {
    static PcState& state(const Preconditioner& p) { return *p.st_; }
};
}  // namespace detail

// ----------------------------------------------------------------- gmres.hpp
struct GmresConfig {  // gmres.hpp:89-97
    index_t restart_m = 50;
    double tol = 1e-8;  // on ||r||_2 / ||b||_2 unless absolute_tol
    index_t max_restarts = 40;
    bool absolute_tol = false;
    PrecisionPolicy policy{};
    double breakdown_tol_factor = 1e2;
    bool collect_ritz = false;
};

struct HistoryPoint {  // gmres.hpp:99-103
    index_t cycle;
    index_t iteration;  // global iteration number; 0 is the initial residual
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
    double setup_seconds = 0.0;  // never written (as in the reference)
    double iterate_seconds = 0.0;
    std::vector<std::complex<double>> ritz;
};

struct SolveResult {
    std::vector<double> x;
    SolveReport report;
};

// hybrid_restart_gmres (gmres.hpp:145-147, gmres.cpp:200-274): every
// numerical step on the device; the host reads a few scalars per cycle.
inline SolveResult hybrid_restart_gmres(const SparseMatrix& a, const Preconditioner& p, std::span<const double> b,
                                        const GmresConfig& config) {
    if (a.rows() != a.cols()) throw std::invalid_argument("gmres: matrix must be square");
    if (static_cast<index_t>(b.size()) != a.rows()) throw std::invalid_argument("gmres: rhs dimension mismatch");
    if (config.restart_m < 1 || config.tol <= 0.0 || config.max_restarts < 1)
        throw std::invalid_argument("gmres: invalid config");
    if (config.collect_ritz)
        throw std::invalid_argument("gmres: collect_ritz (Ritz values) is not computed by the B200 build");
    if (p.dim() != a.rows()) throw std::invalid_argument("preconditioner apply: dimension mismatch");
    const bool hybrid = config.policy.hybrid();
    // Hybrid reads the FP32 copies of A (spmv<float>) and of the factors
    // (lu_solve<float>): the reference's precondition errors
    if (hybrid && !a.has_low()) throw std::logic_error("values_low requested before materialize_low()");
    using Kind = Preconditioner::Kind;
    detail::PcState& st = detail::PcAccess::state(p);
    if (hybrid && p.kind() != Kind::Identity && !st.low)
        throw std::logic_error("values_low requested before materialize_low()");
    if (!hybrid && p.kind() == Kind::BlockJacobi)
        throw std::invalid_argument("gmres: DoubleOnly block Jacobi (FP64 factors) is not implemented on the GPU path");

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
    std::vector<hpbj_history_point> hist(static_cast<size_t>(config.restart_m * config.max_restarts + 2));
    std::vector<double> cyc(static_cast<size_t>(config.max_restarts + 1));
    hpbj_report rep{};
    if (p.kind() == Kind::Identity) {
        std::lock_guard<std::mutex> g(st.mu);
        if (!st.dev) st.dev = std::make_unique<detail::CtxLease>(0);
        detail::DeviceCtx& c = *st.dev->c;
        detail::bind_matrix(c, a.payload(), true);
        c.bj = false;
        detail::check(hpbj_identity_setup(c.ctx), c.ctx);
        detail::check(hpbj_gmres(c.ctx, b.data(), out.x.data(), &o, &rep, hist.data(),
                                 static_cast<int64_t>(hist.size()), cyc.data(), static_cast<int64_t>(cyc.size())),
                      c.ctx);
    } else {
        std::lock_guard<std::mutex> g(st.mu);
        detail::DeviceCtx& c = *st.dev->c;
        detail::bind_matrix(c, a.payload(), false);
        detail::check(hpbj_gmres(c.ctx, b.data(), out.x.data(), &o, &rep, hist.data(),
                                 static_cast<int64_t>(hist.size()), cyc.data(), static_cast<int64_t>(cyc.size())),
                      c.ctx);
    }
    SolveReport& r = out.report;
    r.converged = rep.converged != 0;
    r.total_iterations = rep.total_iterations;
    r.restarts = rep.restarts;
    r.final_residual = rep.final_residual;
    r.breakdown = rep.breakdown != 0;
    r.ls_rank_deficient = rep.ls_rank_deficient != 0;
    r.iterate_seconds = rep.ms_solve * 1e-3;
    const int64_t hn = std::min<int64_t>(rep.history_len, static_cast<int64_t>(hist.size()));
    for (int64_t k = 0; k < hn; ++k) r.residual_history.push_back({hist[k].cycle, hist[k].iteration, hist[k].relative_residual});
    r.cycle_residuals.assign(cyc.begin(), cyc.begin() + std::min<int64_t>(rep.cycles, static_cast<int64_t>(cyc.size())));
    return out;
}

// --------------------------------------------------------- matrix_market.hpp
// read/write_matrix_market_file (matrix_market.cpp:36-121): host parser and
// writer of libhpbj.so, bit-identical to the reference's.
inline SparseMatrix read_matrix_market_file(const std::string& path) {
    int64_t nr = 0, nc = 0, *rp = nullptr, *ci = nullptr;
    double* v = nullptr;
    detail::check(hpbj_mm_read(path.c_str(), &nr, &nc, &rp, &ci, &v), nullptr);
    std::vector<index_t> r(rp, rp + nr + 1), c(ci, ci + rp[nr]);
    std::vector<double> vv(v, v + rp[nr]);
    hpbj_free(rp);
    hpbj_free(ci);
    hpbj_free(v);
    return SparseMatrix(nr, nc, std::move(r), std::move(c), std::move(vv));
}

inline SparseMatrix read_matrix_market(std::istream& in) {
    // through a temporary file: the parser reads whole files
    std::string tmpl = "/tmp/hpbj_mm_XXXXXX";
    std::vector<char> name(tmpl.begin(), tmpl.end());
    name.push_back('\0');
    const int fd = mkstemp(name.data());
    if (fd < 0) throw std::runtime_error("matrix market: cannot create a temporary file");
    close(fd);
    {
        std::ofstream out(name.data(), std::ios::binary);
        out << in.rdbuf();
    }
    try {
        SparseMatrix a = read_matrix_market_file(name.data());
        std::remove(name.data());
        return a;
    } catch (...) {
        std::remove(name.data());
        throw;
    }
}

inline void write_matrix_market_file(const std::string& path, const SparseMatrix& a) {
    detail::check(hpbj_mm_write(path.c_str(), a.rows(), a.cols(), a.row_starts().data(), a.col_indices().data(),
                                a.values().data()),
                  nullptr);
}

inline void write_matrix_market(std::ostream& out, const SparseMatrix& a) {
    char buf[64];
    out << "%%MatrixMarket matrix coordinate real general\n";
    out << a.rows() << " " << a.cols() << " " << a.nnz() << "\n";
    const auto rs = a.row_starts();
    const auto ci = a.col_indices();
    const auto v = a.values();
    for (index_t i = 0; i < a.rows(); ++i)
        for (index_t k = rs[i]; k < rs[i + 1]; ++k) {
            std::snprintf(buf, sizeof buf, "%.17g", v[k]);
            out << (i + 1) << " " << (ci[k] + 1) << " " << buf << "\n";
        }
}

}  // namespace bjgmres

namespace bjgmres_b200 = bjgmres;  // round-1 name
