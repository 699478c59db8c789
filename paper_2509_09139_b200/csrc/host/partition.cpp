// Host-side graph construction and block partitioning — bit-identical to the
// reference (graph.cpp:17-51, partition.cpp:14-144) but O(nnz + n) instead of
// the reference's O(nnz log nnz) std::map build and O(n * s) seed scans.
//
// Why the results are bit-identical:
//  * weights: the reference accumulates 0.0 + |a_lo,hi| (+ |a_hi,lo|) per
//    unordered pair (graph.cpp:27-34) and halves it (:40). With at most two
//    addends of |.| >= 0, 0.0 + x == x and x + y == y + x exactly, so
//    w = 0.5 * (|a_ij| + |a_ji|) (or 0.5 * |single|) from a CSR/CSR^T merge
//    is the same double. Pairs with w <= 0 are dropped (:41); adjacency is
//    sorted by neighbour (:45-49), which the merge produces directly.
//  * seeds: pick_seed (partition.cpp:45-56) returns the lowest-index node of
//    maximal degree among unassigned nodes with degree > 0. Degrees are
//    static and assignments only grow, so a monotone cursor over nodes
//    sorted by (degree desc, index asc) returns the same node.
//  * queue: the reference pushes duplicates and skips assigned nodes on pop
//    (:92-100); de-duplicating on push (flags cleared with the queue per
//    block, :84) pops unassigned nodes in the same order.
//  * leftovers: "first block of minimal size" (:105-112) == a (size, id)
//    min-heap.
//  * refinement: restated verbatim, same accumulation order (:117-141).

#include <algorithm>
#include <cmath>
#include <cstring>
#include <queue>
#include <string>
#include <utility>
#include <vector>

#include "../hpbj_common.hpp"

namespace hpbj {

void check_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val) {
    // SparseMatrix invariants (sparse_matrix.cpp:14-50).
    if (n < 0) fail(HPBJ_EINVAL, "sparse matrix: negative dimension");
    if (!rp || (rp[n] > 0 && (!ci || !val))) fail(HPBJ_EINVAL, "sparse matrix: null array");
    if (rp[0] != 0) fail(HPBJ_EINVAL, "sparse matrix: inconsistent sizes");
    for (int64_t i = 0; i < n; ++i) {
        if (rp[i] > rp[i + 1]) fail(HPBJ_EINVAL, "sparse matrix: row_starts not non-decreasing");
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= n)
                fail(HPBJ_EINVAL, "sparse matrix: column index out of range");
            if (k > rp[i] && ci[k - 1] >= ci[k])
                fail(HPBJ_EINVAL, "sparse matrix: columns not strictly increasing");
        }
    }
}

Adjacency graph_from_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val) {
    const int64_t nnz = rp[n];
    // Transpose pattern + values (counting sort by column; rows ascending
    // inside each column, so every transposed row is sorted).
    std::vector<int64_t> tst(n + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) ++tst[ci[k] + 1];
    for (int64_t i = 0; i < n; ++i) tst[i + 1] += tst[i];
    std::vector<int64_t> trow(nnz);
    std::vector<double> tval(nnz);
    {
        std::vector<int64_t> next(tst.begin(), tst.end() - 1);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int64_t d = next[ci[k]]++;
                trow[d] = i;
                tval[d] = val[k];
            }
    }
    // Merge row u of A (entries a_uj) with row u of A^T (entries a_ju).
    auto merge = [&](int64_t u, int64_t* nb, double* w) -> int64_t {
        int64_t p = rp[u], pe = rp[u + 1], q = tst[u], qe = tst[u + 1], cnt = 0;
        while (p < pe || q < qe) {
            const int64_t jp = p < pe ? ci[p] : INT64_MAX;
            const int64_t jq = q < qe ? trow[q] : INT64_MAX;
            int64_t j;
            double s;
            if (jp == jq) {
                j = jp;
                s = std::fabs(val[p++]) + std::fabs(tval[q++]);
            } else if (jp < jq) {
                j = jp;
                s = std::fabs(val[p++]);
            } else {
                j = jq;
                s = std::fabs(tval[q++]);
            }
            if (j == u) continue;  // diagonal ignored (graph.cpp:30)
            const double wt = 0.5 * s;
            if (wt <= 0.0) continue;  // w <= 0 dropped (graph.cpp:41); NaN kept, as there
            if (nb) {
                nb[cnt] = j;
                w[cnt] = wt;
            }
            ++cnt;
        }
        return cnt;
    };
    Adjacency g;
    g.n = n;
    g.start.assign(n + 1, 0);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t u = 0; u < n; ++u) g.start[u + 1] = merge(u, nullptr, nullptr);
    for (int64_t u = 0; u < n; ++u) g.start[u + 1] += g.start[u];
    g.nbr.resize(g.start[n]);
    g.w.resize(g.start[n]);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t u = 0; u < n; ++u) merge(u, g.nbr.data() + g.start[u], g.w.data() + g.start[u]);
    return g;
}

void partition_from_assignment(int64_t n, const int64_t* assignment, int64_t s, int64_t* perm,
                               int64_t* block_starts) {
    if (s < 1 || s > n) fail(HPBJ_EINVAL, "partition: block count must satisfy 1 <= s <= n");
    std::vector<int64_t> counts(s, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t b = assignment[i];
        if (b < 0 || b >= s) fail(HPBJ_ERANGE, "partition: block index out of range");
        ++counts[b];
    }
    for (int64_t b = 0; b < s; ++b)
        if (counts[b] == 0)
            fail(HPBJ_EINVAL, "partition: block " + std::to_string(b) + " is empty");
    block_starts[0] = 0;
    for (int64_t b = 0; b < s; ++b) block_starts[b + 1] = block_starts[b] + counts[b];
    std::vector<int64_t> next(block_starts, block_starts + s);
    for (int64_t i = 0; i < n; ++i) perm[i] = next[assignment[i]]++;  // stable gather
}

void partition_adjacency(const Adjacency& g, int64_t s, double tol, int64_t* assignment) {
    const int64_t n = g.n;
    if (s < 1) fail(HPBJ_EINVAL, "partition_graph: s must be >= 1");
    if (s > n) fail(HPBJ_EINVAL, "partition_graph: s exceeds node count");
    if (tol < 0.0) fail(HPBJ_EINVAL, "partition_graph: negative imbalance tolerance");

    // cap formula verbatim (partition.cpp:67-69)
    const int64_t cap = std::max<int64_t>(
        static_cast<int64_t>(std::ceil(static_cast<double>(n) / s * (1.0 + tol))),
        (n + s - 1) / s);

    auto deg = [&](int64_t v) { return g.start[v + 1] - g.start[v]; };
    std::fill(assignment, assignment + n, int64_t(-1));
    std::vector<int64_t> sizes(s, 0);

    // Seed order: degree desc, index asc (counting sort on degree).
    int64_t maxdeg = 0, connected = 0;
    for (int64_t v = 0; v < n; ++v) {
        maxdeg = std::max(maxdeg, deg(v));
        if (deg(v) > 0) ++connected;
    }
    std::vector<int64_t> dstart(maxdeg + 2, 0);
    for (int64_t v = 0; v < n; ++v)
        if (deg(v) > 0) ++dstart[maxdeg - deg(v) + 1];
    for (int64_t d = 0; d <= maxdeg; ++d) dstart[d + 1] += dstart[d];
    std::vector<int64_t> order(connected);
    for (int64_t v = 0; v < n; ++v)
        if (deg(v) > 0) order[dstart[maxdeg - deg(v)]++] = v;
    int64_t cursor = 0;

    // Region growing (partition.cpp:74-103).
    std::vector<int64_t> queue(static_cast<size_t>(n));
    std::vector<uint8_t> inq(n, 0);
    int64_t connected_left = connected;
    for (int64_t b = 0; b < s && connected_left > 0; ++b) {
        const int64_t blocks_left = s - b;
        int64_t target = (connected_left + blocks_left - 1) / blocks_left;
        target = std::min(target, cap);
        int64_t head = 0, tail = 0;
        int64_t grown = 0;
        while (grown < target) {
            if (head == tail) {
                while (cursor < connected && assignment[order[cursor]] >= 0) ++cursor;
                if (cursor == connected) break;
                queue[tail++] = order[cursor];
                inq[order[cursor]] = 1;
            }
            const int64_t u = queue[head++];
            inq[u] = 0;
            assignment[u] = b;
            ++sizes[b];
            ++grown;
            --connected_left;
            for (int64_t k = g.start[u]; k < g.start[u + 1]; ++k) {
                const int64_t v = g.nbr[k];
                if (assignment[v] < 0 && !inq[v]) {
                    inq[v] = 1;
                    queue[tail++] = v;
                }
            }
        }
        for (int64_t q = head; q < tail; ++q) inq[queue[q]] = 0;  // queue.clear()
    }

    // Remaining nodes -> first block of minimal size (partition.cpp:105-112).
    {
        using Key = std::pair<int64_t, int64_t>;  // (size, block)
        std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
        bool built = false;
        for (int64_t v = 0; v < n; ++v) {
            if (assignment[v] >= 0) continue;
            if (!built) {
                for (int64_t b = 0; b < s; ++b) heap.push({sizes[b], b});
                built = true;
            }
            const Key k = heap.top();
            heap.pop();
            assignment[v] = k.second;
            ++sizes[k.second];
            heap.push({sizes[k.second], k.second});
        }
    }

    // One boundary-refinement sweep (partition.cpp:117-141), verbatim order.
    std::vector<double> conn(s, 0.0);
    std::vector<int64_t> touched;
    for (int64_t u = 0; u < n; ++u) {
        const int64_t bu = assignment[u];
        if (sizes[bu] <= 1) continue;
        touched.clear();
        for (int64_t k = g.start[u]; k < g.start[u + 1]; ++k) {
            const int64_t bv = assignment[g.nbr[k]];
            if (conn[bv] == 0.0) touched.push_back(bv);
            conn[bv] += g.w[k];
        }
        int64_t best = -1;
        for (int64_t bv : touched) {
            if (bv == bu || sizes[bv] + 1 > cap) continue;
            if (best < 0 || conn[bv] > conn[best] || (conn[bv] == conn[best] && bv < best))
                best = bv;
        }
        if (best >= 0 && conn[best] > conn[bu]) {
            assignment[u] = best;
            --sizes[bu];
            ++sizes[best];
        }
        for (int64_t bv : touched) conn[bv] = 0.0;
    }
}

namespace {
thread_local std::string t_err;
}
void set_thread_error(const std::string& msg) { t_err = msg; }
const char* thread_error() { return t_err.c_str(); }

}  // namespace hpbj

using namespace hpbj;

extern "C" {

int hpbj_graph_from_matrix(int64_t n, const int64_t* row_ptr, const int64_t* col,
                           const double* val, int64_t* adj_start, int64_t* adj_nbr,
                           double* adj_w, int64_t cap) {
    return guard(nullptr, [&] {
        check_csr(n, row_ptr, col, val);
        const Adjacency g = graph_from_csr(n, row_ptr, col, val);
        if (g.start[n] > cap) fail(HPBJ_EINVAL, "graph_from_matrix: adjacency capacity too small");
        std::memcpy(adj_start, g.start.data(), sizeof(int64_t) * (n + 1));
        std::memcpy(adj_nbr, g.nbr.data(), sizeof(int64_t) * g.start[n]);
        std::memcpy(adj_w, g.w.data(), sizeof(double) * g.start[n]);
    });
}

int hpbj_partition_graph(int64_t n, const int64_t* row_ptr, const int64_t* col,
                         const double* val, int64_t s, double imbalance_tol,
                         int64_t* assignment, int64_t* perm, int64_t* block_starts) {
    return guard(nullptr, [&] {
        check_csr(n, row_ptr, col, val);
        const Adjacency g = graph_from_csr(n, row_ptr, col, val);
        partition_adjacency(g, s, imbalance_tol, assignment);
        partition_from_assignment(n, assignment, s, perm, block_starts);
    });
}

int hpbj_partition_adjacency(int64_t n, const int64_t* adj_start, const int64_t* adj_nbr,
                             const double* adj_w, int64_t s, double imbalance_tol,
                             int64_t* assignment, int64_t* perm, int64_t* block_starts) {
    return guard(nullptr, [&] {
        if (n < 0 || !adj_start) fail(HPBJ_EINVAL, "partition_graph: bad graph");
        Adjacency g;
        g.n = n;
        g.start.assign(adj_start, adj_start + n + 1);
        g.nbr.assign(adj_nbr, adj_nbr + adj_start[n]);
        g.w.assign(adj_w, adj_w + adj_start[n]);
        partition_adjacency(g, s, imbalance_tol, assignment);
        partition_from_assignment(n, assignment, s, perm, block_starts);
    });
}

int hpbj_partition_from_assignment(int64_t n, const int64_t* assignment, int64_t s,
                                   int64_t* perm, int64_t* block_starts) {
    return guard(nullptr, [&] { partition_from_assignment(n, assignment, s, perm, block_starts); });
}

}  // extern "C"
