// Host-side graph construction and block partitioning — bit-identical to the
// reference (graph.cpp:17-51, partition.cpp:14-144) but O(nnz + n) instead of
// the reference's O(nnz log nnz) std::map build and O(n * s) seed scans
// (config 3: 1.0e3 s in the reference, ~1 s here).
//
// Why the results are bit-identical:
//  * weights: the reference accumulates 0.0 + |a_lo,hi| (+ |a_hi,lo|) per
//    unordered pair (graph.cpp:27-34) and halves it (:40). With at most two
//    addends of |.| >= 0, 0.0 + x == x and x + y == y + x exactly, so
//    w = 0.5 * (|a_ij| + |a_ji|) (or 0.5 * |single|) is the same double
//    whichever side computes it. Pairs with w <= 0 are dropped (:41);
//    adjacency is sorted by neighbour (:45-49).
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
//
// Performance (config 3, n = 4.1M, on the 16-core GPU-box host: 190 ms in
// round 1, ~137 ms now; the reference's O(n*s) partitioner takes ~600 s):
//  * region growing is one sequential BFS per block by the reference's
//    semantics (a block's seed is the first node left free by every earlier
//    block; measured: with even one block speculated ahead, 37% of the
//    predictions fail, so it stays single-threaded). It reads fixed-stride
//    8-id neighbour records (one cache line per popped node instead of the
//    offset + adjacency lines of a CSR), prefetched 16 pops ahead, tests
//    and sets a taken bitmap (n bits, cache resident), and appends popped
//    nodes to a list; block ids are written from that list in parallel;
//  * on large matrices without explicit off-diagonal zeros the BFS starts on
//    A's own off-diagonal pattern while 8 other cores compute the weights
//    (and with them the symmetry check) and the refinement view; an
//    unsymmetric pattern abandons that BFS for the general path;
//  * the refinement sweep runs as a parallel speculative phase over node
//    ranges plus an exact in-order resolution (refine_sweep_par);
//  * block ids are 16-bit when s fits (half the cache footprint of the
//    refinement's random neighbour lookups); host buffers sit on
//    transparent huge pages.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <queue>
#include <type_traits>
#include <string>
#include <utility>
#include <vector>
#include <exception>
#include <functional>
#include <thread>
#if defined(__x86_64__)
#include <x86intrin.h>
#else
static inline unsigned long long __rdtsc() { return 0; }
#endif

#include <omp.h>
#include <sys/mman.h>
#include <new>

#include "../hpbj_common.hpp"

namespace hpbj {

void check_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val) {
    // SparseMatrix invariants (sparse_matrix.cpp:14-50).
    if (n < 0) fail(HPBJ_EINVAL, "sparse matrix: negative dimension");
    if (!rp || (rp[n] > 0 && (!ci || !val))) fail(HPBJ_EINVAL, "sparse matrix: null array");
    if (rp[0] != 0) fail(HPBJ_EINVAL, "sparse matrix: inconsistent sizes");
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < n; ++i) {
        if (rp[i] > rp[i + 1]) {
            bad |= 1;
            continue;
        }
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= n) bad |= 2;
            else if (k > rp[i] && ci[k - 1] >= ci[k]) bad |= 4;
        }
    }
    if (bad & 1) fail(HPBJ_EINVAL, "sparse matrix: row_starts not non-decreasing");
    if (bad & 2) fail(HPBJ_EINVAL, "sparse matrix: column index out of range");
    if (bad & 4) fail(HPBJ_EINVAL, "sparse matrix: columns not strictly increasing");
}

namespace {

// General path: explicit transpose (rows ascending inside each column) and a
// per-row merge of A(u, :) with A(:, u).
Adjacency graph_general(int64_t n, const int64_t* rp, const int64_t* ci, const double* val) {
    const int64_t nnz = rp[n];
    std::vector<int64_t> tst(n + 1, 0);
    for (int64_t k = 0; k < nnz; ++k) ++tst[ci[k] + 1];
    for (int64_t i = 0; i < n; ++i) tst[i + 1] += tst[i];
    std::vector<int32_t> trow(nnz);
    std::vector<double> tval(nnz);
    {
        std::vector<int64_t> next(tst.begin(), tst.end() - 1);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int64_t d = next[ci[k]]++;
                trow[d] = (int32_t)i;
                tval[d] = val[k];
            }
    }
    auto merge = [&](int64_t u, int32_t* nb, double* w) -> int64_t {
        int64_t p = rp[u], pe = rp[u + 1], q = tst[u], qe = tst[u + 1], cnt = 0;
        while (p < pe || q < qe) {
            const int64_t jp = p < pe ? ci[p] : INT64_MAX;
            const int64_t jq = q < qe ? (int64_t)trow[q] : INT64_MAX;
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
            if (j == u) continue;       // diagonal ignored (graph.cpp:30)
            const double wt = 0.5 * s;
            if (wt <= 0.0) continue;    // w <= 0 dropped (graph.cpp:41); NaN kept, as there
            if (nb) {
                nb[cnt] = (int32_t)j;
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

}  // namespace

Adjacency graph_from_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val) {
    const int64_t nnz = rp[n];
    // Structurally symmetric fast path: w(u, j) from row u and the mirror
    // entry found by binary search in row j; no transpose.
    std::vector<double> wk(nnz);
    int missing = 0;
#pragma omp parallel for schedule(dynamic, 2048) reduction(| : missing)
    for (int64_t u = 0; u < n; ++u) {
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
            const int64_t j = ci[k];
            if (j == u) {
                wk[k] = 0.0;
                continue;
            }
            const int64_t* b = ci + rp[j];
            const int64_t* e = ci + rp[j + 1];
            const int64_t* it = std::lower_bound(b, e, u);
            if (it == e || *it != u) {
                missing = 1;
                break;
            }
            wk[k] = 0.5 * (std::fabs(val[k]) + std::fabs(val[it - ci]));
        }
    }
    if (missing) return graph_general(n, rp, ci, val);
    Adjacency g;
    g.n = n;
    g.start.assign(n + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; ++u) {
        int64_t c = 0;
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k)
            if (ci[k] != u && !(wk[k] <= 0.0)) ++c;  // same keep rule as graph.cpp:41
        g.start[u + 1] = c;
    }
    for (int64_t u = 0; u < n; ++u) g.start[u + 1] += g.start[u];
    g.nbr.resize(g.start[n]);
    g.w.resize(g.start[n]);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < n; ++u) {
        int64_t d = g.start[u];
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k)
            if (ci[k] != u && !(wk[k] <= 0.0)) {
                g.nbr[d] = (int32_t)ci[k];
                g.w[d] = wk[k];
                ++d;
            }
    }
    return g;
}

// Stable gather perm[i] = next[assignment[i]]++ (partition.cpp:14-41), in
// parallel: each thread counts its contiguous chunk per block, the per-block
// offsets of the chunks follow from a prefix over (block, thread), and every
// thread scatters its chunk in order — the same perm as the serial loop.
void partition_from_assignment(int64_t n, const int64_t* assignment, int64_t s, int64_t* perm,
                               int64_t* block_starts) {
    if (s < 1 || s > n) fail(HPBJ_EINVAL, "partition: block count must satisfy 1 <= s <= n");
    const int T = n >= (1 << 16) ? std::max(1, std::min(omp_get_max_threads(), 64)) : 1;
    const int64_t chunk = (n + T - 1) / T;
    std::vector<int64_t> cnt((size_t)T * s, 0);  // [thread][block]
    int bad = 0;
#pragma omp parallel for schedule(static, 1) reduction(| : bad)
    for (int t = 0; t < T; ++t) {  // every chunk exactly once, whatever the team size
        int64_t* c = cnt.data() + (size_t)t * s;
        for (int64_t i = t * chunk; i < std::min(n, (t + 1) * chunk); ++i) {
            const int64_t b = assignment[i];
            if (b < 0 || b >= s) bad = 1;
            else ++c[b];
        }
    }
    if (bad) fail(HPBJ_ERANGE, "partition: block index out of range");
    block_starts[0] = 0;
    for (int64_t b = 0; b < s; ++b) {
        int64_t off = block_starts[b];
        for (int t = 0; t < T; ++t) {
            const int64_t k = cnt[(size_t)t * s + b];
            cnt[(size_t)t * s + b] = off;
            off += k;
        }
        if (off == block_starts[b]) fail(HPBJ_EINVAL, "partition: block " + std::to_string(b) + " is empty");
        block_starts[b + 1] = off;
    }
#pragma omp parallel for schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        int64_t* next = cnt.data() + (size_t)t * s;
        for (int64_t i = t * chunk; i < std::min(n, (t + 1) * chunk); ++i) perm[i] = next[assignment[i]]++;
    }
}

namespace {

// Host buffer on transparent huge pages (2 MB-aligned anonymous mapping +
// MADV_HUGEPAGE): the BFS and the refinement sweep access these arrays at
// random, and with 4 KB pages most of those accesses also miss the TLB.
template <class T>
struct HBuf {
    T* p = nullptr;
    size_t n = 0, len = 0;
    void* base = nullptr;
    HBuf() = default;
    HBuf(const HBuf&) = delete;
    HBuf& operator=(const HBuf&) = delete;
    ~HBuf() { release(); }
    void release() {
        if (base) munmap(base, len);
        base = nullptr;
        p = nullptr;
        n = 0;
    }
    void fit(size_t m) {
        if (m <= n) return;
        release();
        constexpr size_t kHuge = size_t(2) << 20;
        const size_t bytes = (m * sizeof(T) + kHuge - 1) / kHuge * kHuge;
        len = bytes + kHuge;
        base = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (base == MAP_FAILED) {
            base = nullptr;
            throw std::bad_alloc();
        }
        const uintptr_t a = (reinterpret_cast<uintptr_t>(base) + kHuge - 1) & ~(uintptr_t)(kHuge - 1);
        p = reinterpret_cast<T*>(a);
        madvise(p, bytes, MADV_HUGEPAGE);
        n = m;
    }
    T* data() { return p; }
    const T* data() const { return p; }
    size_t size() const { return n; }
    T& operator[](size_t i) { return p[i]; }
};

// Reusable host workspace (repeated setups — e.g. the transient Newton
// sequence — never page-fault fresh buffers).
struct PartWork {
    HBuf<double> wk;
    HBuf<int64_t> deg;
    HBuf<int32_t> state;
    HBuf<int32_t> queue;
    HBuf<uint64_t> taken;
    HBuf<int16_t> state16;
    HBuf<int32_t> order;
    HBuf<int64_t> dstart;
    HBuf<int64_t> sizes;
    HBuf<double> conn;
    HBuf<int32_t> adj_start;
    HBuf<int32_t> adj_nbr;
    HBuf<double> adj_w;
    // refinement (parallel sweep)
    HBuf<uint8_t> spec;  // S per node
    HBuf<uint8_t> fl;
    HBuf<uint64_t> fbits;
    // region growing
    HBuf<int32_t> aorder;
    HBuf<uint32_t> ell;
};
thread_local PartWork t_work;

template <class T>
void fit(std::vector<T>& v, size_t n) {
    if (v.size() < n) v.resize(n);
}
template <class T>
void fit(HBuf<T>& v, size_t n) {
    v.fit(n);
}

// Graph view: neighbours of u are idx[st[u] .. st[u+1]) with weights w[k];
// deg[u] = st[u+1] - st[u]. Every edge takes part in growing and refinement
// (partition.cpp:96-97, :122-125); dropping w <= 0 pairs is graph_from_matrix's
// job (graph.cpp:41) and happens when the view is built (partition_csr).
template <class Idx, class Off = int64_t>
struct GraphView {
    int64_t n;
    const Off* st;
    const Idx* idx;
    const double* w;
    const int64_t* deg;
};

// The reference's decision for node u (partition.cpp:117-141) against a given
// state: -2 skipped (source block of size <= 1), -1 stays, else the target
// block. conn (all zero on entry and on exit) and tch are the caller's.
constexpr int kSmallDeg = 16;

template <class Idx, class Off, class S>
inline int32_t refine_decide(const GraphView<Idx, Off>& g, const S* state, const int64_t* sizes, int64_t cap,
                             double* conn, int32_t* tch, int64_t u) {
    const Off* st = g.st;
    const Idx* nb = g.idx;
    const double* w = g.w;
    const int32_t bu = state[u];
    if (sizes[bu] <= 1) return -2;
    // Interior fast path: with every neighbour in bu the reference touches
    // only bu, which is never a candidate -> no move (no floating-point work).
    {
        Off k = st[u];
        const Off ke = st[u + 1];
        while (k < ke && state[nb[k]] == bu) ++k;
        if (k == ke) return -1;
    }
    const Off k0 = st[u], k1 = st[u + 1];
    if (k1 - k0 <= kSmallDeg) {
        // The touched blocks in first-touch order with their sums kept in
        // registers instead of the s-long conn table (random accesses into
        // it were most of a node's cost). Each sum starts at 0.0 and adds the
        // weights in neighbour order, as conn[bv] does (partition.cpp:121-125).
        // The reference lists a block once more if its sum returns to 0.0
        // (w <= 0 edges of explicit graphs); such a repeat compares equal to
        // its first occurrence and never changes the choice below.
        int32_t blk[kSmallDeg];
        double cw[kSmallDeg];
        int nblk = 0;
        for (Off k = k0; k < k1; ++k) {
            const int32_t bv = state[nb[k]];
            int j = 0;
            while (j < nblk && blk[j] != bv) ++j;
            if (j == nblk) {
                blk[j] = bv;
                cw[j] = 0.0;
                ++nblk;
            }
            cw[j] += w[k];
        }
        int bi = -1;
        double cbest = 0.0, cbu = 0.0;
        for (int t = 0; t < nblk; ++t) {
            const int32_t bv = blk[t];
            if (bv == bu) {
                cbu = cw[t];
                continue;
            }
            if (sizes[bv] + 1 > cap) continue;
            if (bi < 0 || cw[t] > cbest || (cw[t] == cbest && bv < blk[bi])) {
                bi = t;
                cbest = cw[t];
            }
        }
        return (bi >= 0 && cbest > cbu) ? blk[bi] : -1;
    }
    int nt = 0;
    for (Off k = k0; k < k1; ++k) {
        const int32_t bv = state[nb[k]];
        tch[nt] = bv;  // recorded while its conn is still 0.0 (partition.cpp:123-124)
        nt += conn[bv] == 0.0;
        conn[bv] += w[k];
    }
    int32_t best = -1;
    for (int t = 0; t < nt; ++t) {
        const int32_t bv = tch[t];
        if (bv == bu || sizes[bv] + 1 > cap) continue;
        if (best < 0 || conn[bv] > conn[best] || (conn[bv] == conn[best] && bv < best)) best = bv;
    }
    const int32_t dec = (best >= 0 && conn[best] > conn[bu]) ? best : -1;
    for (int t = 0; t < nt; ++t) conn[tch[t]] = 0.0;
    return dec;
}

template <class Idx, class Off>
int64_t max_degree(const GraphView<Idx, Off>& g) {
    int64_t maxdeg = 0;
#pragma omp parallel for schedule(static) reduction(max : maxdeg) if (g.n > 65536)
    for (int64_t u = 0; u < g.n; ++u) maxdeg = std::max<int64_t>(maxdeg, (int64_t)(g.st[u + 1] - g.st[u]));
    return maxdeg;
}

// One refinement sweep (partition.cpp:117-141) in the reference's u order
// over block ids of type S (moves applied immediately, as there). Returns
// the number of moves.
template <class Idx, class Off, class S>
int64_t refine_sweep(const GraphView<Idx, Off>& g, S* state, int64_t* sizes, int64_t cap, double* conn, bool pf) {
    const int64_t n = g.n;
    const Off* st = g.st;
    const Idx* nb = g.idx;
    std::vector<int32_t> tch(max_degree(g) + 1);
    int64_t moves = 0;
    constexpr int64_t kRefAhead = 8;
    for (int64_t u = 0; u < n; ++u) {
        if (pf && u + kRefAhead < n) {
            const int64_t f = u + kRefAhead;
            for (Off k = st[f]; k < st[f + 1] && k < st[f] + 16; ++k) __builtin_prefetch(&state[nb[k]], 0, 1);
        }
        const int32_t d = refine_decide(g, state, sizes, cap, conn, tch.data(), u);
        if (d < 0) continue;
        const int32_t bu = state[u];
        state[u] = (S)d;
        --sizes[bu];
        ++sizes[d];
        ++moves;
    }
    return moves;
}

// The same sweep, exact, with the scan work spread over T threads.
//
// The sequential sweep's decision for u reads (a) the block of every
// neighbour v — final if v < u, initial if v > u (a node changes only at its
// own step) — and (b) the block sizes at step u. Phase 1 (parallel): thread t
// sweeps its contiguous range [lo, hi) as if it were alone — neighbours in
// earlier ranges at their initial blocks, its own moves applied to a private
// copy `spec` and private sizes — and records, for every node with a block
// more strongly connected than its own, the candidates in the reference's
// preference order (conn desc, block asc), each with conn > conn[bu]. For
// such a node the reference's decision under ANY sizes is: skip if
// sizes[bu] <= 1, else the first candidate with sizes + 1 <= cap, else stay;
// every other node stays whatever the sizes. Phase 2 (sequential, in u order,
// on the real state): decide every recorded node from its list with the real
// sizes. A node's list is exact unless some lower neighbour's real final block
// differs from the one phase 1 assumed for it (its `spec` block in the same
// range, its initial block across ranges); whenever a node's real block
// differs from what a higher neighbour assumed, that neighbour is marked dirty
// and phase 2 recomputes it from the real state (refine_decide), as the
// sequential sweep would. Phase 2 only scans the neighbours of nodes whose
// outcome differs from an assumption, so its cost is the cross-range
// boundary plus the few decisions the size limits change.
template <class Idx, class Off, class S>
int64_t refine_sweep_par(const GraphView<Idx, Off>& g, S* state, int64_t* sizes, int64_t s, int64_t cap, int T) {
    const int64_t n = g.n;
    const Off* st = g.st;
    const Idx* nb = g.idx;
    const double* w = g.w;
    const auto t_p0 = std::chrono::steady_clock::now();
    PartWork& W = t_work;
    fit(W.spec, n * sizeof(S));
    fit(W.fl, n);
    S* spec = reinterpret_cast<S*>(W.spec.data());
    // per node: bit 0 recorded, bit 1 has a higher neighbour in a later range, bit 2 dirty
    uint8_t* fl = W.fl.data();
    std::vector<std::vector<int32_t>> rec(T);
    std::vector<int64_t> lo(T + 1);
    for (int t = 0; t <= T; ++t) lo[t] = n * t / T;
    std::vector<int64_t> sizes0(sizes, sizes + s);
#pragma omp parallel num_threads(T)
    {
        const int t = omp_get_thread_num();
        const int64_t a = lo[t], e = lo[t + 1];
        std::memcpy(spec + a, state + a, sizeof(S) * (e - a));
        std::vector<double> conn(s, 0.0);
        std::vector<int64_t> sz(sizes0);
        std::vector<int32_t> tch, cand;
        std::vector<int32_t>& R = rec[t];
        R.reserve((size_t)(e - a) / 2);
        for (int64_t u = a; u < e; ++u) {
            const int32_t bu = spec[u];
            bool cross = false, inter = true;
            for (Off k = st[u]; k < st[u + 1]; ++k) {
                const int64_t v = nb[k];
                cross |= v >= e;
                const int32_t bv = (v >= a && v < e) ? (int32_t)spec[v] : (int32_t)state[v];
                inter &= bv == bu;
            }
            fl[u] = cross ? 2 : 0;
            if (inter) continue;  // only bu touched: stays under any sizes
            if (st[u + 1] - st[u] <= kSmallDeg) {  // sums in registers (see refine_decide)
                int32_t blk[kSmallDeg];
                double cw[kSmallDeg];
                int nblk = 0;
                for (Off k = st[u]; k < st[u + 1]; ++k) {
                    const int64_t v = nb[k];
                    const int32_t bv = (v >= a && v < e) ? (int32_t)spec[v] : (int32_t)state[v];
                    int j = 0;
                    while (j < nblk && blk[j] != bv) ++j;
                    if (j == nblk) {
                        blk[j] = bv;
                        cw[j] = 0.0;
                        ++nblk;
                    }
                    cw[j] += w[k];
                }
                double cbu = 0.0;
                for (int t = 0; t < nblk; ++t)
                    if (blk[t] == bu) cbu = cw[t];
                bool nan = std::isnan(cbu);
                int ci[kSmallDeg];
                int nc = 0;
                for (int t = 0; t < nblk; ++t) {
                    nan |= std::isnan(cw[t]);
                    if (blk[t] != bu && cw[t] > cbu) {  // insertion by (sum desc, block asc)
                        int q = nc++;
                        while (q > 0 && (cw[ci[q - 1]] < cw[t] || (cw[ci[q - 1]] == cw[t] && blk[ci[q - 1]] > blk[t]))) {
                            ci[q] = ci[q - 1];
                            --q;
                        }
                        ci[q] = t;
                    }
                }
                if (nan) {  // NaN weights (explicit graphs): no total order; phase 2 decides it
                    fl[u] |= 4;
                    continue;
                }
                if (nc == 0) continue;
                fl[u] |= 1;
                R.push_back(nc);
                for (int q = 0; q < nc; ++q) R.push_back(blk[ci[q]]);
                if (sz[bu] <= 1) continue;  // speculative decision with this range's sizes
                for (int q = 0; q < nc; ++q) {
                    const int32_t bv = blk[ci[q]];
                    if (sz[bv] + 1 <= cap) {
                        spec[u] = (S)bv;
                        --sz[bu];
                        ++sz[bv];
                        break;
                    }
                }
                continue;
            }
            tch.clear();
            for (Off k = st[u]; k < st[u + 1]; ++k) {
                const int64_t v = nb[k];
                const int32_t bv = (v >= a && v < e) ? (int32_t)spec[v] : (int32_t)state[v];
                if (conn[bv] == 0.0) tch.push_back(bv);
                conn[bv] += w[k];
            }
            cand.clear();
            bool nan = std::isnan(conn[bu]);
            for (int32_t bv : tch) {
                nan |= std::isnan(conn[bv]);
                if (bv != bu && conn[bv] > conn[bu]) cand.push_back(bv);
            }
            if (nan) {  // NaN weights (explicit graphs): no total order; phase 2 decides it
                for (int32_t bv : tch) conn[bv] = 0.0;
                fl[u] |= 4;
                continue;
            }
            std::sort(cand.begin(), cand.end(), [&](int32_t x, int32_t y) {
                return conn[x] > conn[y] || (conn[x] == conn[y] && x < y);
            });
            for (int32_t bv : tch) conn[bv] = 0.0;
            if (cand.empty()) continue;
            fl[u] |= 1;
            R.push_back((int32_t)cand.size());
            R.insert(R.end(), cand.begin(), cand.end());
            if (sz[bu] <= 1) continue;  // speculative decision with this range's sizes
            for (int32_t bv : cand)
                if (sz[bv] + 1 <= cap) {
                    spec[u] = (S)bv;
                    --sz[bu];
                    ++sz[bv];
                    break;
                }
        }
    }
    const auto t_p1 = std::chrono::steady_clock::now();
    // phase 2
    std::vector<double> conn(s, 0.0);
    int64_t ndirty = 0, nrec = 0, nscan = 0;
    const bool dbg = getenv("HPBJ_DEBUG") != nullptr;
    uint64_t cyc_dirty = 0, cyc_scan = 0;
    std::vector<int32_t> tch(max_degree(g) + 1);
    int64_t moves = 0;
    // flagged nodes as a bitmap: phase 2 visits only them (set bits in
    // ascending order; a dirty mark on a higher node of the same word is
    // picked up by re-reading the word)
    const int64_t nw = (n + 63) / 64;
    fit(W.fbits, nw);
    uint64_t* fb = W.fbits.data();
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t w = 0; w < nw; ++w) {
        uint64_t bits = 0;
        const int64_t u0 = w * 64, ue = std::min<int64_t>(n, u0 + 64);
        for (int64_t u = u0; u < ue; ++u) bits |= (uint64_t)(fl[u] != 0) << (u - u0);
        fb[w] = bits;
    }
    for (int t = 0; t < T; ++t) {
        const int32_t* r = rec[t].data();
        const int64_t a = lo[t], e = lo[t + 1];
        if (a >= e) continue;
        for (int64_t w = a >> 6; w <= (e - 1) >> 6; ++w) {
            uint64_t win = ~0ull;
            if (w == (a >> 6)) win &= ~0ull << (a & 63);
            if (w == ((e - 1) >> 6)) win &= ~0ull >> (63 - ((e - 1) & 63));
            uint64_t bits = fb[w] & win;
            while (bits) {
                const int i = __builtin_ctzll(bits);
                const int64_t u = w * 64 + i;
                const uint8_t f = fl[u];
                const int32_t bu = state[u];
                int32_t d = -1;
                ndirty += (f & 4) != 0;
                nrec += (f & 1) != 0;
                if (f & 4) {
                    const uint64_t c0 = dbg ? __rdtsc() : 0;
                    d = refine_decide(g, state, sizes, cap, conn.data(), tch.data(), u);
                    if (dbg) cyc_dirty += __rdtsc() - c0;
                    if (f & 1) r += 1 + r[0];
                } else if (f & 1) {
                    const int nc = r[0];
                    if (sizes[bu] > 1)
                        for (int k = 1; k <= nc; ++k)
                            if (sizes[r[k]] + 1 <= cap) {
                                d = r[k];
                                break;
                            }
                    r += 1 + nc;
                }
                const int32_t fin = d >= 0 ? d : bu;
                if (d >= 0) {
                    state[u] = (S)d;
                    --sizes[bu];
                    ++sizes[d];
                    ++moves;
                }
                const bool same_diff = fin != (int32_t)spec[u];  // what later nodes of this range assumed
                const bool cross_diff = (f & 2) && fin != bu;    // what later ranges assumed (the initial block)
                nscan += same_diff || cross_diff;
                if (same_diff || cross_diff) {
                    const uint64_t c0 = dbg ? __rdtsc() : 0;
                    for (Off k = st[u]; k < st[u + 1]; ++k) {
                        const int64_t v = nb[k];
                        if (v <= u) continue;
                        if (v < e ? same_diff : cross_diff) {
                            fl[v] |= 4;
                            fb[v >> 6] |= 1ull << (v & 63);
                        }
                    }
                    if (dbg) cyc_scan += __rdtsc() - c0;
                }
                bits = i == 63 ? 0ull : fb[w] & win & (~0ull << (i + 1));
            }
        }
    }
    if (getenv("HPBJ_DEBUG"))
        fprintf(stderr,
                "[hpbj]   refine: T=%d phase1 %.1f ms, phase2 %.1f ms, %lld recorded, %lld recomputed (%.1f Mcyc), "
                "%lld scanned (%.1f Mcyc)\n",
                T, std::chrono::duration<double, std::milli>(t_p1 - t_p0).count(),
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_p1).count(),
                (long long)nrec, (long long)ndirty, cyc_dirty * 1e-6, (long long)nscan, cyc_scan * 1e-6);
    return moves;
}

// Share of nodes (every 61st sampled) with a higher neighbour in a later one
// of T equal node ranges: the parallel sweep's phase 2 recomputes about that
// share of the moved nodes' neighbours, so on graphs whose edges ignore the
// node order (random couplings: configs 2 and 4) the one-thread sweep is
// faster.
template <class Idx, class Off>
double cross_range_fraction(const GraphView<Idx, Off>& g, int T) {
    int64_t hit = 0, cnt = 0;
    for (int64_t u = 0; u < g.n; u += 61) {
        const int64_t e = (u * T / g.n + 1) * g.n / T;
        bool c = false;
        for (Off k = g.st[u]; k < g.st[u + 1]; ++k) c |= (int64_t)g.idx[k] >= e;
        hit += c;
        ++cnt;
    }
    return cnt ? (double)hit / cnt : 0.0;
}

// Fixed-stride neighbour records for region growing: 8 ids per node, the
// degree in the top 4 bits of the first (15: longer row, read elsewhere).
// Unused slots hold n, a node whose taken bit is always set (pushes nothing),
// so every record is walked as 8 branch-free pushes.
template <class DegFn, class NbrFn>
void build_ell(int64_t n, uint32_t* ell, DegFn deg, NbrFn nbr) {
#pragma omp parallel for schedule(static, 4096)
    for (int64_t u = 0; u < n; ++u) {
        uint32_t* e = ell + (size_t)u * 8;
        const int64_t d = deg(u);
        if (d > 8) {
            e[0] = 0xFu << 28;
            continue;
        }
        for (int i = 0; i < 8; ++i) e[i] = i < d ? nbr(u, i) : (uint32_t)n;
        e[0] |= (uint32_t)d << 28;
    }
}

struct GrowOpts {
    int ahead = 16;     // prefetch distance (popped nodes), fixed-stride records
    int ahead_csr = 6;  // the same with st + nb (two dependent lines per node)
    int ell = -1;        // fixed-stride neighbour records (-1: for n >= 2^21)
    bool pf = true;
};
inline GrowOpts grow_opts() {
    GrowOpts o;
    if (const char* e = getenv("HPBJ_GROW_PF")) o.ahead = o.ahead_csr = atoi(e);
    if (const char* e = getenv("HPBJ_GROW_ELL")) o.ell = atoi(e);
    return o;
}

// Region growing (partition.cpp:74-103). The free/taken test reads a bitmap
// (n bits: cache-resident) instead of the state array. Returns the connected
// nodes left unassigned.
template <bool ELL, class Idx, class Off, class S>
int64_t grow_blocks(const GraphView<Idx, Off>& g, const uint32_t* ell, const int32_t* order, int64_t connected,
                    int64_t s, int64_t cap, int64_t* sizes, uint64_t* taken, int32_t* queue, S* state,
                    const GrowOpts& go, HBuf<int32_t>& aorder_buf, const int64_t* raw_rp = nullptr,
                    const int64_t* raw_ci = nullptr) {
    const int64_t n = g.n;
    const Off* st = g.st;
    const Idx* nb = g.idx;
    const int K = ELL ? go.ahead : go.ahead_csr;
    const bool pf = go.pf && n > (1 << 18) && K > 0;
    // popped nodes in order (a sequential stream); block ids are written
    // from it afterwards in parallel instead of one random store per pop
    fit(aorder_buf, connected + 1);
    int32_t* ao = aorder_buf.data();
    int64_t fill = 0;
    int64_t cursor = 0;
    int64_t connected_left = connected;
    auto push_csr = [&](int32_t u, int64_t& tail) {
        for (Off k = st[u]; k < st[u + 1]; ++k) {  // branch-free push of the free neighbours
            const int32_t v = (int32_t)nb[k];
            uint64_t& word = taken[v >> 6];
            const uint64_t bit = 1ull << (v & 63);
            queue[tail] = v;
            tail += (word & bit) == 0;
            word |= bit;
        }
    };
    int64_t b = 0;
    for (; b < s && connected_left > 0; ++b) {
        const int64_t blocks_left = s - b;
        int64_t target = (connected_left + blocks_left - 1) / blocks_left;
        target = std::min(target, cap);
        int64_t head = 0, tail = 0;
        int64_t grown = 0;
        while (grown < target) {
            if (head == tail) {  // queue empty: every taken node is assigned
                while (cursor < connected && ((taken[order[cursor] >> 6] >> (order[cursor] & 63)) & 1ull)) ++cursor;
                if (cursor == connected) break;
                const int32_t sd = order[cursor];
                queue[tail++] = sd;
                taken[sd >> 6] |= 1ull << (sd & 63);
            }
            if constexpr (ELL) {
                if (pf && head + K < tail) __builtin_prefetch(ell + (size_t)queue[head + K] * 8, 0, 3);
            } else {
                if (pf && head + 2 * K < tail) __builtin_prefetch(st + queue[head + 2 * K], 0, 1);
                if (pf && head + K < tail) {  // prefetch the adjacency of a node popped soon
                    const int32_t f = queue[head + K];
                    __builtin_prefetch(nb + st[f], 0, 1);
                }
            }
            const int32_t u = queue[head++];
            ao[fill++] = u;
            ++grown;
            --connected_left;
            if constexpr (ELL) {
                const uint32_t* e = ell + (size_t)u * 8;
                const uint32_t h = e[0];
                const uint32_t d = h >> 28;
                if (d <= 8) {  // padding slots name node n (always taken)
#pragma GCC unroll 8
                    for (uint32_t i = 0; i < 8; ++i) {
                        const int32_t v = (int32_t)(i == 0 ? (h & 0x0FFFFFFFu) : e[i]);
                        uint64_t& word = taken[v >> 6];
                        const uint64_t bit = 1ull << (v & 63);
                        queue[tail] = v;
                        tail += (word & bit) == 0;
                        word |= bit;
                    }
                } else if (raw_rp) {  // graph = CSR minus the diagonal, built concurrently: read the CSR
                    for (int64_t k = raw_rp[u]; k < raw_rp[u + 1]; ++k) {
                        const int32_t v = (int32_t)raw_ci[k];
                        if (v == u) continue;
                        uint64_t& word = taken[v >> 6];
                        const uint64_t bit = 1ull << (v & 63);
                        queue[tail] = v;
                        tail += (word & bit) == 0;
                        word |= bit;
                    }
                } else {
                    push_csr(u, tail);
                }
            } else {
                push_csr(u, tail);
            }
        }
        sizes[b] = grown;
        for (int64_t q = head; q < tail; ++q) taken[queue[q] >> 6] &= ~(1ull << (queue[q] & 63));  // queue.clear()
    }
    {  // block ids from the assignment-order list
        std::vector<int64_t> off(b + 1, 0);
        for (int64_t i = 0; i < b; ++i) off[i + 1] = off[i] + sizes[i];
#pragma omp parallel for schedule(dynamic, 64) if (n > 65536)
        for (int64_t i = 0; i < b; ++i)
            for (int64_t k = off[i]; k < off[i + 1]; ++k) state[ao[k]] = (S)i;
    }
    return connected_left;
}

// Region growing overlapped with the graph build: the grow reads prebuilt
// fixed-stride records of A's off-diagonal pattern (and A itself for rows
// longer than a record) while `during_grow` computes the weights and the
// refinement view on the other cores; it returns false when the weighted
// graph turns out not to be A's pattern (structurally unsymmetric), and the
// partition is then abandoned (partition_view returns false).
struct GrowPipeline {
    const uint32_t* ell = nullptr;
    const int64_t* rp = nullptr;
    const int64_t* ci = nullptr;
    std::function<bool()> during_grow;
};

template <class Idx, class Off>
bool partition_view(const GraphView<Idx, Off>& g, int64_t s, double tol, int64_t* assignment,
                    const GrowPipeline* pl = nullptr) {
    const int64_t n = g.n;
    if (s < 1) fail(HPBJ_EINVAL, "partition_graph: s must be >= 1");
    if (s > n) fail(HPBJ_EINVAL, "partition_graph: s exceeds node count");
    if (tol < 0.0) fail(HPBJ_EINVAL, "partition_graph: negative imbalance tolerance");
    if (n >= INT32_MAX) fail(HPBJ_EINVAL, "partition_graph: n must be < 2^31");

    // cap formula verbatim (partition.cpp:67-69)
    const int64_t cap = std::max<int64_t>(
        static_cast<int64_t>(std::ceil(static_cast<double>(n) / s * (1.0 + tol))),
        (n + s - 1) / s);

    const auto t_pv0 = std::chrono::steady_clock::now();
    PartWork& W = t_work;
    const Off* st = g.st;
    const Idx* nb = g.idx;
    const int64_t* deg = g.deg;

    fit(W.sizes, s);
    int64_t* sizes = W.sizes.data();
    std::fill(sizes, sizes + s, int64_t(0));

    // Seed order: degree desc, index asc — a stable counting sort on
    // maxdeg - deg, parallel over contiguous chunks (per-chunk histograms, a
    // prefix over (key, chunk), in-order scatter per chunk).
    int64_t maxdeg = 0, connected = 0;
#pragma omp parallel for schedule(static) reduction(max : maxdeg) reduction(+ : connected) if (n > 65536)
    for (int64_t v = 0; v < n; ++v) {
        maxdeg = std::max(maxdeg, (int64_t)deg[v]);
        connected += deg[v] > 0;
    }
    fit(W.order, connected + 1);
    int32_t* order = W.order.data();
    {
        const int T = n > 65536 ? std::max(1, std::min(omp_get_max_threads(), 32)) : 1;
        const int64_t K = maxdeg + 1, chunk = (n + T - 1) / T;
        fit(W.dstart, (size_t)T * K);
        int64_t* cnt = W.dstart.data();  // [chunk][key]
        std::fill(cnt, cnt + (size_t)T * K, int64_t(0));
#pragma omp parallel for schedule(static, 1)
        for (int t = 0; t < T; ++t)
            for (int64_t v = t * chunk; v < std::min(n, (t + 1) * chunk); ++v)
                if (deg[v] > 0) ++cnt[(size_t)t * K + (maxdeg - deg[v])];
        // prefix over (key, chunk) with row-sequential passes over [chunk][key]
        // (a key-major walk strides T x K: ~100 ns per entry when the hub
        // rows of config 2 make K ~ 10^4)
        std::vector<int64_t> kst(K + 1, 0);
        for (int t = 0; t < T; ++t)
            for (int64_t k = 0; k < K; ++k) kst[k + 1] += cnt[(size_t)t * K + k];
        for (int64_t k = 0; k < K; ++k) kst[k + 1] += kst[k];
        for (int t = 0; t < T; ++t)
            for (int64_t k = 0; k < K; ++k) {
                const int64_t c = cnt[(size_t)t * K + k];
                cnt[(size_t)t * K + k] = kst[k];
                kst[k] += c;
            }
#pragma omp parallel for schedule(static, 1)
        for (int t = 0; t < T; ++t) {
            int64_t* nx = cnt + (size_t)t * K;
            for (int64_t v = t * chunk; v < std::min(n, (t + 1) * chunk); ++v)
                if (deg[v] > 0) order[nx[maxdeg - deg[v]]++] = (int32_t)v;
        }
    }

    const bool dbg = getenv("HPBJ_DEBUG") != nullptr;
    const auto t_seed = std::chrono::steady_clock::now();
    if (dbg)
        fprintf(stderr, "[hpbj]   seed order %.2f ms\n",
                std::chrono::duration<double, std::milli>(t_seed - t_pv0).count());

    fit(W.conn, s);
    double* conn = W.conn.data();
    std::fill(conn, conn + s, 0.0);
    fit(W.queue, n + 1);
    int32_t* queue = W.queue.data();
    fit(W.taken, (n + 64) / 64);
    uint64_t* taken = W.taken.data();  // bit v: assigned or queued
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t w = 0; w < (n + 64) / 64; ++w) taken[w] = 0ull;
    taken[n >> 6] |= 1ull << (n & 63);  // the records' padding node

    // Block ids are stored as S (16-bit when s fits: half the cache footprint
    // of the refinement's random neighbour lookups); -1 = unassigned.
    // Software prefetch in the sequential sweeps only once the per-node arrays
    // outgrow the core's L2 (measured on the B200 host: -7% on config 1's
    // 2.1e5 nodes without it, +20% on config 2's 10^6 random-graph nodes).
    const bool pf = n > (1 << 18);
    auto run = [&](auto* state) -> bool {
        using S = std::remove_pointer_t<decltype(state)>;
#pragma omp parallel for schedule(static) if (n > 65536)
        for (int64_t v = 0; v < n; ++v) state[v] = (S)-1;
        // Region growing (partition.cpp:74-103). The free/taken test reads a
        // bitmap (n bits: cache-resident) instead of the state array; state
        // receives the block id once per node.
        int64_t connected_left = connected;
        const GrowOpts go = grow_opts();
        if (pl) {
            std::exception_ptr gerr;
            const GraphView<Idx, Off> gg = g;  // during_grow replaces the caller's view
            std::thread thr([&] {
                try {
                    connected_left = grow_blocks<true>(gg, pl->ell, order, connected, s, cap, sizes, taken, queue,
                                                       state, go, W.aorder, pl->rp, pl->ci);
                } catch (...) {
                    gerr = std::current_exception();
                }
            });
            bool ok = false;
            try {
                ok = pl->during_grow();
            } catch (...) {
                thr.join();
                throw;
            }
            thr.join();
            if (gerr) std::rethrow_exception(gerr);
            if (!ok) return false;
        } else if (go.ell != 0 && (go.ell > 0 || n >= (int64_t(1) << 21)) && n < (int64_t(1) << 28)) {
            // fixed-stride neighbour records (8 ids, degree in the top bits of
            // the first): one cache line per popped node instead of st + nb
            const auto t_e0 = std::chrono::steady_clock::now();
            fit(W.ell, (size_t)n * 8);
            build_ell(n, W.ell.data(), [&](int64_t u) { return (int64_t)(st[u + 1] - st[u]); },
                      [&](int64_t u, int i) { return (uint32_t)nb[st[u] + i]; });
            if (dbg)
                fprintf(stderr, "[hpbj]   ell build %.1f ms\n",
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_e0).count());
            connected_left = grow_blocks<true>(g, W.ell.data(), order, connected, s, cap, sizes, taken, queue, state,
                                               go, W.aorder);
        } else {
            connected_left = grow_blocks<false>(g, nullptr, order, connected, s, cap, sizes, taken, queue, state, go,
                                                W.aorder);
        }
        const bool leftovers = connected < n || connected_left > 0;
        const auto t_grown = std::chrono::steady_clock::now();
        // Remaining nodes -> first block of minimal size (partition.cpp:105-112).
        if (leftovers) {
            using Key = std::pair<int64_t, int64_t>;  // (size, block)
            std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
            bool built = false;
            for (int64_t v = 0; v < n; ++v) {
                if (state[v] >= 0) continue;
                if (!built) {
                    for (int64_t b = 0; b < s; ++b) heap.push({sizes[b], b});
                    built = true;
                }
                const Key k = heap.top();
                heap.pop();
                state[v] = (S)k.second;
                ++sizes[k.second];
                heap.push({sizes[k.second], k.second});
            }
        }
        // HPBJ_PART_SEQ=1: the one-thread sweep (the parallel one is exact; the
        // switch exists for the equality test)
        // HPBJ_REFINE_T=k forces the parallel sweep with k ranges (tests)
        const bool seq = getenv("HPBJ_PART_SEQ") != nullptr;
        const char* force = getenv("HPBJ_REFINE_T");
        const int T = force ? std::max(2, atoi(force)) : std::min(omp_get_max_threads(), 32);
        const int64_t moves = (seq || (!force && (T < 2 || n <= 65536 || cross_range_fraction(g, T) > 0.25)))
                                  ? refine_sweep(g, state, sizes, cap, conn, pf)
                                  : refine_sweep_par(g, state, sizes, s, cap, T);
        if (dbg)
            fprintf(stderr, "[hpbj]   grow %.1f ms, refine %.1f ms (%lld moves)\n",
                    std::chrono::duration<double, std::milli>(t_grown - t_seed).count(),
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_grown).count(),
                    (long long)moves);
#pragma omp parallel for schedule(static) if (n > 65536)
        for (int64_t v = 0; v < n; ++v) assignment[v] = state[v];
        return true;
    };
    if (s <= 32767) {
        fit(W.state16, n);
        return run(W.state16.data());
    }
    fit(W.state, n);
    return run(W.state.data());
}

}  // namespace

void partition_adjacency(const Adjacency& g, int64_t s, double tol, int64_t* assignment) {
    std::vector<int64_t> deg(g.n);
    for (int64_t v = 0; v < g.n; ++v) deg[v] = g.start[v + 1] - g.start[v];
    GraphView<int32_t> view{g.n, g.start.data(), g.nbr.data(), g.w.data(), deg.data()};
    partition_view(view, s, tol, assignment);
}

// graph_from_matrix + partition_graph without materialising the adjacency
// when the pattern is structurally symmetric: the CSR itself is the graph,
// with per-entry weights (diagonal / w <= 0 entries masked as -1).
void partition_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* val, int64_t s, double tol,
                   int64_t* assignment) {
    const int64_t nnz = rp[n];
    if (nnz >= INT32_MAX) {  // beyond 4-byte offsets: the general (int64) path
        const Adjacency g = graph_general(n, rp, ci, val);
        partition_adjacency(g, s, tol, assignment);
        return;
    }
    const bool dbg = getenv("HPBJ_DEBUG") != nullptr;
    auto ms_since = [](std::chrono::steady_clock::time_point t) {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
    };
    PartWork& W = t_work;
    fit(W.wk, nnz);
    fit(W.deg, n);
    double* wk = W.wk.data();
    int64_t* deg = W.deg.data();
    // Weights of the upper-triangle entries, written to both the entry and its
    // mirror (one binary search per pair). w = 0.5 * (|a_pq| + |a_qp|) with
    // p < q, the reference's accumulation order (graph.cpp:24-33). The pattern
    // is symmetric iff every upper entry finds its mirror and the upper and
    // lower entry counts agree (the mirrors are then all the lower entries).
    // Returns true when the pattern is symmetric.
    auto weights = [&](int nthr) -> bool {
        const auto t_w0 = std::chrono::steady_clock::now();
        int missing = 0;
        int64_t nup = 0, nlo = 0;
#pragma omp parallel for num_threads(nthr) schedule(dynamic, 2048) reduction(| : missing) reduction(+ : nup, nlo)
        for (int64_t u = 0; u < n; ++u) {
            for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
                const int64_t j = ci[k];
                if (j < u) {
                    ++nlo;
                    continue;
                }
                if (j == u) {
                    wk[k] = -1.0;
                    continue;
                }
                ++nup;
                const int64_t* b = ci + rp[j];
                const int64_t* e = ci + rp[j + 1];
                const int64_t* it = std::lower_bound(b, e, u);
                if (it == e || *it != u) {
                    missing = 1;
                    continue;
                }
                const double wt = 0.5 * (std::fabs(val[k]) + std::fabs(val[it - ci]));
                wk[k] = wt;
                wk[it - ci] = wt;
            }
        }
        if (dbg) fprintf(stderr, "[hpbj]   weights %.1f ms\n", ms_since(t_w0));
        return !missing && nup == nlo;
    };
    // compact int32 adjacency (kept entries only): 4 B/neighbour and 4-byte
    // offsets for the sequential sweeps instead of 16 B (int64 column +
    // weight) per CSR entry; deg[] already holds the kept counts
    auto adjacency = [&](int nthr) -> GraphView<int32_t, int32_t> {
        const auto t_a0 = std::chrono::steady_clock::now();
        fit(W.adj_start, n + 1);
        int32_t* ast = W.adj_start.data();
        // offsets: chunked parallel prefix over deg
        const int C = std::max(1, std::min(nthr, 64));
        std::vector<int64_t> csum(C + 1, 0);
#pragma omp parallel for num_threads(nthr) schedule(static, 1)
        for (int c = 0; c < C; ++c) {
            int64_t t = 0;
            for (int64_t u = n * c / C; u < n * (c + 1) / C; ++u) t += deg[u];
            csum[c + 1] = t;
        }
        for (int c = 0; c < C; ++c) csum[c + 1] += csum[c];
#pragma omp parallel for num_threads(nthr) schedule(static, 1)
        for (int c = 0; c < C; ++c) {
            int64_t t = csum[c];
            for (int64_t u = n * c / C; u < n * (c + 1) / C; ++u) {
                ast[u] = (int32_t)t;
                t += deg[u];
            }
        }
        ast[n] = (int32_t)csum[C];
        fit(W.adj_nbr, ast[n] + 1);
        fit(W.adj_w, ast[n] + 1);
        int32_t* anb = W.adj_nbr.data();
        double* aw = W.adj_w.data();
#pragma omp parallel for num_threads(nthr) schedule(static, 4096)
        for (int64_t u = 0; u < n; ++u) {
            int64_t d = ast[u];
            for (int64_t k = rp[u]; k < rp[u + 1]; ++k)
                if (!(wk[k] <= 0.0)) {
                    anb[d] = (int32_t)ci[k];
                    aw[d] = wk[k];
                    ++d;
                }
        }
        if (dbg) fprintf(stderr, "[hpbj]   adjacency %.1f ms\n", ms_since(t_a0));
        return GraphView<int32_t, int32_t>{n, ast, anb, aw, deg};
    };

    // Large graphs: region growing needs only the pattern, so when A has no
    // explicit off-diagonal zero (every entry is an edge iff the pattern is
    // symmetric) it starts on A's off-diagonal pattern right away and the
    // weights + refinement view are built on the other cores meanwhile.
    const GrowOpts go = grow_opts();
    const int nth = omp_get_max_threads();
    if ((go.ell > 0 || (go.ell < 0 && n >= (int64_t(1) << 21))) && n < (int64_t(1) << 28) && nth >= 2 &&
        !getenv("HPBJ_GROW_NOPIPE")) {
        const auto t_q0 = std::chrono::steady_clock::now();
        int zero = 0;
        fit(W.ell, (size_t)n * 8);
        uint32_t* ell = W.ell.data();
        // one pass: off-diagonal counts, explicit zeros, the records
#pragma omp parallel for schedule(static, 4096) reduction(| : zero)
        for (int64_t u = 0; u < n; ++u) {
            uint32_t e[8];
            for (int i = 0; i < 8; ++i) e[i] = (uint32_t)n;
            int64_t d = 0;
            for (int64_t k = rp[u]; k < rp[u + 1]; ++k)
                if (ci[k] != u) {
                    if (d < 8) e[d] = (uint32_t)ci[k];
                    ++d;
                    zero |= val[k] == 0.0;
                }
            deg[u] = d;
            e[0] = d > 8 ? 0xFu << 28 : (e[0] | (uint32_t)d << 28);
            std::memcpy(ell + (size_t)u * 8, e, sizeof e);
        }
        if (!zero) {
            if (dbg) fprintf(stderr, "[hpbj]   pattern + records %.1f ms\n", ms_since(t_q0));
            GraphView<int32_t, int32_t> view{n, nullptr, nullptr, nullptr, deg};
            GrowPipeline pl;
            pl.ell = ell;
            pl.rp = rp;
            pl.ci = ci;
            // fewer threads than cores: the build's memory traffic slows the
            // latency-bound grow, and it has the grow's whole duration
            int wt = std::max(1, std::min(nth - 1, 8));
            if (const char* e = getenv("HPBJ_GROW_WT")) wt = std::max(1, atoi(e));
            pl.during_grow = [&, wt]() -> bool {
                if (!weights(wt)) return false;
                view = adjacency(wt);
                return true;
            };
            if (partition_view(view, s, tol, assignment, &pl)) return;
            // structurally unsymmetric: the graph has one-sided edges
            const Adjacency g = graph_general(n, rp, ci, val);
            partition_adjacency(g, s, tol, assignment);
            return;
        }
    }

    if (!weights(nth)) {
        const Adjacency g = graph_general(n, rp, ci, val);
        partition_adjacency(g, s, tol, assignment);
        return;
    }
#pragma omp parallel for schedule(static, 4096)
    for (int64_t u = 0; u < n; ++u) {
        int64_t d = 0;
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) d += !(wk[k] <= 0.0);
        deg[u] = d;
    }
    const GraphView<int32_t, int32_t> view = adjacency(nth);
    partition_view(view, s, tol, assignment);
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
        for (int64_t k = 0; k < g.start[n]; ++k) adj_nbr[k] = g.nbr[k];
        std::memcpy(adj_w, g.w.data(), sizeof(double) * g.start[n]);
    });
}

int hpbj_partition_graph(int64_t n, const int64_t* row_ptr, const int64_t* col,
                         const double* val, int64_t s, double imbalance_tol,
                         int64_t* assignment, int64_t* perm, int64_t* block_starts) {
    return guard(nullptr, [&] {
        const bool dbg = getenv("HPBJ_DEBUG") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t0 = now();
        check_csr(n, row_ptr, col, val);
        if (n >= INT32_MAX) fail(HPBJ_EINVAL, "partition_graph: n must be < 2^31");
        const auto t1 = now();
        const auto t2 = now();
        partition_csr(n, row_ptr, col, val, s, imbalance_tol, assignment);
        const auto t3 = now();
        partition_from_assignment(n, assignment, s, perm, block_starts);
        const auto t4 = now();
        if (dbg)
            fprintf(stderr, "[hpbj] partition: check %.1f graph %.1f grow+refine %.1f gather %.1f ms\n", ms(t0, t1),
                    ms(t1, t2), ms(t2, t3), ms(t3, t4));
    });
}

int hpbj_partition_adjacency(int64_t n, const int64_t* adj_start, const int64_t* adj_nbr,
                             const double* adj_w, int64_t s, double imbalance_tol,
                             int64_t* assignment, int64_t* perm, int64_t* block_starts) {
    return guard(nullptr, [&] {
        if (n < 0 || !adj_start) fail(HPBJ_EINVAL, "partition_graph: bad graph");
        if (n >= INT32_MAX) fail(HPBJ_EINVAL, "partition_graph: n must be < 2^31");
        Adjacency g;
        g.n = n;
        g.start.assign(adj_start, adj_start + n + 1);
        g.nbr.resize(adj_start[n]);
        for (int64_t k = 0; k < adj_start[n]; ++k) {
            if (adj_nbr[k] < 0 || adj_nbr[k] >= n) fail(HPBJ_EINVAL, "partition_graph: neighbour out of range");
            g.nbr[k] = (int32_t)adj_nbr[k];
        }
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
