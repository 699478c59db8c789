// Deterministic synthetic workloads for the five BASELINE.json configs.
//
// The paper's Table 1 (SuiteSparse circuit) matrices are not available
// offline; these seeded generators stand in for them with the shapes,
// sizes and value distributions BASELINE.json names (DESIGN.md §Workloads
// pins every ambiguity). Both the CUDA path and the CPU oracle consume the
// exact same CSR arrays produced here, so generator choices never affect
// parity.
//
// RNG: SplitMix64, the reference's own test convention
// (proj/tests/oracles.hpp:205-226, bjgmres_cli.cpp:67-79). Each logical
// stream (topology, source selection, slack, x_true, ...) has its own
// generator seeded by mix(seed, stream) so streams are independent.
//
// CSR assembly follows SparseMatrix::from_triplets (sparse_matrix.cpp:52-88):
// entries sorted by (row, col, value bits) and duplicates summed in that
// order, columns strictly increasing.
//
// Compiled with -ffp-contract=off so b = A*x_true matches the reference's
// sequential left-to-right FP64 row sums bit for bit.

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace {

struct Rng {
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double u01() { return static_cast<double>(next() >> 11) * 0x1p-53; }
    double uniform(double a, double b) { return a + (b - a) * u01(); }
    uint64_t below(uint64_t k) { return next() % k; }
    double normal() {  // Box-Muller, cosine branch only (pinned)
        const double u1 = 1.0 - u01();  // (0, 1]
        const double u2 = u01();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
    double lognormal(double mu, double sigma) { return std::exp(mu + sigma * normal()); }
};

uint64_t stream_seed(uint64_t seed, uint64_t stream) {
    Rng r(seed * 0x100000001b3ULL + stream * 0x9e3779b97f4a7c15ULL + 0x51ed2701ULL);
    return r.next();
}

struct Edge {
    int64_t i, j;
    double g;
};

struct Entry {
    int64_t col;
    double v;
};

enum Stream : uint64_t {
    kTopo = 1,
    kCond = 2,
    kSource = 3,
    kSlack = 4,
    kXtrue = 5,
    kPhase = 6,
};

struct Spec {
    int64_t n;
    std::vector<Edge> edges;
    double src_frac, src_lo, src_hi;  // controlled-source asymmetry
    double d_lo, d_hi;                // diagonal slack
};

// Controlled sources: one decision per *directed* entry, in edge order
// (i->j, then j->i). Selected entries get a_ij += u * g_ij.
struct Source {
    int64_t edge;
    int dir;  // 0: (i,j), 1: (j,i)
    double u;
};

std::vector<Source> pick_sources(const Spec& sp, uint64_t seed) {
    std::vector<Source> out;
    if (sp.src_frac <= 0.0) return out;
    Rng r(stream_seed(seed, kSource));
    for (int64_t e = 0; e < static_cast<int64_t>(sp.edges.size()); ++e)
        for (int dir = 0; dir < 2; ++dir)
            if (r.u01() < sp.src_frac) out.push_back({e, dir, r.uniform(sp.src_lo, sp.src_hi)});
    return out;
}

struct Csr {
    int64_t n = 0;
    std::vector<int64_t> rp, ci;
    std::vector<double> val;
    std::vector<double> b, xtrue;
};

// Assemble A from edges (with per-edge conductance scale), sources and slack.
Csr assemble(const Spec& sp, const std::vector<double>& gscale,
             const std::vector<Source>& src, const std::vector<double>& slack) {
    const int64_t n = sp.n;
    // directed off-diagonal triplets bucketed by row
    std::vector<int64_t> cnt(n + 1, 0);
    for (const Edge& e : sp.edges) {
        ++cnt[e.i + 1];
        ++cnt[e.j + 1];
    }
    for (const Source& s : src) {
        const Edge& e = sp.edges[s.edge];
        ++cnt[(s.dir == 0 ? e.i : e.j) + 1];
    }
    for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<Entry> trip(cnt[n]);
    std::vector<int64_t> next(cnt.begin(), cnt.end() - 1);
    for (size_t k = 0; k < sp.edges.size(); ++k) {
        const Edge& e = sp.edges[k];
        const double g = e.g * gscale[k];
        trip[next[e.i]++] = {e.j, -g};
        trip[next[e.j]++] = {e.i, -g};
    }
    for (const Source& s : src) {
        const Edge& e = sp.edges[s.edge];
        const double g = e.g * gscale[s.edge];
        if (s.dir == 0) trip[next[e.i]++] = {e.j, s.u * g};
        else trip[next[e.j]++] = {e.i, s.u * g};
    }
    Csr a;
    a.n = n;
    a.rp.assign(n + 1, 0);
    a.ci.reserve(cnt[n] + n);
    a.val.reserve(cnt[n] + n);
    std::vector<Entry> row;
    for (int64_t i = 0; i < n; ++i) {
        row.assign(trip.begin() + cnt[i], trip.begin() + cnt[i + 1]);
        std::sort(row.begin(), row.end(), [](const Entry& x, const Entry& y) {
            if (x.col != y.col) return x.col < y.col;
            return std::bit_cast<uint64_t>(x.v) < std::bit_cast<uint64_t>(y.v);
        });
        // sum duplicates (from_triplets rule), then insert the diagonal
        std::vector<Entry> merged;
        merged.reserve(row.size() + 1);
        for (size_t k = 0; k < row.size();) {
            const int64_t c = row[k].col;
            double sum = 0.0;
            while (k < row.size() && row[k].col == c) sum += row[k++].v;
            merged.push_back({c, sum});
        }
        double offsum = 0.0;
        for (const Entry& e : merged) offsum += std::fabs(e.v);
        const double diag = (1.0 + slack[i]) * offsum;
        bool placed = false;
        for (const Entry& e : merged) {
            if (!placed && e.col > i) {
                a.ci.push_back(i);
                a.val.push_back(diag);
                placed = true;
            }
            a.ci.push_back(e.col);
            a.val.push_back(e.v);
        }
        if (!placed) {
            a.ci.push_back(i);
            a.val.push_back(diag);
        }
        a.rp[i + 1] = static_cast<int64_t>(a.ci.size());
    }
    return a;
}

void finish_rhs(Csr& a, uint64_t xseed) {
    Rng r(xseed);
    a.xtrue.resize(a.n);
    for (double& v : a.xtrue) v = r.uniform(-1.0, 1.0);
    a.b.resize(a.n);
    for (int64_t i = 0; i < a.n; ++i) {
        double s = 0.0;
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) s += a.val[k] * a.xtrue[a.ci[k]];
        a.b[i] = s;
    }
}

std::vector<double> draw_slack(int64_t n, uint64_t seed, double lo, double hi) {
    Rng r(seed);
    std::vector<double> d(n);
    for (double& v : d) v = r.uniform(lo, hi);
    return d;
}

// Random circuit graph: a ring over all nodes plus `extra` random neighbours
// per node (self-picks redrawn; duplicate pairs kept and summed later).
// `half_extra`: one more random neighbour for every even node.
void circuit_edges(Spec& sp, uint64_t seed, int extra, bool half_extra, double mu,
                   double sigma) {
    const int64_t n = sp.n;
    Rng topo(stream_seed(seed, kTopo));
    Rng cond(stream_seed(seed, kCond));
    for (int64_t i = 0; i < n; ++i) sp.edges.push_back({i, (i + 1) % n, cond.lognormal(mu, sigma)});
    for (int64_t i = 0; i < n; ++i) {
        const int picks = extra + ((half_extra && (i % 2 == 0)) ? 1 : 0);
        for (int p = 0; p < picks; ++p) {
            int64_t j;
            do j = static_cast<int64_t>(topo.below(n)); while (j == i);
            sp.edges.push_back({i, j, cond.lognormal(mu, sigma)});
        }
    }
}

Csr build_config(int config, int step) {
    Spec sp{};
    uint64_t seed = 0;
    switch (config) {
        case 0: {  // small MNA-like circuit, n = 10,000
            seed = 1;
            sp.n = 10000;
            circuit_edges(sp, seed, 2, false, 0.0, 2.0);
            sp.src_frac = 0.05, sp.src_lo = -0.5, sp.src_hi = 0.5;
            sp.d_lo = 1e-3, sp.d_hi = 1e-1;
            break;
        }
        case 1: {  // 447 x 447 5-point power-grid mesh + 1% vias
            seed = 2;
            const int64_t nx = 447;
            sp.n = nx * nx;
            Rng topo(stream_seed(seed, kTopo));
            Rng cond(stream_seed(seed, kCond));
            for (int64_t iy = 0; iy < nx; ++iy)
                for (int64_t ix = 0; ix < nx; ++ix) {
                    const int64_t c = iy * nx + ix;
                    if (ix + 1 < nx) sp.edges.push_back({c, c + 1, cond.lognormal(0.0, 1.5)});
                    if (iy + 1 < nx) sp.edges.push_back({c, c + nx, cond.lognormal(0.0, 1.5)});
                }
            for (int64_t i = 0; i < sp.n; ++i) {
                if (topo.u01() < 0.01) {
                    const int64_t j = i + 10 + static_cast<int64_t>(topo.below(41));
                    const double g = cond.lognormal(1.0, 1.0);
                    if (j < sp.n) sp.edges.push_back({i, j, g});
                }
            }
            sp.src_frac = 0.0;
            sp.d_lo = 1e-4, sp.d_hi = 1e-2;
            break;
        }
        case 2: {  // 1M circuit, avg degree 6, 50 supply-rail hubs x 10,000
            seed = 3;
            sp.n = 1000000;
            circuit_edges(sp, seed, 2, false, 0.0, 2.0);
            Rng topo(stream_seed(seed, kTopo + 100));
            Rng cond(stream_seed(seed, kCond + 100));
            std::vector<uint8_t> is_hub(sp.n, 0);
            std::vector<int64_t> hubs;
            while (hubs.size() < 50) {
                const int64_t h = static_cast<int64_t>(topo.below(sp.n));
                if (!is_hub[h]) {
                    is_hub[h] = 1;
                    hubs.push_back(h);
                }
            }
            std::vector<int64_t> mark(sp.n, -1);
            for (int64_t hi = 0; hi < 50; ++hi) {
                const int64_t h = hubs[hi];
                int64_t got = 0;
                while (got < 10000) {
                    const int64_t j = static_cast<int64_t>(topo.below(sp.n));
                    if (j == h || mark[j] == hi) continue;
                    mark[j] = hi;
                    sp.edges.push_back({h, j, cond.lognormal(0.0, 1.0)});
                    ++got;
                }
            }
            sp.src_frac = 0.10, sp.src_lo = -0.8, sp.src_hi = 0.8;
            sp.d_lo = 1e-4, sp.d_hi = 5e-2;
            break;
        }
        case 3: {  // 160^3 7-point interconnect mesh + 0.5% long-range couplings
            seed = 4;
            const int64_t m = 160;
            sp.n = m * m * m;
            Rng topo(stream_seed(seed, kTopo));
            Rng cond(stream_seed(seed, kCond));
            sp.edges.reserve(3 * sp.n + sp.n / 100);
            for (int64_t iz = 0; iz < m; ++iz)
                for (int64_t iy = 0; iy < m; ++iy)
                    for (int64_t ix = 0; ix < m; ++ix) {
                        const int64_t c = (iz * m + iy) * m + ix;
                        if (ix + 1 < m) sp.edges.push_back({c, c + 1, cond.lognormal(0.0, 1.5)});
                        if (iy + 1 < m) sp.edges.push_back({c, c + m, cond.lognormal(0.0, 1.5)});
                        if (iz + 1 < m) sp.edges.push_back({c, c + m * m, cond.lognormal(0.0, 1.5)});
                    }
            for (int64_t i = 0; i < sp.n; ++i) {
                if (topo.u01() < 0.005) {
                    int64_t j;
                    do j = static_cast<int64_t>(topo.below(sp.n)); while (j == i);
                    sp.edges.push_back({i, j, cond.lognormal(-2.0, 1.0)});
                }
            }
            sp.src_frac = 0.05, sp.src_lo = -0.5, sp.src_hi = 0.5;
            sp.d_lo = 1e-4, sp.d_hi = 1e-2;
            break;
        }
        case 4: {  // transient Newton sequence: n = 100,000, avg degree 5
            seed = 5;
            sp.n = 100000;
            circuit_edges(sp, seed, 1, true, 0.0, 2.0);
            sp.src_frac = 0.05, sp.src_lo = -0.5, sp.src_hi = 0.5;
            sp.d_lo = 1e-3, sp.d_hi = 1e-1;
            break;
        }
        default:
            return Csr{};
    }
    const std::vector<Source> src = pick_sources(sp, seed);
    std::vector<double> gscale(sp.edges.size(), 1.0);
    uint64_t slack_seed = stream_seed(seed, kSlack);
    uint64_t x_seed = stream_seed(seed, kXtrue);
    if (config == 4) {
        // per-edge phase (drawn once); per step k: g * (1 + 0.05 sin(k + phi))
        Rng ph(stream_seed(seed, kPhase));
        for (double& s : gscale) {
            const double phi = ph.uniform(0.0, 6.283185307179586);
            s = 1.0 + 0.05 * std::sin(static_cast<double>(step) + phi);
        }
        slack_seed = stream_seed(seed * 1000 + static_cast<uint64_t>(step), kSlack);
        x_seed = stream_seed(seed * 1000 + static_cast<uint64_t>(step), kXtrue);
    }
    const std::vector<double> slack = draw_slack(sp.n, slack_seed, sp.d_lo, sp.d_hi);
    Csr a = assemble(sp, gscale, src, slack);
    finish_rhs(a, x_seed);
    return a;
}

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

}  // namespace

extern "C" {

struct hpbj_gen_system {
    int64_t n;
    int64_t nnz;
    int64_t* row_ptr;
    int64_t* col;
    double* val;
    double* b;
    double* x_true;
    // solver parameters of the config (BASELINE.json)
    int64_t block_size;
    int64_t num_blocks;  // ceil(n / block_size)
    int64_t restart_m;
    double tol;
    int64_t maxit;
    int64_t max_restarts;  // ceil(maxit / m); config 4: reference default 40
};

int hpbj_gen_config(int config, int step, hpbj_gen_system* out) {
    static const int64_t bs[5] = {32, 64, 128, 256, 64};
    static const int64_t mm[5] = {30, 50, 50, 100, 30};
    static const double tl[5] = {1e-10, 1e-10, 1e-10, 1e-9, 1e-10};
    static const int64_t mi[5] = {1000, 2000, 3000, 5000, 0};
    if (config < 0 || config > 4 || !out) return 1;
    if (config == 4 && (step < 0 || step >= 64)) return 1;
    Csr a = build_config(config, step);
    out->n = a.n;
    out->nnz = a.rp[a.n];
    out->row_ptr = dup(a.rp);
    out->col = dup(a.ci);
    out->val = dup(a.val);
    out->b = dup(a.b);
    out->x_true = dup(a.xtrue);
    out->block_size = bs[config];
    out->num_blocks = (a.n + bs[config] - 1) / bs[config];
    out->restart_m = mm[config];
    out->tol = tl[config];
    out->maxit = mi[config];
    out->max_restarts = config == 4 ? 40 : (mi[config] + mm[config] - 1) / mm[config];
    return 0;
}

void hpbj_gen_free(hpbj_gen_system* s) {
    if (!s) return;
    std::free(s->row_ptr);
    std::free(s->col);
    std::free(s->val);
    std::free(s->b);
    std::free(s->x_true);
    std::memset(s, 0, sizeof(*s));
}

}  // extern "C"
