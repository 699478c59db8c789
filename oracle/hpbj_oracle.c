/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference algorithm
 * (see hpbj_oracle.h). Every function cites the reference lines it follows
 * (paths under /root/reference/proj). Built with -ffp-contract=off like the
 * reference (CMakeLists.txt:12-14). Binary32 arithmetic is emulated exactly
 * by rounding every binary64 result to binary32 (R32): for + - * / the
 * double result rounded to float equals the float operation (53 >= 2*24+2),
 * so the emulation is bit-exact with native float code.
 */
#include "hpbj_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t idx;

static double R32(double x) { return (double)(float)x; }
static double RT(double x, int fp32) { return fp32 ? R32(x) : x; }

/* ------------------------------------------------------------------ CSR */
typedef struct {
    idx n, nnz;
    idx *rp, *ci;
    double *val;
} csr;

static csr csr_alloc(idx n, idx nnz) {
    csr a;
    a.n = n;
    a.nnz = nnz;
    a.rp = (idx*)calloc((size_t)n + 1, sizeof(idx));
    a.ci = (idx*)malloc(sizeof(idx) * (size_t)(nnz ? nnz : 1));
    a.val = (double*)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    return a;
}
static void csr_free(csr* a) {
    free(a->rp);
    free(a->ci);
    free(a->val);
}

/* spmv<T> (spmv.hpp:31-47): row sums left to right in the precision of T. */
static void spmv_t(const csr* a, const double* x, double* y, int fp32) {
    for (idx i = 0; i < a->n; ++i) {
        double s = 0.0;
        for (idx k = a->rp[i]; k < a->rp[i + 1]; ++k)
            s = RT(s + RT(RT(a->val[k], fp32) * x[a->ci[k]], fp32), fp32);
        y[i] = s;
    }
}

/* dot<T> / norm2<T> (dense_ops.hpp:14-46): sequential binary64 accumulation. */
static double dot(const double* a, const double* b, idx n) {
    double acc = 0.0;
    for (idx i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}
static double norm2(const double* a, idx n) { return sqrt(dot(a, a, n)); }

/* matrix_inf_norm (sparse_matrix.cpp:155-166) */
static double inf_norm(const csr* a) {
    double nm = 0.0;
    for (idx i = 0; i < a->n; ++i) {
        double rs = 0.0;
        for (idx k = a->rp[i]; k < a->rp[i + 1]; ++k) rs += fabs(a->val[k]);
        if (rs > nm) nm = rs;
    }
    return nm;
}

/* ---------------------------------------------------- graph + partition */
typedef struct {
    idx lo, hi;
    double v;
} pairv;
static int cmp_pair(const void* x, const void* y) {
    const pairv* a = (const pairv*)x;
    const pairv* b = (const pairv*)y;
    if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
    if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
    return 0; /* stable order restored below by the index tie-break */
}
typedef struct {
    idx lo, hi, ord;
    double v;
} pairo;
static int cmp_pairo(const void* x, const void* y) {
    const pairo* a = (const pairo*)x;
    const pairo* b = (const pairo*)y;
    if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
    if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
    return a->ord < b->ord ? -1 : (a->ord > b->ord ? 1 : 0);
}

typedef struct {
    idx n;
    idx* st;
    idx* nb;
    double* w;
} graph;

/* graph_from_matrix (graph.cpp:17-51): pair_sum[{min,max}] += |a_ij| in row
 * scan order (std::map), w = 0.5 * sum, skip w <= 0, adjacency sorted. */
static graph build_graph(const csr* a) {
    idx cnt = 0;
    pairo* P = (pairo*)malloc(sizeof(pairo) * (size_t)(a->nnz ? a->nnz : 1));
    for (idx i = 0; i < a->n; ++i)
        for (idx k = a->rp[i]; k < a->rp[i + 1]; ++k) {
            const idx j = a->ci[k];
            if (i == j) continue;
            P[cnt].lo = i < j ? i : j;
            P[cnt].hi = i < j ? j : i;
            P[cnt].ord = cnt;
            P[cnt].v = fabs(a->val[k]);
            ++cnt;
        }
    qsort(P, (size_t)cnt, sizeof(pairo), cmp_pairo);
    graph g;
    g.n = a->n;
    g.st = (idx*)calloc((size_t)a->n + 1, sizeof(idx));
    idx* deg = (idx*)calloc((size_t)a->n, sizeof(idx));
    pairv* U = (pairv*)malloc(sizeof(pairv) * (size_t)(cnt ? cnt : 1));
    idx nu = 0;
    for (idx k = 0; k < cnt;) {
        double sum = 0.0;
        const idx lo = P[k].lo, hi = P[k].hi;
        while (k < cnt && P[k].lo == lo && P[k].hi == hi) sum += P[k++].v;
        const double w = 0.5 * sum;
        if (w <= 0.0) continue;
        U[nu].lo = lo;
        U[nu].hi = hi;
        U[nu].v = w;
        ++nu;
        ++deg[lo];
        ++deg[hi];
    }
    for (idx i = 0; i < a->n; ++i) g.st[i + 1] = g.st[i] + deg[i];
    g.nb = (idx*)malloc(sizeof(idx) * (size_t)(g.st[a->n] ? g.st[a->n] : 1));
    g.w = (double*)malloc(sizeof(double) * (size_t)(g.st[a->n] ? g.st[a->n] : 1));
    idx* next = (idx*)malloc(sizeof(idx) * (size_t)(a->n ? a->n : 1));
    for (idx i = 0; i < a->n; ++i) next[i] = g.st[i];
    /* pairs come sorted by (lo, hi): neighbours pushed in map order, then
     * each adjacency is sorted by neighbour (graph.cpp:45-49). */
    for (idx k = 0; k < nu; ++k) {
        g.nb[next[U[k].lo]] = U[k].hi;
        g.w[next[U[k].lo]++] = U[k].v;
        g.nb[next[U[k].hi]] = U[k].lo;
        g.w[next[U[k].hi]++] = U[k].v;
    }
    for (idx u = 0; u < a->n; ++u) { /* insertion sort by neighbour */
        for (idx p = g.st[u] + 1; p < g.st[u + 1]; ++p) {
            const idx kn = g.nb[p];
            const double kw = g.w[p];
            idx q = p - 1;
            while (q >= g.st[u] && g.nb[q] > kn) {
                g.nb[q + 1] = g.nb[q];
                g.w[q + 1] = g.w[q];
                --q;
            }
            g.nb[q + 1] = kn;
            g.w[q + 1] = kw;
        }
    }
    free(P);
    free(U);
    free(deg);
    free(next);
    return g;
}

/* pick_seed (partition.cpp:45-56) */
static idx pick_seed(const graph* g, const idx* asg) {
    idx seed = -1, best = 0;
    for (idx v = 0; v < g->n; ++v) {
        const idx d = g->st[v + 1] - g->st[v];
        if (asg[v] >= 0 || d == 0) continue;
        if (seed < 0 || d > best) {
            seed = v;
            best = d;
        }
    }
    return seed;
}

/* partition_graph (partition.cpp:60-144), queue with duplicates as there. */
static int partition_graph(const graph* g, idx s, double tol, idx* asg) {
    const idx n = g->n;
    if (s < 1 || s > n || tol < 0.0) return 1;
    idx cap = (idx)ceil((double)n / (double)s * (1.0 + tol));
    if ((n + s - 1) / s > cap) cap = (n + s - 1) / s;
    idx* sizes = (idx*)calloc((size_t)s, sizeof(idx));
    for (idx v = 0; v < n; ++v) asg[v] = -1;
    idx left = 0;
    for (idx v = 0; v < n; ++v)
        if (g->st[v + 1] > g->st[v]) ++left;
    idx qcap = 2 * (g->st[n] + n) + 16;
    idx* q = (idx*)malloc(sizeof(idx) * (size_t)qcap);
    for (idx b = 0; b < s && left > 0; ++b) {
        const idx bl = s - b;
        idx target = (left + bl - 1) / bl;
        if (target > cap) target = cap;
        idx head = 0, tail = 0, grown = 0;
        while (grown < target) {
            if (head == tail) {
                const idx seed = pick_seed(g, asg);
                if (seed < 0) break;
                q[tail++] = seed;
            }
            const idx u = q[head++];
            if (asg[u] >= 0) continue;
            asg[u] = b;
            ++sizes[b];
            ++grown;
            --left;
            for (idx k = g->st[u]; k < g->st[u + 1]; ++k)
                if (asg[g->nb[k]] < 0) {
                    if (tail >= qcap) {
                        qcap *= 2;
                        q = (idx*)realloc(q, sizeof(idx) * (size_t)qcap);
                    }
                    q[tail++] = g->nb[k];
                }
        }
    }
    for (idx v = 0; v < n; ++v) { /* partition.cpp:105-112 */
        if (asg[v] >= 0) continue;
        idx sm = 0;
        for (idx b = 1; b < s; ++b)
            if (sizes[b] < sizes[sm]) sm = b;
        asg[v] = sm;
        ++sizes[sm];
    }
    double* conn = (double*)calloc((size_t)s, sizeof(double)); /* partition.cpp:117-141 */
    idx* touched = (idx*)malloc(sizeof(idx) * (size_t)(n + 1));
    for (idx u = 0; u < n; ++u) {
        const idx bu = asg[u];
        if (sizes[bu] <= 1) continue;
        idx nt = 0;
        for (idx k = g->st[u]; k < g->st[u + 1]; ++k) {
            const idx bv = asg[g->nb[k]];
            if (conn[bv] == 0.0) touched[nt++] = bv;
            conn[bv] += g->w[k];
        }
        idx best = -1;
        for (idx t = 0; t < nt; ++t) {
            const idx bv = touched[t];
            if (bv == bu || sizes[bv] + 1 > cap) continue;
            if (best < 0 || conn[bv] > conn[best] || (conn[bv] == conn[best] && bv < best)) best = bv;
        }
        if (best >= 0 && conn[best] > conn[bu]) {
            asg[u] = best;
            --sizes[bu];
            ++sizes[best];
        }
        for (idx t = 0; t < nt; ++t) conn[touched[t]] = 0.0;
    }
    free(sizes);
    free(q);
    free(conn);
    free(touched);
    return 0;
}

/* partition_from_assignment (partition.cpp:14-41): stable gather. */
static int gather(idx n, const idx* asg, idx s, idx* perm, idx* bst) {
    idx* cnt = (idx*)calloc((size_t)s, sizeof(idx));
    for (idx i = 0; i < n; ++i) {
        if (asg[i] < 0 || asg[i] >= s) {
            free(cnt);
            return 1;
        }
        ++cnt[asg[i]];
    }
    bst[0] = 0;
    for (idx b = 0; b < s; ++b) {
        if (cnt[b] == 0) {
            free(cnt);
            return 1;
        }
        bst[b + 1] = bst[b] + cnt[b];
    }
    for (idx b = 0; b < s; ++b) cnt[b] = bst[b];
    for (idx i = 0; i < n; ++i) perm[i] = cnt[asg[i]]++;
    free(cnt);
    return 0;
}

/* permute_symmetric (sparse_matrix.cpp:113-153) + slice_diag_block
 * (preconditioner.cpp:20-40): block b of Q A Q^T as CSR, sorted columns. */
typedef struct {
    idx c;
    double v;
} ent;
static int cmp_ent(const void* x, const void* y) {
    const ent* a = (const ent*)x;
    const ent* b = (const ent*)y;
    return a->c < b->c ? -1 : (a->c > b->c ? 1 : 0);
}
static csr permute(const csr* a, const idx* perm) {
    csr b = csr_alloc(a->n, a->nnz);
    for (idx i = 0; i < a->n; ++i) b.rp[perm[i] + 1] = a->rp[i + 1] - a->rp[i];
    for (idx i = 0; i < a->n; ++i) b.rp[i + 1] += b.rp[i];
    ent* row = (ent*)malloc(sizeof(ent) * (size_t)(a->nnz ? a->nnz : 1));
    for (idx i = 0; i < a->n; ++i) {
        idx len = 0;
        for (idx k = a->rp[i]; k < a->rp[i + 1]; ++k) {
            row[len].c = perm[a->ci[k]];
            row[len].v = a->val[k];
            ++len;
        }
        qsort(row, (size_t)len, sizeof(ent), cmp_ent);
        idx d = b.rp[perm[i]];
        for (idx k = 0; k < len; ++k) {
            b.ci[d] = row[k].c;
            b.val[d] = row[k].v;
            ++d;
        }
    }
    free(row);
    return b;
}
static csr slice(const csr* a, idx begin, idx end) {
    idx cnt = 0;
    for (idx i = begin; i < end; ++i)
        for (idx k = a->rp[i]; k < a->rp[i + 1]; ++k)
            if (a->ci[k] >= begin && a->ci[k] < end) ++cnt;
    csr b = csr_alloc(end - begin, cnt);
    idx d = 0;
    for (idx i = begin; i < end; ++i) {
        for (idx k = a->rp[i]; k < a->rp[i + 1]; ++k)
            if (a->ci[k] >= begin && a->ci[k] < end) {
                b.ci[d] = a->ci[k] - begin;
                b.val[d] = a->val[k];
                ++d;
            }
        b.rp[i - begin + 1] = d;
    }
    return b;
}

/* --------------------------------------------------------------- gp_lu */
typedef struct {
    idx* r;
    double* v;
    idx len, cap;
} colv;
static void col_push(colv* c, idx r, double v) {
    if (c->len == c->cap) {
        c->cap = c->cap ? 2 * c->cap : 8;
        c->r = (idx*)realloc(c->r, sizeof(idx) * (size_t)c->cap);
        c->v = (double*)realloc(c->v, sizeof(double) * (size_t)c->cap);
    }
    c->r[c->len] = r;
    c->v[c->len] = v;
    ++c->len;
}
typedef struct {
    idx n;
    csr L, U;
    idx* piv;
    idx npert;
} lufac;

static csr cols_to_csr(idx n, colv* cols) { /* columns_to_csr (lu.cpp:58-76) */
    idx nnz = 0;
    for (idx j = 0; j < n; ++j) nnz += cols[j].len;
    csr a = csr_alloc(n, nnz);
    for (idx j = 0; j < n; ++j)
        for (idx t = 0; t < cols[j].len; ++t) ++a.rp[cols[j].r[t] + 1];
    for (idx i = 0; i < n; ++i) a.rp[i + 1] += a.rp[i];
    idx* next = (idx*)malloc(sizeof(idx) * (size_t)(n ? n : 1));
    for (idx i = 0; i < n; ++i) next[i] = a.rp[i];
    for (idx j = 0; j < n; ++j)
        for (idx t = 0; t < cols[j].len; ++t) {
            const idx d = next[cols[j].r[t]]++;
            a.ci[d] = j;
            a.val[d] = cols[j].v[t];
        }
    free(next);
    return a;
}

/* regularize_pivot (lu.cpp:10-20) */
static double regularize(double p, double nm, double eps, int* perturbed) {
    const int keep = nm == 0.0 ? p != 0.0 : fabs(p) / nm >= eps;
    *perturbed = !keep;
    if (keep) return p;
    return (p < 0.0 ? -1.0 : 1.0) * eps * nm;
}

/* gp_lu (lu.cpp:134-225): left-looking Gilbert-Peierls with DFS reach
 * (:80-130), partial pivoting ties -> smallest row (:171-181), empty-column
 * fallback (:182-186), Eq. 7 regularisation (:188-197). Returns the
 * singular column or -1. */
static idx gp_lu(const csr* blk, double eps, lufac* f) {
    const idx n = blk->n;
    const double nm = inf_norm(blk);
    /* CSC of the block (csr_to_csc, lu.cpp:31-50) */
    idx* cst = (idx*)calloc((size_t)n + 1, sizeof(idx));
    idx* cr = (idx*)malloc(sizeof(idx) * (size_t)(blk->nnz ? blk->nnz : 1));
    double* cv = (double*)malloc(sizeof(double) * (size_t)(blk->nnz ? blk->nnz : 1));
    for (idx k = 0; k < blk->nnz; ++k) ++cst[blk->ci[k] + 1];
    for (idx j = 0; j < n; ++j) cst[j + 1] += cst[j];
    idx* nx = (idx*)malloc(sizeof(idx) * (size_t)(n ? n : 1));
    for (idx j = 0; j < n; ++j) nx[j] = cst[j];
    for (idx i = 0; i < n; ++i)
        for (idx k = blk->rp[i]; k < blk->rp[i + 1]; ++k) {
            const idx d = nx[blk->ci[k]]++;
            cr[d] = i;
            cv[d] = blk->val[k];
        }
    colv* lc = (colv*)calloc((size_t)n, sizeof(colv));
    colv* uc = (colv*)calloc((size_t)n, sizeof(colv));
    idx* pinv = (idx*)malloc(sizeof(idx) * (size_t)(n ? n : 1));
    f->piv = (idx*)malloc(sizeof(idx) * (size_t)(n ? n : 1));
    double* x = (double*)calloc((size_t)n, sizeof(double));
    idx* mark = (idx*)calloc((size_t)n, sizeof(idx));
    idx* nstack = (idx*)malloc(sizeof(idx) * (size_t)(n + 1));
    idx* cstack = (idx*)malloc(sizeof(idx) * (size_t)(n + 1));
    idx* post = (idx*)malloc(sizeof(idx) * (size_t)(n + 1));
    idx* topo = (idx*)malloc(sizeof(idx) * (size_t)(n + 1));
    for (idx i = 0; i < n; ++i) pinv[i] = -1;
    idx epoch = 0, next_unused = 0, sing = -1;
    f->npert = 0;
    for (idx k = 0; k < n && sing < 0; ++k) {
        /* reach of column k's pattern through the partial L graph */
        ++epoch;
        idx np = 0;
        for (idx t = cst[k]; t < cst[k + 1]; ++t) {
            const idx seed = cr[t];
            if (mark[seed] == epoch) continue;
            idx sp = 0;
            nstack[sp] = seed;
            cstack[sp] = 0;
            ++sp;
            mark[seed] = epoch;
            while (sp > 0) {
                const idx u = nstack[sp - 1];
                const idx c = pinv[u];
                const idx dg = c >= 0 ? lc[c].len : 0;
                int desc = 0;
                while (cstack[sp - 1] < dg) {
                    const idx v = lc[c].r[cstack[sp - 1]++];
                    if (mark[v] != epoch) {
                        mark[v] = epoch;
                        nstack[sp] = v;
                        cstack[sp] = 0;
                        ++sp;
                        desc = 1;
                        break;
                    }
                }
                if (!desc) {
                    --sp;
                    post[np++] = u;
                }
            }
        }
        for (idx t = 0; t < np; ++t) topo[t] = post[np - 1 - t];
        /* sparse L-solve over the reach (lu.cpp:160-169) */
        for (idx t = cst[k]; t < cst[k + 1]; ++t) x[cr[t]] = cv[t];
        for (idx t = 0; t < np; ++t) {
            const idx j = topo[t];
            const idx c = pinv[j];
            if (c < 0) continue;
            const double xj = x[j];
            if (xj != 0.0)
                for (idx e = 0; e < lc[c].len; ++e) x[lc[c].r[e]] -= lc[c].v[e] * xj;
        }
        idx prow = -1;
        double pabs = -1.0;
        for (idx t = 0; t < np; ++t) {
            const idx i = topo[t];
            if (pinv[i] >= 0) continue;
            const double a = fabs(x[i]);
            if (a > pabs || (a == pabs && i < prow)) {
                pabs = a;
                prow = i;
            }
        }
        if (prow < 0) {
            while (pinv[next_unused] >= 0) ++next_unused;
            prow = next_unused;
        }
        int pert = 0;
        const double pvv = x[prow];
        const double reg = regularize(pvv, nm, eps, &pert);
        if (reg == 0.0) {
            sing = k;
            break;
        }
        if (pert) ++f->npert;
        pinv[prow] = k;
        f->piv[k] = prow;
        col_push(&uc[k], k, reg);
        for (idx t = 0; t < np; ++t) {
            const idx i = topo[t];
            if (i == prow) continue;
            if (pinv[i] >= 0) col_push(&uc[k], pinv[i], x[i]);
            else if (x[i] != 0.0) col_push(&lc[k], i, x[i] / reg);
        }
        for (idx t = 0; t < np; ++t) x[topo[t]] = 0.0;
    }
    if (sing < 0) {
        for (idx j = 0; j < n; ++j)
            for (idx t = 0; t < lc[j].len; ++t) lc[j].r[t] = pinv[lc[j].r[t]];
        f->n = n;
        f->L = cols_to_csr(n, lc);
        f->U = cols_to_csr(n, uc);
    }
    for (idx j = 0; j < n; ++j) {
        free(lc[j].r);
        free(lc[j].v);
        free(uc[j].r);
        free(uc[j].v);
    }
    free(lc);
    free(uc);
    free(cst);
    free(cr);
    free(cv);
    free(nx);
    free(pinv);
    free(x);
    free(mark);
    free(nstack);
    free(cstack);
    free(post);
    free(topo);
    return sing;
}

/* lu_solve<T> (lu.hpp:88-112). fp32_vals: use binary32-rounded factor values
 * (values_low); fp32_arith: binary32 arithmetic. */
static void lu_solve(const lufac* f, const double* rhs, double* x, int fp32_vals, int fp32_arith) {
    const idx n = f->n;
    for (idx i = 0; i < n; ++i) {
        double s = rhs[f->piv[i]];
        for (idx k = f->L.rp[i]; k < f->L.rp[i + 1]; ++k)
            s = RT(s - RT(RT(f->L.val[k], fp32_vals) * x[f->L.ci[k]], fp32_arith), fp32_arith);
        x[i] = s;
    }
    for (idx i = n - 1; i >= 0; --i) {
        const idx d = f->U.rp[i];
        double s = x[i];
        for (idx k = d + 1; k < f->U.rp[i + 1]; ++k)
            s = RT(s - RT(RT(f->U.val[k], fp32_vals) * x[f->U.ci[k]], fp32_arith), fp32_arith);
        x[i] = RT(s / RT(f->U.val[d], fp32_vals), fp32_arith);
    }
}

/* Preconditioner::block_jacobi (preconditioner.cpp:100-153) */
typedef struct {
    idx n, s;
    idx *perm, *bst;
    lufac* fac;
    idx sing_block, sing_col, npert;
} bjac;

static int bj_build(const csr* a, idx s, const idx* asg, double eps, bjac* P) {
    P->n = a->n;
    P->s = s;
    P->perm = (idx*)malloc(sizeof(idx) * (size_t)a->n);
    P->bst = (idx*)malloc(sizeof(idx) * (size_t)(s + 1));
    P->fac = (lufac*)calloc((size_t)s, sizeof(lufac));
    P->sing_block = P->sing_col = -1;
    P->npert = 0;
    if (gather(a->n, asg, s, P->perm, P->bst)) return 1;
    csr pa = permute(a, P->perm);
    for (idx b = 0; b < s; ++b) {
        csr blk = slice(&pa, P->bst[b], P->bst[b + 1]);
        const idx sc = gp_lu(&blk, eps, &P->fac[b]);
        csr_free(&blk);
        if (sc >= 0 && P->sing_block < 0) { /* rethrown in block order (:147-148) */
            P->sing_block = b;
            P->sing_col = sc;
        }
        P->npert += P->fac[b].npert;
    }
    csr_free(&pa);
    return P->sing_block >= 0 ? 3 : 0;
}
static void bj_free(bjac* P) {
    for (idx b = 0; b < P->s; ++b) {
        if (P->fac[b].n) {
            csr_free(&P->fac[b].L);
            csr_free(&P->fac[b].U);
        }
        free(P->fac[b].piv);
    }
    free(P->fac);
    free(P->perm);
    free(P->bst);
}

/* apply_impl (preconditioner.cpp:159-188): scatter by perm, per-block
 * lu_solve, gather. */
static void bj_apply(const bjac* P, const double* v, double* z, int fp32_vals, int fp32_arith) {
    const idx n = P->n;
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    for (idx i = 0; i < n; ++i) w[P->perm[i]] = v[i];
    for (idx b = 0; b < P->s; ++b) lu_solve(&P->fac[b], w + P->bst[b], y + P->bst[b], fp32_vals, fp32_arith);
    for (idx i = 0; i < n; ++i) z[i] = y[P->perm[i]];
    free(w);
    free(y);
}

/* ------------------------------------------------------------- GMRES */
typedef struct {
    const csr* a;
    const bjac* P;
    int mode;
    double* tmp;
} opctx;

/* the Arnoldi operator w = A M^-1 v (gmres.cpp:125-128) per mode */
static void op_apply(const opctx* o, const double* v, double* w) {
    const idx n = o->a->n;
    if (o->mode == ORC_DOUBLE) {
        bj_apply(o->P, v, o->tmp, 0, 0);
        spmv_t(o->a, o->tmp, w, 0);
    } else if (o->mode == ORC_HYBRID) {
        bj_apply(o->P, v, o->tmp, 1, 1); /* apply<float> */
        spmv_t(o->a, o->tmp, w, 1);      /* spmv<float>  */
    } else {                             /* MIX: FP32 apply of the rounded FP64 v, FP64 SpMV */
        double* vf = (double*)malloc(sizeof(double) * (size_t)n);
        for (idx i = 0; i < n; ++i) vf[i] = R32(v[i]);
        bj_apply(o->P, vf, o->tmp, 1, 1);
        spmv_t(o->a, o->tmp, w, 0);
        free(vf);
    }
}

/* One cycle: run_cycle<T> (gmres.cpp:97-166) with arnoldi_step (gmres.hpp:
 * 43-75) and GivensLs (gmres.cpp:16-73). Returns iterations. */
static idx run_cycle(const opctx* o, const double* b, const double* x0, double* x, idx m, double thr,
                     double bnorm, double* est, int* conv, int* brk, int* rank) {
    const idx n = o->a->n;
    const int t32 = o->mode == ORC_HYBRID; /* basis precision T */
    const double u_T = t32 ? 0x1p-24 : 0x1p-53;
    const double u_work = o->mode == ORC_DOUBLE ? 0x1p-53 : 0x1p-24;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(x, x0, sizeof(double) * (size_t)n);
    *conv = *brk = *rank = 0;
    (void)bnorm;
    spmv_t(o->a, x0, r, 0);
    for (idx i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double beta = norm2(r, n);
    if (beta <= thr) {
        *conv = 1;
        free(r);
        return 0;
    }
    double* V = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
    for (idx i = 0; i < n; ++i) V[i] = RT(r[i] / beta, t32);
    double* H = (double*)calloc((size_t)(m + 1) * (size_t)m, sizeof(double));
    double* R = (double*)calloc((size_t)(m + 1) * (size_t)m, sizeof(double));
    double* cs = (double*)calloc((size_t)m, sizeof(double));
    double* sn = (double*)calloc((size_t)m, sizeof(double));
    double* g = (double*)calloc((size_t)m + 1, sizeof(double));
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    g[0] = beta;
    const double attainable = 10.0 * u_work * beta;
    idx steps = 0;
    while (steps < m) {
        const idx j = steps;
        op_apply(o, V + (size_t)j * n, w);
        const double pre = norm2(w, n);
        for (idx i = 0; i <= j; ++i) {
            const double h = dot(V + (size_t)i * n, w, n);
            H[j * (m + 1) + i] = h;
            const double hc = RT(h, t32);
            const double* vi = V + (size_t)i * n;
            for (idx q = 0; q < n; ++q) w[q] = RT(w[q] - RT(hc * vi[q], t32), t32);
        }
        const double hn = norm2(w, n);
        H[j * (m + 1) + j + 1] = hn;
        steps = j + 1;
        int bd = hn <= 1e2 * u_T * pre;
        if (!bd) {
            const double inv = RT(1.0 / hn, t32);
            for (idx q = 0; q < n; ++q) V[(size_t)(j + 1) * n + q] = RT(w[q] * inv, t32);
        }
        /* push_column */
        double* Rj = R + j * (m + 1);
        for (idx i = 0; i <= j + 1; ++i) Rj[i] = H[j * (m + 1) + i];
        for (idx i = 0; i < j; ++i) {
            const double t = cs[i] * Rj[i] + sn[i] * Rj[i + 1];
            Rj[i + 1] = -sn[i] * Rj[i] + cs[i] * Rj[i + 1];
            Rj[i] = t;
        }
        const double aa = Rj[j], bb = Rj[j + 1];
        if (bb == 0.0) {
            cs[j] = 1.0;
            sn[j] = 0.0;
        } else {
            const double hh = hypot(aa, bb);
            cs[j] = aa / hh;
            sn[j] = bb / hh;
        }
        Rj[j] = cs[j] * aa + sn[j] * bb;
        Rj[j + 1] = 0.0;
        if (Rj[j] == 0.0) *rank = 1;
        const double t = cs[j] * g[j] + sn[j] * g[j + 1];
        g[j + 1] = -sn[j] * g[j] + cs[j] * g[j + 1];
        g[j] = t;
        const double e = fabs(g[j + 1]);
        est[j] = e;
        if (e <= thr) *conv = 1;
        if (bd) *brk = 1;
        if (*conv || *brk || e <= attainable) break;
    }
    /* y = R^-1 g (gmres.cpp:57-66); u = V y in FP64; x = x0 + M^-1 u */
    double* y = (double*)calloc((size_t)(steps ? steps : 1), sizeof(double));
    for (idx i = steps - 1; i >= 0; --i) {
        if (R[i * (m + 1) + i] == 0.0) continue;
        double sm = g[i];
        for (idx k = i + 1; k < steps; ++k) sm -= R[k * (m + 1) + i] * y[k];
        y[i] = sm / R[i * (m + 1) + i];
    }
    double* u = (double*)calloc((size_t)n, sizeof(double));
    for (idx i = 0; i < steps; ++i)
        for (idx q = 0; q < n; ++q) u[q] += y[i] * V[(size_t)i * n + q];
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    if (o->mode == ORC_MIX) bj_apply(o->P, u, z, 1, 0); /* FP32 factors, FP64 arithmetic */
    else bj_apply(o->P, u, z, 0, 0);                   /* preconditioned<double> (:158) */
    for (idx q = 0; q < n; ++q) x[q] = x0[q] + z[q];
    free(r);
    free(V);
    free(H);
    free(R);
    free(cs);
    free(sn);
    free(g);
    free(w);
    free(y);
    free(u);
    free(z);
    return steps;
}

/* ------------------------------------------------------------- C ABI */
static csr wrap(idx n, const idx* rp, const idx* ci, const double* v) {
    csr a;
    a.n = n;
    a.nnz = rp[n];
    a.rp = (idx*)rp;
    a.ci = (idx*)ci;
    a.val = (double*)v;
    return a;
}

int orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x, double* y,
             int fp32) {
    csr a = wrap(n, rp, ci, v);
    if (fp32) {
        double* xf = (double*)malloc(sizeof(double) * (size_t)n);
        for (idx i = 0; i < n; ++i) xf[i] = R32(x[i]);
        spmv_t(&a, xf, y, 1);
        free(xf);
    } else {
        spmv_t(&a, x, y, 0);
    }
    return 0;
}

int orc_graph(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t* st, int64_t* nb,
              double* w, int64_t cap) {
    csr a = wrap(n, rp, ci, v);
    graph g = build_graph(&a);
    int rc = 0;
    if (g.st[n] > cap) rc = 1;
    else {
        memcpy(st, g.st, sizeof(idx) * (size_t)(n + 1));
        memcpy(nb, g.nb, sizeof(idx) * (size_t)g.st[n]);
        memcpy(w, g.w, sizeof(double) * (size_t)g.st[n]);
    }
    free(g.st);
    free(g.nb);
    free(g.w);
    return rc;
}

int orc_partition(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s, double tol,
                  int64_t* assignment) {
    csr a = wrap(n, rp, ci, v);
    graph g = build_graph(&a);
    const int rc = partition_graph(&g, s, tol, assignment);
    free(g.st);
    free(g.nb);
    free(g.w);
    return rc;
}

int orc_factors(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
                const int64_t* assignment, double eps, double* f64, int64_t* pivot_rows, int64_t* pert,
                int64_t* sing_block, int64_t* sing_col) {
    csr a = wrap(n, rp, ci, v);
    bjac P;
    const int rc = bj_build(&a, s, assignment, eps, &P);
    *sing_block = P.sing_block;
    *sing_col = P.sing_col;
    if (rc == 0) {
        idx off = 0;
        for (idx b = 0; b < s; ++b) {
            const lufac* f = &P.fac[b];
            const idx d = f->n;
            memset(f64 + off, 0, sizeof(double) * (size_t)(d * d));
            for (idx i = 0; i < d; ++i) {
                for (idx k = f->L.rp[i]; k < f->L.rp[i + 1]; ++k) f64[off + i * d + f->L.ci[k]] = f->L.val[k];
                for (idx k = f->U.rp[i]; k < f->U.rp[i + 1]; ++k) f64[off + i * d + f->U.ci[k]] = f->U.val[k];
            }
            for (idx k = 0; k < d; ++k) pivot_rows[P.bst[b] + k] = f->piv[k];
            pert[b] = f->npert;
            off += d * d;
        }
    }
    bj_free(&P);
    return rc;
}

int orc_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
              const int64_t* assignment, double eps, int fp32, const double* vin, double* zout) {
    csr a = wrap(n, rp, ci, v);
    bjac P;
    const int rc = bj_build(&a, s, assignment, eps, &P);
    if (rc == 0) {
        if (fp32) {
            double* vf = (double*)malloc(sizeof(double) * (size_t)n);
            for (idx i = 0; i < n; ++i) vf[i] = R32(vin[i]);
            bj_apply(&P, vf, zout, 1, 1);
            free(vf);
        } else {
            bj_apply(&P, vin, zout, 0, 0);
        }
    }
    bj_free(&P);
    return rc;
}

/* hybrid_restart_gmres (gmres.cpp:200-274) */
int orc_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
              const int64_t* assignment, const double* b, int64_t m, double tol, int64_t max_restarts,
              int mode, double eps, double* x, orc_report* rep, double* hist, int64_t hist_cap, double* cycres,
              int64_t cyc_cap) {
    memset(rep, 0, sizeof(*rep));
    rep->singular_block = rep->singular_column = -1;
    if (m < 1 || tol <= 0.0 || max_restarts < 1) return 1;
    csr a = wrap(n, rp, ci, v);
    bjac P;
    int rc = bj_build(&a, s, assignment, eps, &P);
    if (rc) {
        rep->singular_block = P.sing_block;
        rep->singular_column = P.sing_col;
        bj_free(&P);
        return rc;
    }
    opctx o = {&a, &P, mode, (double*)malloc(sizeof(double) * (size_t)n)};
    for (idx i = 0; i < n; ++i) x[i] = 0.0;
    idx hl = 0, cl = 0;
#define PUSH(c, it, rel)                        \
    do {                                        \
        if (hl < hist_cap) {                    \
            hist[3 * hl + 0] = (double)(c);     \
            hist[3 * hl + 1] = (double)(it);    \
            hist[3 * hl + 2] = (rel);           \
        }                                       \
        ++hl;                                   \
    } while (0)
    const double bnorm = norm2(b, n);
    if (bnorm == 0.0) {
        rep->converged = 1;
        PUSH(0, 0, 0.0);
        rep->hist_len = hl;
        free(o.tmp);
        bj_free(&P);
        return 0;
    }
    const double thr = tol * bnorm;
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double* xn = (double*)malloc(sizeof(double) * (size_t)n);
    double* est = (double*)malloc(sizeof(double) * (size_t)m);
    spmv_t(&a, x, r, 0);
    for (idx i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double rn = norm2(r, n);
    PUSH(0, 0, rn / bnorm);
    rep->final_residual = rn / bnorm;
    if (rn <= thr) {
        rep->converged = 1;
    } else {
        idx cycles = 0, git = 0;
        for (idx cyc = 0; cyc < max_restarts; ++cyc) {
            int conv, brk, rank;
            const idx its = run_cycle(&o, b, x, xn, m, thr, bnorm, est, &conv, &brk, &rank);
            ++cycles;
            for (idx k = 0; k < its; ++k) PUSH(cyc, ++git, est[k] / bnorm);
            rep->total_iterations += its;
            rep->breakdown |= brk;
            rep->rank_deficient |= rank;
            memcpy(x, xn, sizeof(double) * (size_t)n);
            spmv_t(&a, x, r, 0);
            for (idx i = 0; i < n; ++i) r[i] = b[i] - r[i];
            rn = norm2(r, n);
            if (cl < cyc_cap) cycres[cl] = rn / bnorm;
            ++cl;
            if (rn <= thr) {
                rep->converged = 1;
                break;
            }
            if (its == 0) break;
        }
        rep->restarts = cycles > 0 ? cycles - 1 : 0;
        rep->final_residual = rn / bnorm;
    }
#undef PUSH
    rep->hist_len = hl;
    rep->cyc_len = cl;
    free(r);
    free(xn);
    free(est);
    free(o.tmp);
    bj_free(&P);
    return 0;
}
