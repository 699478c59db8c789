// Arnoldi orthogonalisation + progressive Givens, device resident — replaces
// arnoldi_step (gmres.hpp:43-75), dot/norm2 (dense_ops.hpp:14-46) and
// GivensLs::push_column (gmres.cpp:26-52) plus the loop exits of run_cycle
// (gmres.cpp:130-146).
//
// Both kernels below apply the modified Gram-Schmidt projector
//     P = (I - v_j v_j^T) ... (I - v_0 v_0^T)
// to w = A M^-1 v_j in FP64, and keep the slice of w each CTA owns in shared
// memory for the whole step (w never round-trips to HBM). They differ only
// in how the j+1 inner products are synchronised:
//
//  k_mgs_pipe (large n, the default there): textbook MGS with the grid-wide
//          reductions taken off the critical path - see the kernel.
//  k_mgs  (its fallback: w slice not in shared memory, HPBJ_MGS=bar): the
//          textbook sequence, one grid-wide reduction per
//          projection, h_i = <v_i, w - sum_{k<i} h_k v_k>; each v_i streams
//          once from HBM for its dot and once more (L2-hot) for its axpy.
//          (Two projections per reduction with a Gram correction was
//          measured slower on config 3, 240 -> 262 us/step: the pass then
//          re-reads two vectors, 66 MB, that no longer stay in L2.)
//  k_icwy (small/medium n: barrier-latency bound): the compact-WY form of the
//          same projector, P = I - V T V^T with T = (I + L)^-1, L = strictly
//          lower part of V^T V (Swirydowicz et al., "Low synchronization
//          Gram-Schmidt and GMRES algorithms", NLA 2020). One fused multi-dot
//          pass yields c = V^T w and the new Gram row <v_j, v_k>; the MGS
//          coefficients h = (I + L)^-1 c follow from the triangular
//          recurrence h_i = c_i - sum_{k<i} L_ik h_k (identical to MGS's
//          h_i in exact arithmetic; two Jacobi sweeps are exact to O(|L|^3),
//          far below FP64 roundoff since |L| ~ loss of orthogonality); one
//          multi-axpy pass forms w - V h in MGS order. Two grid barriers per
//          step instead of j + 2.
//
// Reductions are deterministic: every CTA deposits per-value partials and
// every CTA sums them in CTA order, so all CTAs hold bit-identical totals
// and repeated solves are bit-reproducible. CTA 0 finishes the step:
// Hessenberg column, Givens rotation, residual estimate, cycle-exit flags
// (SolveState) — no host round-trip per iteration.

#include <cstdio>
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "kernels.cuh"
#include "sync_dev.cuh"

namespace hpbj {

namespace {

using sync::grid_barrier;
using sync::transpose_reduce;

constexpr int kMgsThreads = 1024;
constexpr int kMgsPre = 4;  // double2 per thread of the next vector in flight across a grid barrier
constexpr int kIcwyThreads = 1024;
constexpr size_t kSmemMax = 227 * 1024;

// Sum of partials[0..count) in a fixed order; every thread of warp 0 gets it.
__device__ __forceinline__ double sum_partials(const double* p, int count) {
    return warp_sum_partials(p, count);
}

// ---------------------------------------------------------------------------
struct OrthArgs {
    KrylovBufs kb;
    double* gram;        // (m+1) x (m+1): row i holds <v_i, v_k>, k < i
    SolveState* st;
    GridBarrier* gb;
    int n;
    int slice;           // rows per CTA (even)
    int npad;            // n rounded up to even (vectors zero padded)
    cudaGraphConditionalHandle cond;  // Arnoldi WHILE node (0: not in a graph)
    int scr;             // doubles of Givens scratch at the front of the dynamic smem (>= 3m+2, even)
    unsigned long long* prof;  // HPBJ_MGS_PROF=1: per CTA [stream, CTA reduce, grid barrier, broadcast, passes] cycles
};

// Shared finish of a step: normalise, Hessenberg column, Givens, exit flags.
__device__ void finish_step(const OrthArgs& a, double2* w2, double* scratch, int r0, int nv2, int j,
                            double pre_norm, double hnext, int nthreads) {
    SolveState* st = a.st;
    const int m = a.kb.m;
    const int ldv = a.kb.ldv;
    const bool breakdown = hnext <= st->breakdown_factor * pre_norm;  // gmres.hpp:66-71
    if (!breakdown) {
        const double inv = 1.0 / hnext;  // gmres.hpp:72-73: multiply by the reciprocal
        double2* vn = reinterpret_cast<double2*>(a.kb.V + (size_t)(j + 1) * ldv + r0);
        for (int e = threadIdx.x; e < nv2; e += nthreads) {
            double2 wv = w2[e];
            wv.x *= inv;
            wv.y *= inv;
            vn[e] = wv;
        }
    }
    if (blockIdx.x != 0) return;
    // CTA 0: coalesced staging of the rotation data by warp 0 into its own
    // scratch (3j+2 <= 3m+2 doubles, sized by plan_mgs independently of the
    // w slice), then one thread rotates out of shared memory.
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    double* Hj = a.kb.H + (size_t)j * (m + 1);
    double* Rj = a.kb.R + (size_t)j * (m + 1);
    double* cs = a.kb.cs;
    double* sn = a.kb.sn;
    double* g = a.kb.g;
    double* sR = scratch;                        // j + 2
    double* scs = sR + (j + 2);                  // j
    double* ssn = scs + j;                       // j
    for (int i = lane; i <= j; i += 32) sR[i] = __ldcg(Hj + i);
    for (int i = lane; i < j; i += 32) {
        scs[i] = __ldcg(cs + i);
        ssn[i] = __ldcg(sn + i);
    }
    __syncwarp();
    if (lane == 0) {
        sR[j + 1] = hnext;
        Hj[j + 1] = hnext;
        // GivensLs::push_column (gmres.cpp:26-52)
        double ri = sR[0];
        for (int i = 0; i < j; ++i) {
            const double rn = sR[i + 1];
            const double t = scs[i] * ri + ssn[i] * rn;
            const double r2 = -ssn[i] * ri + scs[i] * rn;
            sR[i] = t;
            ri = r2;
        }
        sR[j] = ri;
        const double aa = sR[j], bb = sR[j + 1];
        double c, sg;
        if (bb == 0.0) {
            c = 1.0;
            sg = 0.0;
        } else {
            const double hh = hypot(aa, bb);
            c = aa / hh;
            sg = bb / hh;
        }
        cs[j] = c;
        sn[j] = sg;
        sR[j] = c * aa + sg * bb;
        sR[j + 1] = 0.0;
        if (sR[j] == 0.0) st->rank_deficient = 1;
        const double gj = g[j], gj1 = g[j + 1];
        g[j + 1] = -sg * gj + c * gj1;
        g[j] = c * gj + sg * gj1;
        const double est = fabs(g[j + 1]);
        a.kb.est[j] = est;
        // cycle exits (gmres.cpp:137-146)
        const bool conv = est <= st->thr;
        if (conv) st->converged_est = 1;
        if (breakdown) st->breakdown = 1;
        st->pre_norm = pre_norm;
        st->last_est = est;
        st->j = j + 1;
        const int done = (conv || breakdown || est <= st->attainable || j + 1 >= m) ? 1 : 0;
        st->done = done;
        if (a.cond) cudaGraphSetConditional(a.cond, done ? 0u : 1u);
    }
    __syncwarp();
    for (int i = lane; i <= j + 1; i += 32) Rj[i] = sR[i];
}

// ---------------------------------------------------------------------------
template <bool SMEM>
__global__ void __launch_bounds__(kMgsThreads, 1) k_mgs(OrthArgs a) {
    SolveState* st = a.st;
    if (st->done) return;  // uniform: nothing writes done before the final barrier
    extern __shared__ __align__(16) double dsm_mgs[];
    double* wsh = dsm_mgs + a.scr;
    __shared__ double red[2][kMgsThreads / 32];
    __shared__ double bc[2];

    const int j = st->j;
    const int m = a.kb.m;
    const int ldv = a.kb.ldv;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int r0 = blockIdx.x * a.slice;
    const int len = max(0, min(a.slice, a.npad - r0));
    const int nv2 = len >> 1;
    double* P = a.kb.partials;  // [2 parity][2 quantity][G]

    double2* w2 = SMEM ? reinterpret_cast<double2*>(wsh) : reinterpret_cast<double2*>(a.kb.w + r0);
    const double2* win = reinterpret_cast<const double2*>(a.kb.w + r0);
    const double* V = a.kb.V;

    unsigned long long pacc[5] = {0, 0, 0, 0, 0};
    long long tp = a.prof ? clock64() : 0;
    auto reduce2 = [&](double x0, double x1, int parity) {
        x0 = warp_sum(x0);
        x1 = warp_sum(x1);
        if (lane == 0) {
            red[0][wid] = x0;
            red[1][wid] = x1;
        }
        __syncthreads();
        long long t1 = 0;
        if (a.prof) {
            t1 = clock64();
            pacc[0] += t1 - tp;
        }
        if (wid == 0) {
            double t0 = lane < kMgsThreads / 32 ? red[0][lane] : 0.0;
            double t1 = lane < kMgsThreads / 32 ? red[1][lane] : 0.0;
            t0 = warp_sum(t0);
            t1 = warp_sum(t1);
            if (lane == 0) {
                P[(parity * 2 + 0) * G + blockIdx.x] = t0;
                P[(parity * 2 + 1) * G + blockIdx.x] = t1;
            }
        }
        long long t2 = 0;
        if (a.prof) t2 = clock64();
        grid_barrier(a.gb);
        long long t3 = 0;
        if (a.prof) t3 = clock64();
        if (wid < 2) {  // the two totals by two warps at once
            const double t = sum_partials(P + (parity * 2 + wid) * G, G);
            if (lane == 0) bc[wid] = t;
        }
        __syncthreads();
        if (a.prof) {
            tp = clock64();
            pacc[1] += t2 - t1;
            pacc[2] += t3 - t2;
            pacc[3] += tp - t3;
            pacc[4] += 1;
        }
    };

    // The first kMgsPre loads of every pass's HBM vector are issued before
    // the previous pass's grid barrier, so they land while the CTA waits.
    double2 pre[kMgsPre];
    auto preload = [&](int i) {
        const double2* vi = reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0);
#pragma unroll
        for (int g = 0; g < kMgsPre; ++g) {
            const int e = tid + g * kMgsThreads;
            pre[g] = e < nv2 ? __ldg(vi + e) : make_double2(0.0, 0.0);
        }
    };

    // pass 0: stage w on chip, ||w||^2 and <v_0, w>
    double ss = 0.0, dt = 0.0;
    {
        const double2* v0 = reinterpret_cast<const double2*>(V + r0);
#pragma unroll 4
        for (int e = tid; e < nv2; e += kMgsThreads) {
            const double2 wv = __ldcg(win + e);
            const double2 vv = __ldg(v0 + e);
            if (SMEM) w2[e] = wv;
            ss = fma(wv.x, wv.x, ss);
            ss = fma(wv.y, wv.y, ss);
            dt = fma(vv.x, wv.x, dt);
            dt = fma(vv.y, wv.y, dt);
        }
    }
    if (j >= 1) preload(1);
    reduce2(ss, dt, 0);
    const double pre_norm = sqrt(bc[0]);
    double h = bc[1];
    if (blockIdx.x == 0 && tid == 0) a.kb.H[(size_t)j * (m + 1) + 0] = h;

    // passes 1..j: w -= h_{i-1} v_{i-1}; h_i = <v_i, w>
    for (int i = 1; i <= j; ++i) {
        const double2* vp = reinterpret_cast<const double2*>(V + (size_t)(i - 1) * ldv + r0);
        const double2* vi = reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0);
        dt = 0.0;
#pragma unroll
        for (int g = 0; g < kMgsPre; ++g) {
            const int e = tid + g * kMgsThreads;
            if (e < nv2) {
                double2 wv = w2[e];
                const double2 pv = __ldg(vp + e);
                const double2 qv = pre[g];
                wv.x = fma(-h, pv.x, wv.x);
                wv.y = fma(-h, pv.y, wv.y);
                w2[e] = wv;
                dt = fma(qv.x, wv.x, dt);
                dt = fma(qv.y, wv.y, dt);
            }
        }
#pragma unroll 4
        for (int e = tid + kMgsPre * kMgsThreads; e < nv2; e += kMgsThreads) {
            double2 wv = w2[e];
            const double2 pv = __ldg(vp + e);
            const double2 qv = __ldg(vi + e);
            wv.x = fma(-h, pv.x, wv.x);
            wv.y = fma(-h, pv.y, wv.y);
            w2[e] = wv;
            dt = fma(qv.x, wv.x, dt);
            dt = fma(qv.y, wv.y, dt);
        }
        if (i + 1 <= j) preload(i + 1);
        reduce2(0.0, dt, i & 1);
        h = bc[1];
        if (blockIdx.x == 0 && tid == 0) a.kb.H[(size_t)j * (m + 1) + i] = h;
    }

    // final pass: w -= h_j v_j; ||w||
    {
        const double2* vp = reinterpret_cast<const double2*>(V + (size_t)j * ldv + r0);
        ss = 0.0;
#pragma unroll 4
        for (int e = tid; e < nv2; e += kMgsThreads) {
            double2 wv = w2[e];
            const double2 pv = __ldg(vp + e);
            wv.x = fma(-h, pv.x, wv.x);
            wv.y = fma(-h, pv.y, wv.y);
            w2[e] = wv;
            ss = fma(wv.x, wv.x, ss);
            ss = fma(wv.y, wv.y, ss);
        }
    }
    reduce2(ss, 0.0, (j + 1) & 1);
    if (a.prof && tid == 0)
        for (int k = 0; k < 5; ++k) atomicAdd(a.prof + (size_t)blockIdx.x * 5 + k, pacc[k]);
    finish_step(a, w2, dsm_mgs, r0, nv2, j, pre_norm, sqrt(bc[0]), kMgsThreads);
}

// ---------------------------------------------------------------------------
// Pipelined textbook MGS (w slice in shared memory): no projection pass waits
// for the grid.
//
// Warps 0..30 stream; warp 31 only communicates. Pass i (streaming warps)
// merges u -= h_{i-2} v_{i-2} (v_{i-2} read two passes ago: about half of it
// still in L2; loaded evict-first, its last use) with
// d_i = <v_i, u>; at the dot u lacks only h_{i-1} v_{i-1}, so
//   h_i = d_i - h_{i-1} <v_i, v_{i-1}>
// is exactly <v_i, w - sum_{k<i} h_k v_k> (the missing term is linear).
// <v_{k+1}, v_k> is a by-product of the step that created v_{k+1} (final pass:
// <u, v_k> / ||u||), kept in gram[(k+1)(m+1) + k].
//
// While pass i+1 streams, the communication warp exchanges the partial sums
// of pass i: every CTA stores its two partials into ll[slot i & 3][cta] as
// four 64-bit words (32 payload bits << 32 | 32-bit epoch). A 64-bit word is
// single-copy atomic, so data and flag arrive together: relaxed stores and
// loads, no fence, no atomic. CTA 0 polls all CTAs' words (all loads of a
// round in flight together), sums the partials in the order of sum_partials
// (run-to-run reproducible), and stores the totals the same way into
// tot[slot], which the other CTAs poll (one line). The warp then forms h_i
// and leaves it in shared memory for pass i+2. A slot is reused four passes
// later: a CTA that publishes pass p + 4 has read the totals of pass p + 3,
// which CTA 0 stored after reading every partial of pass p + 3, which each
// CTA stored after reading the totals of pass p. Only h_j and the final norm
// wait for the grid.
constexpr int kPipeStream = kMgsThreads - 32;  // streaming threads
__device__ __forceinline__ unsigned long long l2_policy_evict_normal() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, unsigned long long pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

__global__ void __launch_bounds__(kMgsThreads, 1) k_mgs_pipe(OrthArgs a) {
    SolveState* st = a.st;
    if (st->done) return;
    extern __shared__ __align__(16) double dsm_mgs[];
    double* wsh = dsm_mgs + a.scr;
    __shared__ double red[2][2][32];  // [pass parity][quantity][warp]
    __shared__ double hs[2];          // h_i by pass parity
    __shared__ double misc[2];        // pre_norm^2, final ||w||^2

    const int j = st->j;
    const int m = a.kb.m;
    const int ldv = a.kb.ldv;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const bool comm = wid == kMgsThreads / 32 - 1;
    const int r0 = blockIdx.x * a.slice;
    const int len = max(0, min(a.slice, a.npad - r0));
    const int nv2 = len >> 1;
    GridBarrier* gb = a.gb;
    const unsigned long long seq = __ldcg(&gb->seq);
    const unsigned long long ebase = (seq + 1ull) << 12;  // passes per launch <= m + 2 < 4096
    // The epoch is 32 bits (2^20 launches): every 2^16 launches each CTA wipes
    // its own words, so no stale word is old enough to match after the wrap.
    if ((seq & 0xffffull) == 0 && tid < kFlagSlots * 4) {
        gb->ll[tid >> 2][blockIdx.x][tid & 3] = 0ull;
        if (blockIdx.x == 0) gb->tot[tid >> 2][tid & 3] = 0ull;
    }

    double2* w2 = reinterpret_cast<double2*>(wsh);
    const double2* win = reinterpret_cast<const double2*>(a.kb.w + r0);
    const double* V = a.kb.V;
    const double* gsub = a.gram;  // <v_i, v_{i-1}> at gram[i (m+1) + i-1]
    double* Hj = a.kb.H + (size_t)j * (m + 1);
    // The stream keeps the default priority; the re-read is the last use of a
    // line (evict-first). Measured on config 3: 201 us/step; without the
    // evict-first 255; with the stream also evict-last 201, but the lines that
    // stay behind slow the next apply by 10 us.
    const unsigned long long pol_last = l2_policy_evict_normal(), pol_first = l2_policy_evict_first();

    // streaming warps: leave the warp partials of pass p
    auto deposit = [&](double x0, double x1, int p) {
        x0 = warp_sum(x0);
        x1 = warp_sum(x1);
        if (lane == 0) {
            red[p & 1][0][wid] = x0;
            red[p & 1][1][wid] = x1;
        }
    };
    // communication warp, after the CTA barrier that ends pass p: publish the
    // CTA partial, gather all CTAs'; returns the two totals (all lanes)
    double hlast = 0.0;  // communication warp: h_{p-1}
    auto ll_store = [&](unsigned long long* q, double x0, double x1, unsigned long long ep) {
        const unsigned long long b0 = (unsigned long long)__double_as_longlong(x0);
        const unsigned long long b1 = (unsigned long long)__double_as_longlong(x1);
        sync::st_relaxed_v2u64(q, (b0 << 32) | ep, (b0 & 0xffffffff00000000ull) | ep);
        sync::st_relaxed_v2u64(q + 2, (b1 << 32) | ep, (b1 & 0xffffffff00000000ull) | ep);
    };
    auto ll_decode = [](unsigned long long lo, unsigned long long hi) {
        return __longlong_as_double((long long)((lo >> 32) | (hi & 0xffffffff00000000ull)));
    };
    auto exchange = [&](int p, double& c0, double& c1) {
        const int slot = p & (kFlagSlots - 1);
        const unsigned long long want = ebase + (unsigned)p;  // low 32 bits are the epoch
        const unsigned ep32 = (unsigned)want;
        double t0 = lane < kPipeStream / 32 ? red[p & 1][0][lane] : 0.0;
        double t1 = lane < kPipeStream / 32 ? red[p & 1][1][lane] : 0.0;
        t0 = warp_sum(t0);
        t1 = warp_sum(t1);
        if (blockIdx.x != 0) {
            if (lane == 0) ll_store(gb->ll[slot][blockIdx.x], t0, t1, want & 0xffffffffull);
            // the totals come back from CTA 0 (one line, one request per poll)
            unsigned long long w0, w1, w2, w3;
            for (;;) {
                sync::ld_relaxed_v2u64(gb->tot[slot], w0, w1);
                sync::ld_relaxed_v2u64(gb->tot[slot] + 2, w2, w3);
                if ((unsigned)w0 == ep32 && (unsigned)w1 == ep32 && (unsigned)w2 == ep32 && (unsigned)w3 == ep32) break;
                __nanosleep(64);
            }
            c0 = ll_decode(w0, w1);
            c1 = ll_decode(w2, w3);
            return;
        }
        // CTA 0: lane l gathers CTAs l, l + 32, ... (all loads of a round in
        // flight together); a word whose low half is the epoch carries this
        // pass's data. Its own partial goes in directly.
        constexpr int kPer = kFlagMaxCtas / 32;
        unsigned long long wd[kPer][4];
        for (;;) {
            bool ok = true;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int c = lane + 32 * k;
                if (c < G && c > 0) {
                    sync::ld_relaxed_v2u64(gb->ll[slot][c], wd[k][0], wd[k][1]);
                    sync::ld_relaxed_v2u64(gb->ll[slot][c] + 2, wd[k][2], wd[k][3]);
                }
            }
#pragma unroll
            for (int k = 0; k < kPer; ++k)
                if (lane + 32 * k < G && lane + 32 * k > 0)
                    ok &= (unsigned)wd[k][0] == ep32 && (unsigned)wd[k][1] == ep32 && (unsigned)wd[k][2] == ep32 &&
                          (unsigned)wd[k][3] == ep32;
            if (ok) break;
        }
        // the summation order of sum_partials: lane-strided, then the xor tree
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int c = lane + 32 * k;
            if (c == 0) {
                s0 += t0;
                s1 += t1;
            } else if (c < G) {
                s0 += ll_decode(wd[k][0], wd[k][1]);
                s1 += ll_decode(wd[k][2], wd[k][3]);
            }
        }
        c0 = warp_sum(s0);
        c1 = warp_sum(s1);
        if (lane == 0) ll_store(gb->tot[slot], c0, c1, want & 0xffffffffull);
    };
    // communication warp: h_p from the totals of pass p -> hs[p & 1], H
    auto coefficient = [&](int p, double c0, double c1) {
        double h = c1;
        if (p == 0) {
            if (lane == 0) misc[0] = c0;
        } else {
            h = fma(-hlast, __ldcg(gsub + (size_t)p * (m + 1) + (p - 1)), c1);
        }
        hlast = h;
        if (lane == 0) {
            hs[p & 1] = h;
            if (blockIdx.x == 0) Hj[p] = h;
        }
    };

    // pass 0: stage w on chip, ||w||^2 and <v_0, w>
    if (!comm) {
        double ss = 0.0, dt = 0.0;
        const double2* v0 = reinterpret_cast<const double2*>(V + r0);
#pragma unroll 4
        for (int e = tid; e < nv2; e += kPipeStream) {
            const double2 wv = __ldcg(win + e);
            const double2 vv = ld_hint(v0 + e, pol_last);
            w2[e] = wv;
            ss = fma(wv.x, wv.x, ss);
            ss = fma(wv.y, wv.y, ss);
            dt = fma(vv.x, wv.x, dt);
            dt = fma(vv.y, wv.y, dt);
        }
        deposit(ss, dt, 0);
    }
    __syncthreads();  // end of pass 0

    // passes 1..j; the communication warp works one pass behind
    for (int i = 1; i <= j; ++i) {
        if (comm) {
            double c0, c1;
            exchange(i - 1, c0, c1);
            coefficient(i - 1, c0, c1);
        } else {
            const double2* vi = reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0);
            double dt = 0.0;
            if (i >= 2) {
                const double h = hs[i & 1];  // h_{i-2}: written before the barrier that ended pass i-1
                const double2* vp = reinterpret_cast<const double2*>(V + (size_t)(i - 2) * ldv + r0);
#pragma unroll 4
                for (int e = tid; e < nv2; e += kPipeStream) {
                    double2 wv = w2[e];
                    const double2 pv = ld_hint(vp + e, pol_first);
                    const double2 qv = ld_hint(vi + e, pol_last);
                    wv.x = fma(-h, pv.x, wv.x);
                    wv.y = fma(-h, pv.y, wv.y);
                    w2[e] = wv;
                    dt = fma(qv.x, wv.x, dt);
                    dt = fma(qv.y, wv.y, dt);
                }
            } else {
#pragma unroll 8
                for (int e = tid; e < nv2; e += kPipeStream) {
                    const double2 wv = w2[e];
                    const double2 qv = ld_hint(vi + e, pol_last);
                    dt = fma(qv.x, wv.x, dt);
                    dt = fma(qv.y, wv.y, dt);
                }
            }
            deposit(0.0, dt, i);
        }
        __syncthreads();  // end of pass i: red[i & 1] and hs[(i - 1) & 1] are published
    }

    // h_j: the one projection coefficient the CTA waits for
    if (comm) {
        double c0, c1;
        exchange(j, c0, c1);
        coefficient(j, c0, c1);
    }
    __syncthreads();
    const double pre_norm = sqrt(misc[0]);

    // final pass: w -= h_{j-1} v_{j-1} + h_j v_j; ||w||^2 and <w, v_j>
    if (!comm) {
        const double hj = hs[j & 1];
        const double hj1 = j >= 1 ? hs[(j - 1) & 1] : 0.0;
        const double2* vp = reinterpret_cast<const double2*>(V + (size_t)j * ldv + r0);
        const double2* vq = reinterpret_cast<const double2*>(V + (size_t)max(j - 1, 0) * ldv + r0);
        double ss = 0.0, gv = 0.0;
        if (j >= 1) {
#pragma unroll 4
            for (int e = tid; e < nv2; e += kPipeStream) {
                double2 wv = w2[e];
                const double2 qv = ld_hint(vq + e, pol_first);
                const double2 pv = __ldg(vp + e);
                wv.x = fma(-hj1, qv.x, wv.x);  // MGS order: v_{j-1} first
                wv.y = fma(-hj1, qv.y, wv.y);
                wv.x = fma(-hj, pv.x, wv.x);
                wv.y = fma(-hj, pv.y, wv.y);
                w2[e] = wv;
                ss = fma(wv.x, wv.x, ss);
                ss = fma(wv.y, wv.y, ss);
                gv = fma(wv.x, pv.x, gv);
                gv = fma(wv.y, pv.y, gv);
            }
        } else {
#pragma unroll 4
            for (int e = tid; e < nv2; e += kPipeStream) {
                double2 wv = w2[e];
                const double2 pv = __ldg(vp + e);
                wv.x = fma(-hj, pv.x, wv.x);
                wv.y = fma(-hj, pv.y, wv.y);
                w2[e] = wv;
                ss = fma(wv.x, wv.x, ss);
                ss = fma(wv.y, wv.y, ss);
                gv = fma(wv.x, pv.x, gv);
                gv = fma(wv.y, pv.y, gv);
            }
        }
        deposit(ss, gv, j + 1);
    }
    __syncthreads();
    if (comm) {
        double c0, c1;
        exchange(j + 1, c0, c1);
        if (lane == 0) {
            misc[1] = c0;
            if (blockIdx.x == 0) {
                const double hn = sqrt(c0);
                a.gram[(size_t)(j + 1) * (m + 1) + j] = hn > 0.0 ? c1 / hn : 0.0;
                gb->seq = ebase >> 12;  // every CTA read seq before its first publish, all of which this warp has seen
            }
        }
    }
    __syncthreads();
    finish_step(a, w2, dsm_mgs, r0, nv2, j, pre_norm, sqrt(misc[1]), kMgsThreads);
}

// ---------------------------------------------------------------------------
constexpr int kIcwyWarps = kIcwyThreads / 32;
constexpr int kBatch = 8;  // basis vectors per multi-dot batch (16 dot products; 1024 threads x 64 registers:
                           // the multi-dot pass is latency bound, more rows in flight beat longer batches)

template <bool SMEM>
__global__ void __launch_bounds__(kIcwyThreads, 1) k_icwy(OrthArgs a) {
    SolveState* st = a.st;
    if (st->done) return;
    extern __shared__ __align__(16) double dsm[];
    // dynamic smem: [w slice][v_j slice] when SMEM
    __shared__ double red[kIcwyWarps][2 * kBatch];  // per-warp batch partials
    __shared__ double acc_sh[kMaxRestart * 2 + 4];  // CTA partials of c, l, ss
    __shared__ double tot[kMaxRestart * 2 + 4];     // grid totals
    __shared__ double hsh[kMaxRestart + 1];
    __shared__ double h1[kMaxRestart + 1];
    __shared__ double wred[kIcwyWarps];

    const int j = st->j;
    const int m = a.kb.m;
    const int ldv = a.kb.ldv;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int r0 = blockIdx.x * a.slice;
    const int len = max(0, min(a.slice, a.npad - r0));
    const int nv2 = len >> 1;
    const int nval = 2 * (j + 1) + 1;  // c_0..c_j, l_0..l_j, ||w||^2
    double* P = a.kb.partials;         // [value][G]

    double2* w2 = SMEM ? reinterpret_cast<double2*>(dsm + a.scr) : reinterpret_cast<double2*>(a.kb.w + r0);
    const double2* vj2 = reinterpret_cast<const double2*>(a.kb.V + (size_t)j * ldv + r0);
    const double2* win = reinterpret_cast<const double2*>(a.kb.w + r0);
    const double* V = a.kb.V;

    // ---- stage w, ||w||^2
    double ss = 0.0;
    for (int e = tid; e < nv2; e += kIcwyThreads) {
        const double2 wv = __ldcg(win + e);
        if (SMEM) w2[e] = wv;
        ss = fma(wv.x, wv.x, ss);
        ss = fma(wv.y, wv.y, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) wred[wid] = ss;
    __syncthreads();

    // ---- pass A: fused multi-dot  c_i = <v_i, w>,  l_i = <v_i, v_j>
    for (int i0 = 0; i0 <= j; i0 += kBatch) {
        const int nb = min(kBatch, j + 1 - i0);
        double acc[2 * kBatch];
#pragma unroll
        for (int q = 0; q < 2 * kBatch; ++q) acc[q] = 0.0;
        for (int e = tid; e < nv2; e += kIcwyThreads) {
            const double2 wv = w2[e];
            const double2 jv = __ldg(vj2 + e);
#pragma unroll
            for (int q = 0; q < kBatch; ++q) {
                if (q < nb) {
                    const double2 vv = __ldg(reinterpret_cast<const double2*>(V + (size_t)(i0 + q) * ldv + r0) + e);
                    acc[q] = fma(vv.x, wv.x, acc[q]);
                    acc[q] = fma(vv.y, wv.y, acc[q]);
                    acc[kBatch + q] = fma(vv.x, jv.x, acc[kBatch + q]);
                    acc[kBatch + q] = fma(vv.y, jv.y, acc[kBatch + q]);
                }
            }
        }
        const double r = transpose_reduce<2 * kBatch>(acc, lane);
        if (lane < 2 * kBatch) red[wid][lane] = r;
        __syncthreads();
        if (tid < 2 * kBatch) {
            double s = 0.0;
            for (int w = 0; w < kIcwyWarps; ++w) s += red[w][tid];
            const int q = tid & (kBatch - 1);
            if (q < nb) acc_sh[(tid < kBatch ? 0 : (j + 1)) + i0 + q] = s;
        }
        __syncthreads();
    }
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kIcwyWarps; ++w) s += wred[w];
        acc_sh[2 * (j + 1)] = s;
    }
    __syncthreads();
    for (int t = tid; t < nval; t += kIcwyThreads) P[(size_t)t * G + blockIdx.x] = acc_sh[t];
    grid_barrier(a.gb);
    // grid totals: one warp per value, lane-strided over CTAs then a fixed
    // xor tree (every CTA computes the same bits)
    for (int t0 = wid; t0 < nval; t0 += 4 * kIcwyWarps) {
        double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // all loads of four values in flight together
            const int t = t0 + u * kIcwyWarps;
            if (t < nval)
                part[u] = lane_sum_partials(P + (size_t)t * G, G);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double tv = warp_sum(part[u]);
            const int t = t0 + u * kIcwyWarps;
            if (lane == 0 && t < nval) tot[t] = tv;
        }
    }
    __syncthreads();
    const double pre_norm = sqrt(tot[2 * (j + 1)]);
    const int ldl = m + 1;
    // ---- h = (I + L)^-1 c, L_ik = <v_i, v_k> (k < i); row j is new.
    // Two Jacobi sweeps h <- c - L h (exact to O(|L|^3)); warp per row,
    // lanes over k, fixed reduction order.
    auto sweep = [&](const double* src, double* dst) {
        for (int i = wid; i <= j; i += kIcwyWarps) {
            const double* Lrow = (i == j) ? tot + (j + 1) : a.gram + (size_t)i * ldl;
            double sacc = 0.0;
            for (int k = lane; k < i; k += 32) sacc = fma(i == j ? Lrow[k] : __ldcg(Lrow + k), src[k], sacc);
            sacc = warp_sum(sacc);
            if (lane == 0) dst[i] = tot[i] - sacc;
        }
        __syncthreads();
    };
    sweep(tot, h1);
    sweep(h1, hsh);
    if (blockIdx.x == 0) {
        for (int i = tid; i <= j; i += kIcwyThreads) a.kb.H[(size_t)j * (m + 1) + i] = hsh[i];
        for (int k = tid; k < j; k += kIcwyThreads) a.gram[(size_t)j * ldl + k] = tot[(j + 1) + k];
    }

    // ---- pass B: w -= sum_i h_i v_i in MGS order; ||w||^2
    double ss2 = 0.0;
    // rows in reverse: pass A streamed the rows ascending, so the highest rows
    // of its last batch of vectors are the ones still in L2
    for (int e = nv2 - 1 - tid; e >= 0; e -= kIcwyThreads) {
        double2 wv = w2[e];
        for (int i = 0; i <= j; ++i) {
            const double2 vv = __ldg(reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0) + e);
            const double hi = hsh[i];
            wv.x = fma(-hi, vv.x, wv.x);
            wv.y = fma(-hi, vv.y, wv.y);
        }
        w2[e] = wv;
        ss2 = fma(wv.x, wv.x, ss2);
        ss2 = fma(wv.y, wv.y, ss2);
    }
    ss2 = warp_sum(ss2);
    if (lane == 0) wred[wid] = ss2;
    __syncthreads();
    double* P2 = P + (size_t)(2 * kMaxRestart + 4) * G;
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kIcwyWarps; ++w) s += wred[w];
        P2[blockIdx.x] = s;
    }
    grid_barrier(a.gb);
    if (wid == 0) {
        const double t0 = sum_partials(P2, G);
        if (lane == 0) wred[0] = t0;
    }
    __syncthreads();
    finish_step(a, w2, dsm, r0, nv2, j, pre_norm, sqrt(wred[0]), kIcwyThreads);
}

// v_0 = r0 / beta (element-wise division, gmres.cpp:120-122); cycle state.
__global__ void k_cycle_init(KrylovBufs kb, SolveState* st, const double* __restrict__ r, int n,
                             cudaGraphConditionalHandle cond) {
    const double beta = st->rnorm;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        kb.V[i] = r[i] / beta;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->beta = beta;
        st->attainable = 10.0 * st->floor_roundoff * beta;
        st->j = 0;
        const bool conv = beta <= st->thr;
        st->done = conv ? 1 : 0;
        st->converged_est = conv ? 1 : 0;
        st->breakdown = 0;
        st->rank_deficient = 0;
        kb.g[0] = beta;
        for (int i = 1; i <= kb.m; ++i) kb.g[i] = 0.0;
        if (cond) cudaGraphSetConditional(cond, conv ? 0u : 1u);
    }
}

// Restart-driver bookkeeping (gmres.cpp:236-258) on the device: history rows
// (cycle, ++iteration, est/||b||), cycle residual, exit test. One warp.
__global__ void k_cycle_end(KrylovBufs kb, SolveState* st, cudaGraphConditionalHandle cond) {
    if (blockIdx.x != 0) return;
    const int steps = st->j;
    const int cyc = st->cycles;
    const int h0 = st->hist_len;
    const double bnorm = st->bnorm;
    for (int k = threadIdx.x; k < steps; k += blockDim.x) {
        kb.hist[h0 + k] = kb.est[k] / bnorm;
        kb.hist_cycle[h0 + k] = cyc;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    st->hist_len = h0 + steps;
    st->total_iterations += steps;
    st->breakdown_any |= st->breakdown;
    st->rank_any |= st->rank_deficient;
    const double rnorm = st->rnorm;
    kb.cycres[cyc] = rnorm / bnorm;
    st->cycles = cyc + 1;
    st->last_steps = steps;
    const bool conv = rnorm <= st->thr;
    st->converged = conv ? 1 : 0;
    const bool more = !conv && st->cycles < st->max_restarts && steps > 0;
    if (cond) cudaGraphSetConditional(cond, more ? 1u : 0u);
}

// y = R^-1 g with the zero-rotation convention (gmres.cpp:57-66), same
// operation order as the reference. The triangle is staged in shared memory
// by the whole CTA so the single-thread recurrence runs at smem latency.
constexpr int kSolveYThreads = 256;
constexpr int kSolveYStagedMax = 160;  // m^2 doubles of shared memory
template <bool STAGED>
__global__ void __launch_bounds__(kSolveYThreads) k_solve_y(KrylovBufs kb, const SolveState* st) {
    extern __shared__ double rs[];  // steps x steps, rs[k * steps + i] = R(i, k)
    __shared__ double ysh[1024];
    const int steps = st->j;
    const int ld = kb.m + 1;
    if (STAGED) {
        for (int t = threadIdx.x; t < steps * steps; t += kSolveYThreads) {
            const int k = t / steps, i = t - k * steps;
            rs[t] = kb.R[(size_t)k * ld + i];
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    auto R = [&](int i, int k) { return STAGED ? rs[k * steps + i] : kb.R[(size_t)k * ld + i]; };
    for (int i = steps - 1; i >= 0; --i) {
        const double rii = R(i, i);
        if (rii == 0.0) {
            ysh[i] = 0.0;
            continue;
        }
        double s = kb.g[i];
        for (int k = i + 1; k < steps; ++k) s -= R(i, k) * ysh[k];
        ysh[i] = s / rii;
    }
    for (int i = 0; i < steps; ++i) kb.y[i] = ysh[i];
}

}  // namespace

size_t orth_partials_doubles(int num_sms) { return (size_t)(2 * kMaxRestart + 8) * num_sms * 2; }

MgsLaunch plan_mgs(int n, int num_sms, int m) {
    MgsLaunch L;
    const int npad = (n + 1) & ~1;
    // compact-WY when a basis vector streams faster than a grid barrier
    // (~1.5 us: 8 n bytes at HBM rate) and the Gram/accumulator tables fit.
    const char* env = getenv("HPBJ_ORTH");
    bool icwy = (size_t)n * 8 <= (size_t)12 * 1024 * 1024 && m <= kMaxRestart;
    if (env && std::string(env) == "mgs") icwy = false;
    if (env && std::string(env) == "icwy" && m <= kMaxRestart) icwy = true;
    L.icwy = icwy;
    const char* fm = getenv("HPBJ_MGS");  // bar: the grid-barrier kernel
    L.pipelined = !(fm && std::string(fm) == "bar");
    L.threads = icwy ? kIcwyThreads : kMgsThreads;
    const int min_rows = icwy ? 1024 : 4096;
    int grid = std::max(1, std::min(num_sms, (npad + min_rows - 1) / min_rows));
    int slice = (npad + grid - 1) / grid;
    slice = (slice + 1) & ~1;
    L.grid = grid;
    L.slice = slice;
    L.scr = (3 * m + 2 + 1) & ~1;  // Givens scratch of finish_step (CTA 0)
    const size_t scr_bytes = (size_t)L.scr * sizeof(double);
    const size_t static_smem = icwy ? (size_t)(kIcwyWarps * 2 * kBatch + 3 * (kMaxRestart * 2 + 4)) * 8 + 1024
                                    : 2048;
    L.w_in_smem = scr_bytes + (size_t)slice * sizeof(double) + static_smem <= kSmemMax;
    L.smem = scr_bytes + (L.w_in_smem ? (size_t)slice * sizeof(double) : 0);
    return L;
}

void launch_mgs(const MgsLaunch& L, const KrylovBufs& kb, double* gram, GridBarrier* gb, SolveState* sst,
                int n, cudaGraphConditionalHandle cond, cudaStream_t st, int64_t* launches) {
    static unsigned long long* prof = nullptr;
    static int prof_calls = 0;
    static const bool want_prof = getenv("HPBJ_MGS_PROF") != nullptr;
    if (want_prof && !prof) {
        HPBJ_CUDA(cudaMallocManaged(&prof, sizeof(unsigned long long) * 5 * L.grid));
        HPBJ_CUDA(cudaMemset(prof, 0, sizeof(unsigned long long) * 5 * L.grid));
    }
    OrthArgs a{kb, gram, sst, gb, n, L.slice, (n + 1) & ~1, cond, L.scr, want_prof && !L.icwy ? prof : nullptr};
    void (*fn)(OrthArgs);
    if (L.icwy) fn = L.w_in_smem ? k_icwy<true> : k_icwy<false>;
    else if (L.w_in_smem && L.pipelined && L.grid <= kFlagMaxCtas) fn = k_mgs_pipe;
    else fn = L.w_in_smem ? k_mgs<true> : k_mgs<false>;
    if (L.smem > 48 * 1024)
        HPBJ_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
    // cooperative attribute: co-residency guaranteed, capturable into graphs
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L.grid);
    cfg.blockDim = dim3(L.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HPBJ_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
    *launches += 1;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (a.prof && cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone &&
        ++prof_calls % 200 == 0) {
        HPBJ_CUDA(cudaStreamSynchronize(st));
        // per phase: min / mean / max over CTAs of the cycles per pass
        double mn[4] = {1e30, 1e30, 1e30, 1e30}, mx[4] = {0, 0, 0, 0}, me[4] = {0, 0, 0, 0};
        for (int c = 0; c < L.grid; ++c) {
            const double np = (double)std::max(1ull, prof[(size_t)c * 5 + 4]);
            for (int k = 0; k < 4; ++k) {
                const double v = prof[(size_t)c * 5 + k] / np;
                mn[k] = std::min(mn[k], v);
                mx[k] = std::max(mx[k], v);
                me[k] += v / L.grid;
            }
        }
        fprintf(stderr, "[hpbj mgs prof] %d launches, %.0f passes/launch; cycles per pass (min/mean/max over CTAs): "
                "stream %.0f/%.0f/%.0f  cta-reduce %.0f/%.0f/%.0f  grid-barrier %.0f/%.0f/%.0f  broadcast %.0f/%.0f/%.0f\n",
                prof_calls, (double)prof[4] / prof_calls, mn[0], me[0], mx[0], mn[1], me[1], mx[1], mn[2], me[2], mx[2],
                mn[3], me[3], mx[3]);
    }
}

void launch_cycle_init(const KrylovBufs& kb, SolveState* sst, const double* r, int n,
                       cudaGraphConditionalHandle cond, cudaStream_t st, int64_t* launches) {
    const int grid = std::max(1, std::min((n + 255) / 256, 148 * 8));
    k_cycle_init<<<grid, 256, 0, st>>>(kb, sst, r, n, cond);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_cycle_end(const KrylovBufs& kb, SolveState* sst, cudaGraphConditionalHandle cond, cudaStream_t st,
                      int64_t* launches) {
    k_cycle_end<<<1, 128, 0, st>>>(kb, sst, cond);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_solve_y(const KrylovBufs& kb, SolveState* sst, cudaStream_t st, int64_t* launches) {
    if (kb.m <= kSolveYStagedMax) {
        const size_t smem = sizeof(double) * (size_t)kb.m * kb.m;
        if (smem > 48 * 1024)
            HPBJ_CUDA(cudaFuncSetAttribute(k_solve_y<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_solve_y<true><<<1, kSolveYThreads, smem, st>>>(kb, sst);
    } else {
        k_solve_y<false><<<1, kSolveYThreads, 0, st>>>(kb, sst);
    }
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
