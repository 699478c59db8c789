// Arnoldi modified Gram-Schmidt + progressive Givens, device resident —
// replaces arnoldi_step (gmres.hpp:43-75), dot/norm2 (dense_ops.hpp:14-46)
// and GivensLs::push_column (gmres.cpp:26-52) plus the loop exits of
// run_cycle (gmres.cpp:130-146).
//
// k_mgs is a persistent cooperative kernel: every CTA owns a contiguous
// slice of w = A M^-1 v_j and keeps it in shared memory for the whole MGS
// sweep (config 3: 4.1M doubles over 148 SMs = 221 KB/SM), so each basis
// vector streams from HBM once for its dot product and once more (L2-hot)
// for its axpy, while w never round-trips to HBM. Per inner step i:
//     w -= h_{i-1} v_{i-1};  partial <v_i, w>;  grid sync;  h_i = sum(partials)
// Every CTA sums the per-CTA partials in the same fixed order, so all CTAs
// hold a bit-identical h_i without a second barrier, and the reduction is
// run-to-run deterministic. CTA 0 finishes the step: Hessenberg column,
// Givens rotation, residual estimate and the cycle-exit flags, all written
// to device memory (SolveState) — no host round-trip per iteration.

#include <cooperative_groups.h>

#include "device.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace hpbj {

namespace {

constexpr int kMgsThreads = 1024;
constexpr size_t kMgsSmemMax = 227 * 1024 - 1024;

struct MgsArgs {
    KrylovBufs kb;
    SolveState* st;
    int n;
    int slice;  // rows per CTA (even)
    int npad;   // n rounded up to even; vectors are zero padded to npad
};

template <bool SMEM>
__global__ void __launch_bounds__(kMgsThreads, 1) k_mgs(MgsArgs a) {
    cg::grid_group grid = cg::this_grid();
    SolveState* st = a.st;
    if (st->done) return;  // uniform: nothing writes done before the final barrier
    extern __shared__ __align__(16) double wsh[];
    __shared__ double red[2][kMgsThreads / 32];
    __shared__ double bc[2];

    const int j = st->j;
    const int m = a.kb.m;
    const int ldv = a.kb.ldv;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int r0 = blockIdx.x * a.slice;
    const int len = max(0, min(a.slice, a.npad - r0));
    const int nv2 = len >> 1;  // double2 per slice
    double* P = a.kb.partials;  // [2 parity][2 quantity][G]

    double2* w2 = SMEM ? reinterpret_cast<double2*>(wsh) : reinterpret_cast<double2*>(a.kb.w + r0);
    const double2* win = reinterpret_cast<const double2*>(a.kb.w + r0);
    const double* V = a.kb.V;

    auto reduce2 = [&](double x0, double x1, int parity) {
        // block sums (fixed order) -> partials -> grid sync -> fixed-order totals
        x0 = warp_sum(x0);
        x1 = warp_sum(x1);
        if (lane == 0) {
            red[0][wid] = x0;
            red[1][wid] = x1;
        }
        __syncthreads();
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
        grid.sync();
        if (wid == 0) {
            const double t0 = warp_sum_partials(P + (parity * 2 + 0) * G, G);
            const double t1 = warp_sum_partials(P + (parity * 2 + 1) * G, G);
            if (lane == 0) {
                bc[0] = t0;
                bc[1] = t1;
            }
        }
        __syncthreads();
    };

    // ---- pass 0: stage w on chip, ||w||^2 and <v_0, w>
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
    reduce2(ss, dt, 0);
    const double pre_norm = sqrt(bc[0]);
    double h = bc[1];
    if (blockIdx.x == 0 && tid == 0) a.kb.H[(size_t)j * (m + 1) + 0] = h;

    // ---- passes 1..j: w -= h_{i-1} v_{i-1}; h_i = <v_i, w>
    for (int i = 1; i <= j; ++i) {
        const double2* vp = reinterpret_cast<const double2*>(V + (size_t)(i - 1) * ldv + r0);
        const double2* vi = reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0);
        dt = 0.0;
#pragma unroll 4
        for (int e = tid; e < nv2; e += kMgsThreads) {
            double2 wv = w2[e];
            const double2 pv = __ldg(vp + e);
            const double2 qv = __ldg(vi + e);
            wv.x = fma(-h, pv.x, wv.x);
            wv.y = fma(-h, pv.y, wv.y);
            w2[e] = wv;
            dt = fma(qv.x, wv.x, dt);
            dt = fma(qv.y, wv.y, dt);
        }
        reduce2(0.0, dt, i & 1);
        h = bc[1];
        if (blockIdx.x == 0 && tid == 0) a.kb.H[(size_t)j * (m + 1) + i] = h;
    }

    // ---- final pass: w -= h_j v_j; ||w||
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
    const double hnext = sqrt(bc[0]);
    // breakdown test (gmres.hpp:66-71): ||w|| <= factor * u * ||w_pre||
    const bool breakdown = hnext <= st->breakdown_factor * pre_norm;
    if (!breakdown) {
        const double inv = 1.0 / hnext;  // gmres.hpp:72-73 multiplies by the reciprocal
        double2* vn = reinterpret_cast<double2*>(a.kb.V + (size_t)(j + 1) * ldv + r0);
#pragma unroll 4
        for (int e = tid; e < nv2; e += kMgsThreads) {
            double2 wv = w2[e];
            wv.x *= inv;
            wv.y *= inv;
            vn[e] = wv;
        }
    }

    if (blockIdx.x == 0 && tid == 0) {
        double* Hj = a.kb.H + (size_t)j * (m + 1);
        Hj[j + 1] = hnext;
        // ---- GivensLs::push_column (gmres.cpp:26-52)
        double* Rj = a.kb.R + (size_t)j * (m + 1);
        double* cs = a.kb.cs;
        double* sn = a.kb.sn;
        double* g = a.kb.g;
        for (int i = 0; i <= j + 1; ++i) Rj[i] = Hj[i];
        for (int i = 0; i < j; ++i) {
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
        if (Rj[j] == 0.0) st->rank_deficient = 1;
        const double t = cs[j] * g[j] + sn[j] * g[j + 1];
        g[j + 1] = -sn[j] * g[j] + cs[j] * g[j + 1];
        g[j] = t;
        const double est = fabs(g[j + 1]);
        a.kb.est[j] = est;
        // ---- cycle exits (gmres.cpp:137-146)
        const bool conv = est <= st->thr;
        if (conv) st->converged_est = 1;
        if (breakdown) st->breakdown = 1;
        st->pre_norm = pre_norm;
        st->last_est = est;
        st->j = j + 1;
        st->done = (conv || breakdown || est <= st->attainable || j + 1 >= m) ? 1 : 0;
    }
}

// v_0 = r0 / beta (element-wise division, gmres.cpp:120-122); cycle state.
__global__ void k_cycle_init(KrylovBufs kb, SolveState* st, const double* __restrict__ r, int n) {
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
    }
}

// y = R^-1 g with the zero-rotation convention (gmres.cpp:57-66).
__global__ void k_solve_y(KrylovBufs kb, const SolveState* st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int steps = st->j;
    const int ld = kb.m + 1;
    for (int i = steps - 1; i >= 0; --i) {
        const double rii = kb.R[(size_t)i * ld + i];
        if (rii == 0.0) {
            kb.y[i] = 0.0;
            continue;
        }
        double s = kb.g[i];
        for (int k = i + 1; k < steps; ++k) s -= kb.R[(size_t)k * ld + i] * kb.y[k];
        kb.y[i] = s / rii;
    }
}

}  // namespace

MgsLaunch plan_mgs(int n, int num_sms) {
    MgsLaunch L;
    L.threads = kMgsThreads;
    const int npad = (n + 1) & ~1;
    // enough CTAs to stream at full HBM rate, few enough to keep the barrier cheap
    int grid = num_sms;
    const int min_rows = 4096;
    grid = std::max(1, std::min(grid, (npad + min_rows - 1) / min_rows));
    int slice = (npad + grid - 1) / grid;
    slice = (slice + 1) & ~1;
    L.grid = grid;
    L.slice = slice;
    L.smem = (size_t)slice * sizeof(double);
    L.w_in_smem = L.smem <= kMgsSmemMax;
    if (!L.w_in_smem) L.smem = 0;
    return L;
}

void launch_mgs(const MgsLaunch& L, const KrylovBufs& kb, SolveState* sst, int n, cudaStream_t st,
                int64_t* launches) {
    MgsArgs a{kb, sst, n, L.slice, (n + 1) & ~1};
    void* args[] = {&a};
    if (L.w_in_smem) {
        static bool attr = false;
        if (!attr) {
            HPBJ_CUDA(cudaFuncSetAttribute(k_mgs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kMgsSmemMax));
            attr = true;
        }
        HPBJ_CUDA(cudaLaunchCooperativeKernel((const void*)k_mgs<true>, dim3(L.grid), dim3(L.threads), args,
                                              L.smem, st));
    } else {
        HPBJ_CUDA(cudaLaunchCooperativeKernel((const void*)k_mgs<false>, dim3(L.grid), dim3(L.threads), args,
                                              0, st));
    }
    *launches += 1;
}

void launch_cycle_init(const KrylovBufs& kb, SolveState* sst, const double* r, int n, cudaStream_t st,
                       int64_t* launches) {
    const int grid = std::max(1, std::min((n + 255) / 256, 148 * 8));
    k_cycle_init<<<grid, 256, 0, st>>>(kb, sst, r, n);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_solve_y(const KrylovBufs& kb, SolveState* sst, cudaStream_t st, int64_t* launches) {
    k_solve_y<<<1, 32, 0, st>>>(kb, sst);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
