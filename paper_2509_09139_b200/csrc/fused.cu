// One Arnoldi cycle of hybrid_restart_gmres as a single persistent
// cooperative kernel — run_cycle's step loop (gmres.cpp:124-147) with
// Preconditioner::apply<float> (preconditioner.cpp:159-188), spmv<double>
// (spmv.hpp:31-47), arnoldi_step (gmres.hpp:43-75) and GivensLs::push_column
// (gmres.cpp:26-52) fused, so a step costs three grid barriers and no kernel
// launches.
//
// One CTA of 1024 threads per SM (up to the SM count). CTA c owns the row
// slice [c*slice, (c+1)*slice) of every Krylov vector and keeps its slice of
// w = A M^-1 v_j in shared memory for the whole step. Per step j:
//
//   phase 1  z = M^-1 v_j (FP32, SPK substitution, one warp per block, all
//            warps of the grid but one); v_j is read as w_prev * (1/h_{j,j-1})
//            straight from the previous step's unnormalised w in HBM — the
//            same FP64 product the normalised basis vector holds, so no barrier
//            is spent publishing v_j. Meanwhile warp 0 of CTA 0 rotates the
//            previous step's Hessenberg column (Givens, residual estimate,
//            cycle-exit flags).
//   barrier  (z complete; exit flags visible)
//   phase 2  w = A z for the CTA's rows into shared memory (FP64, G lanes per
//            row as in spmv.cu; the CTA's matrix rows are loaded into shared
//            memory once per cycle)
//   phase 3  compact-WY multi-dot c = V^T w, l = V^T v_j, ||w||^2 (see
//            arnoldi.cu k_icwy), one warp per basis vector
//   barrier  (partials)
//   phase 4  h = (I + L)^-1 c by two Jacobi sweeps (every CTA keeps its own
//            copy of the Gram table in shared memory); w -= V h in MGS order;
//            w slice to HBM; ||w||^2
//   barrier  (partials, w)
//   phase 5  h_{j+1,j} = ||w||, breakdown test, v_{j+1} = w / h for the own slice
//
// Determinism: all grid reductions sum per-CTA partials in CTA order, every
// CTA computes identical totals. The apply, SpMV and Givens arithmetic is the
// same as the unfused kernels (spk.cu, spmv.cu, arnoldi.cu); only the
// Gram-Schmidt partial-sum grouping differs (warp per basis vector).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "kernels.cuh"
#include "spk_dev.cuh"
#include "sync_dev.cuh"

namespace hpbj {

namespace {

using sync::grid_barrier;

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr size_t kSmemMax = 227 * 1024;

// per warp: y/x buffer, descriptors, [row metadata], block cache (header + pivots)
__host__ __device__ inline size_t apply_warp_bytes(int ystride, bool rows) {
    return sizeof(float) * ystride + sizeof(SpkPanel) * (ystride / 32) + (rows ? 128 * (ystride / 32) : 0) + 16 +
           sizeof(int) * ystride;
}

struct SrcScaled {  // (float)(v[row] * scale): v_j = w * (1/h) (gmres.hpp:72-73)
    const double* v;
    double scale;
    __device__ float operator()(int row) const { return __double2float_rn(__ldcg(v + row) * scale); }
    __device__ void prefetch(int, int, int) const {}
};
struct DstZ {
    float* z;
    __device__ void operator()(int row, float v) const { z[row] = v; }
};

struct FusedArgs {
    SpkView pc;
    DevCsr a;
    int group;         // SpMV lanes per row
    int long_thresh;
    int n_long;
    const int* long_rows;
    KrylovBufs kb;
    double* gram;
    SolveState* st;
    GridBarrier* gb;
    float* z32;
    int n;
    int npad;
    int slice;
    int ystride;
    int nnz_cap;               // matrix slice capacity (entries) in shared memory
    unsigned long long* prof;  // optional: CTA 0 phase timers [4], ns
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct GivensSmem {
    double cs[kMaxRestart];
    double sn[kMaxRestart];
    double g[kMaxRestart + 1];
    double R[kMaxRestart + 2];
};

// GivensLs::push_column (gmres.cpp:26-52) for column j with H entries h[0..j]
// and subdiagonal hnext, plus the cycle exits of run_cycle (gmres.cpp:137-146).
// Executed by one warp (lane 0 rotates); writes H, R, cs, sn, g, est, st.
__device__ void givens_step(const FusedArgs& a, GivensSmem& gs, const double* h, int j, double hnext,
                            double pre_norm, bool breakdown, int lane) {
    SolveState* st = a.st;
    const int m = a.kb.m;
    double* Hj = a.kb.H + (size_t)j * (m + 1);
    double* Rj = a.kb.R + (size_t)j * (m + 1);
    for (int i = lane; i <= j; i += 32) gs.R[i] = h[i];
    __syncwarp();
    if (lane == 0) {
        gs.R[j + 1] = hnext;
        Hj[j + 1] = hnext;
        double ri = gs.R[0];
        for (int i = 0; i < j; ++i) {
            const double rn = gs.R[i + 1];
            const double t = gs.cs[i] * ri + gs.sn[i] * rn;
            const double r2 = -gs.sn[i] * ri + gs.cs[i] * rn;
            gs.R[i] = t;
            ri = r2;
        }
        gs.R[j] = ri;
        const double aa = gs.R[j], bb = gs.R[j + 1];
        double c, sg;
        if (bb == 0.0) {
            c = 1.0;
            sg = 0.0;
        } else {
            const double hh = hypot(aa, bb);
            c = aa / hh;
            sg = bb / hh;
        }
        gs.cs[j] = c;
        gs.sn[j] = sg;
        a.kb.cs[j] = c;
        a.kb.sn[j] = sg;
        gs.R[j] = c * aa + sg * bb;
        gs.R[j + 1] = 0.0;
        if (gs.R[j] == 0.0) st->rank_deficient = 1;
        const double gj = gs.g[j], gj1 = gs.g[j + 1];
        gs.g[j + 1] = -sg * gj + c * gj1;
        gs.g[j] = c * gj + sg * gj1;
        a.kb.g[j] = gs.g[j];
        a.kb.g[j + 1] = gs.g[j + 1];
        const double est = fabs(gs.g[j + 1]);
        a.kb.est[j] = est;
        const bool conv = est <= st->thr;
        if (conv) st->converged_est = 1;
        if (breakdown) st->breakdown = 1;
        st->pre_norm = pre_norm;
        st->last_est = est;
        st->j = j + 1;
        st->done = (conv || breakdown || est <= st->attainable || j + 1 >= m) ? 1 : 0;
        __threadfence();
    }
    __syncwarp();
    for (int i = lane; i <= j + 1; i += 32) Rj[i] = gs.R[i];
}

// The apply folds row-sorted off-panel runs (SpkView::rows == 0): the row-quad
// layout pads the fused configs' short rows by ~46%.
__global__ void __launch_bounds__(kThreads, 1) k_arnoldi_cycle(FusedArgs a) {
    constexpr bool ROWS = false;
    SolveState* st = a.st;
    if (*(volatile int*)&st->done) return;  // converged at restart (k_cycle_init)
    extern __shared__ __align__(16) double dsm[];
    __shared__ double acc_sh[2 * kMaxRestart + 4];
    __shared__ double tot[2 * kMaxRestart + 4];
    __shared__ double hsh[kMaxRestart + 1];
    __shared__ double h1[kMaxRestart + 1];
    __shared__ double wred[kWarps];
    __shared__ GivensSmem gs;

    const int m = a.kb.m;
    const int ldv = a.kb.ldv;
    const int G = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int r0 = blockIdx.x * a.slice;
    const int len = max(0, min(a.slice, a.npad - r0));
    const int nv2 = len >> 1;
    double* wsh = dsm;
    double2* w2 = reinterpret_cast<double2*>(dsm);
    double2* vj2 = reinterpret_cast<double2*>(dsm + a.slice);  // v_j slice (normalised)
    double* P = a.kb.partials;
    double* P2 = P + (size_t)(2 * kMaxRestart + 4) * G;
    const double* V = a.kb.V;
    const int ldl = m + 1;
    __shared__ unsigned long long tsh[5];  // phase timers (CTA 0, thread 0)
    const bool timer = a.prof && blockIdx.x == 0 && tid == 0;
    if (timer) {
        for (int k = 0; k < 4; ++k) tsh[k] = 0ull;
        tsh[4] = gtimer();
    }
    auto lap = [&](int k) {
        if (timer) {
            const unsigned long long t = gtimer();
            tsh[k] += t - tsh[4];
            tsh[4] = t;
        }
    };

    // dynamic shared memory: [w slice][v_j slice][Gram (m+1)^2][matrix slice:
    // val, ci, local rp][per-warp apply buffers]
    double* gram = dsm + 2 * a.slice;                         // row i: <v_i, v_k>, k < i
    double* mval = gram + (size_t)ldl * ldl;
    int* mci = reinterpret_cast<int*>(mval + a.nnz_cap);
    int* mrp = mci + a.nnz_cap;                               // slice + 1 local row starts
    float* ybuf;
    SpkPanel* dsh;
    uint16_t* msh;
    spk::BlockCache* bcache;
    {
        unsigned char* base = reinterpret_cast<unsigned char*>(mrp + ((a.slice + 2) & ~1) + 2);
        base = reinterpret_cast<unsigned char*>(((uintptr_t)base + 15) & ~(uintptr_t)15);
        const size_t per = apply_warp_bytes(a.ystride, ROWS);
        ybuf = reinterpret_cast<float*>(base + per * wid);
        dsh = reinterpret_cast<SpkPanel*>(base + per * wid + sizeof(float) * a.ystride);
        msh = reinterpret_cast<uint16_t*>(base + per * wid + sizeof(float) * a.ystride +
                                          sizeof(SpkPanel) * (a.ystride / 32));
        bcache = reinterpret_cast<spk::BlockCache*>(base + per * wid + sizeof(float) * a.ystride +
                                                    sizeof(SpkPanel) * (a.ystride / 32) +
                                                    (ROWS ? 128 * (a.ystride / 32) : 0));
    }
    // the CTA's rows of the (permuted) matrix stay in shared memory for the cycle
    const int nrows = max(0, min(len, a.n - r0));
    {
        const int kb = nrows > 0 ? __ldg(a.a.rp + r0) : 0;
        for (int r = tid; r <= nrows; r += kThreads) mrp[r] = __ldg(a.a.rp + r0 + r) - kb;
        const int ke = nrows > 0 ? __ldg(a.a.rp + r0 + nrows) : 0;
        for (int q = tid; q < ke - kb; q += kThreads) {
            mval[q] = __ldg(a.a.val + kb + q);
            mci[q] = __ldg(a.a.ci + kb + q);
        }
    }
    if (blockIdx.x == 0)
        for (int i = tid; i <= m; i += kThreads) gs.g[i] = (i == 0) ? st->beta : 0.0;

    // warp slots run across the CTAs first (slot = wid * G + cta), so the
    // apply's blocks — and their factor traffic — spread over every SM
    // instead of filling the first CTAs' warps (per-SM bandwidth bound)
    // (plan_fused guarantees G * kWarps - 1 >= the number of blocks: one block per apply warp)
    const int gw = wid * G + blockIdx.x;  // 0: the Givens warp (CTA 0, warp 0)
    if (gw != 0 && gw - 1 < a.pc.s) spk::spk_cache_block<ROWS>(a.pc, gw - 1, dsh, msh, bcache, lane);
    const double bdf = st->breakdown_factor;
    const double* asrc = V;  // v_0 (k_cycle_init)
    double ascale = 1.0;
    double pre_norm = 0.0, hnext = 0.0;
    bool pending = false;
    int j = st->j;
    {
        const double2* v0 = reinterpret_cast<const double2*>(V + (size_t)j * ldv + r0);
        for (int e = tid; e < nv2; e += kThreads) vj2[e] = __ldcg(v0 + e);
    }
    __syncthreads();

    for (;;) {
        // ---- phase 1: z = M^-1 v_j; Givens of step j-1
        if (gw == 0) {
            if (pending) givens_step(a, gs, hsh, j - 1, hnext, pre_norm, false, lane);
        } else {
            const int aw = gw - 1;
            if (aw < a.pc.s)
                spk::spk_solve_block<float, uint16_t, false, ROWS, true>(a.pc, aw, -1, SrcScaled{asrc, ascale},
                                                                        DstZ{a.z32}, ybuf, dsh, lane, nullptr, msh,
                                                                        bcache);
        }
        grid_barrier(a.gb);
        if (pending && *(volatile int*)&st->done) break;  // converged at step j-1
        pending = false;
        lap(0);

        // ---- phase 2: w = A z on the own rows (as spmv.cu k_spmv: G lanes per
        // row, four strides of loads in flight), matrix slice from shared memory
        {
            const int Gl = a.group;
            const int gl = tid & (Gl - 1);
            const unsigned gmask = (Gl == 32) ? 0xffffffffu : (((1u << Gl) - 1u) << (lane & ~(Gl - 1)));
            for (int r = tid / Gl; r < len; r += kThreads / Gl) {
                double sum = 0.0;
                if (r < nrows) {
                    const int b = mrp[r], e = mrp[r + 1];
                    for (int q0 = b + gl; q0 < e; q0 += 4 * Gl) {
                        int c[4];
                        double v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int q = q0 + u * Gl;
                            c[u] = q < e ? mci[q] : 0;
                            v[u] = q < e ? mval[q] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (q0 + u * Gl < e) sum = fma(v[u], (double)__ldcg(a.z32 + c[u]), sum);
                    }
                    for (int o = Gl / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(gmask, sum, o, Gl);
                }
                if (gl == 0) wsh[r] = sum;
            }
        }
        __syncthreads();
        lap(1);

        // ---- phase 3: c_i = <v_i, w>, l_i = <v_i, v_j> (warp per basis
        // vector, w and v_j from shared memory), ||w||^2
        {
            double ss = 0.0;
            for (int e = tid; e < nv2; e += kThreads) {
                const double2 wv = w2[e];
                ss = fma(wv.x, wv.x, ss);
                ss = fma(wv.y, wv.y, ss);
            }
            ss = warp_sum(ss);
            if (lane == 0) wred[wid] = ss;
            for (int i = wid; i <= j; i += kWarps) {
                const double2* vi = reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0);
                double c = 0.0, l = 0.0;
#pragma unroll 8
                for (int e = lane; e < nv2; e += 32) {
                    const double2 vv = __ldcg(vi + e);
                    const double2 wv = w2[e];
                    const double2 jv = vj2[e];
                    c = fma(vv.x, wv.x, c);
                    c = fma(vv.y, wv.y, c);
                    l = fma(vv.x, jv.x, l);
                    l = fma(vv.y, jv.y, l);
                }
                c = warp_sum(c);
                l = warp_sum(l);
                if (lane == 0) {
                    acc_sh[i] = c;
                    acc_sh[(j + 1) + i] = l;
                }
            }
            __syncthreads();
        }
        const int nval = 2 * (j + 1) + 1;
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < kWarps; ++w) s += wred[w];
            acc_sh[2 * (j + 1)] = s;
        }
        __syncthreads();
        for (int t = tid; t < nval; t += kThreads) P[(size_t)t * G + blockIdx.x] = acc_sh[t];
        grid_barrier(a.gb);
        lap(2);

        // ---- phase 4: totals, h = (I + L)^-1 c, w -= V h, ||w||^2
        for (int t0v = wid; t0v < nval; t0v += 4 * kWarps) {
            double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = t0v + u * kWarps;
                if (t < nval)
                    part[u] = lane_sum_partials(P + (size_t)t * G, G);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double tv = warp_sum(part[u]);
                const int t = t0v + u * kWarps;
                if (lane == 0 && t < nval) tot[t] = tv;
            }
        }
        __syncthreads();
        pre_norm = sqrt(tot[2 * (j + 1)]);
        auto sweep = [&](const double* src, double* dst) {
            for (int i = wid; i <= j; i += kWarps) {
                const double* Lrow = (i == j) ? tot + (j + 1) : gram + (size_t)i * ldl;
                double sacc = 0.0;
                for (int k = lane; k < i; k += 32) sacc = fma(Lrow[k], src[k], sacc);
                sacc = warp_sum(sacc);
                if (lane == 0) dst[i] = tot[i] - sacc;
            }
            __syncthreads();
        };
        sweep(tot, h1);
        sweep(h1, hsh);
        for (int k = tid; k < j; k += kThreads) gram[(size_t)j * ldl + k] = tot[(j + 1) + k];  // every CTA's copy
        if (blockIdx.x == 0)
            for (int i = tid; i <= j; i += kThreads) a.kb.H[(size_t)j * (m + 1) + i] = hsh[i];
        double ss2 = 0.0;
        {
            double2* wg = reinterpret_cast<double2*>(a.kb.w + r0);
            for (int e = tid; e < nv2; e += kThreads) {
                double2 wv = w2[e];
                for (int i = 0; i <= j; ++i) {
                    const double2 vv = __ldcg(reinterpret_cast<const double2*>(V + (size_t)i * ldv + r0) + e);
                    const double hi = hsh[i];
                    wv.x = fma(-hi, vv.x, wv.x);
                    wv.y = fma(-hi, vv.y, wv.y);
                }
                w2[e] = wv;
                wg[e] = wv;
                ss2 = fma(wv.x, wv.x, ss2);
                ss2 = fma(wv.y, wv.y, ss2);
            }
        }
        ss2 = warp_sum(ss2);
        if (lane == 0) wred[wid] = ss2;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < kWarps; ++w) s += wred[w];
            P2[blockIdx.x] = s;
        }
        grid_barrier(a.gb);
        lap(3);

        // ---- phase 5: h_{j+1,j}, breakdown (gmres.hpp:66-73), v_{j+1} own slice
        if (wid == 0) {
            const double t = warp_sum_partials(P2, G);
            if (lane == 0) wred[0] = t;
        }
        __syncthreads();
        hnext = sqrt(wred[0]);
        const bool breakdown = hnext <= bdf * pre_norm;
        const double inv = 1.0 / hnext;
        if (!breakdown) {
            double2* vn = reinterpret_cast<double2*>(a.kb.V + (size_t)(j + 1) * ldv + r0);
            for (int e = tid; e < nv2; e += kThreads) {
                double2 wv = w2[e];
                wv.x *= inv;
                wv.y *= inv;
                vn[e] = wv;
                vj2[e] = wv;
            }
        }
        pending = true;
        if (breakdown || j + 1 >= m) {  // cycle ends regardless of the estimate
            if (gw == 0) givens_step(a, gs, hsh, j, hnext, pre_norm, breakdown, lane);
            break;
        }
        asrc = a.kb.w;
        ascale = inv;
        ++j;
        __syncthreads();  // v_{j} slice and hsh stable before the next step
    }
    if (timer)
        for (int k = 0; k < 4; ++k) a.prof[k] += tsh[k];
}


}  // namespace

static int fused_grid(int n, int num_sms) {
    // every SM: the apply phase is latency bound, more warps in flight win
    return std::max(1, std::min(num_sms, ((n + 1) & ~1) / 64));
}

bool fused_possible(int n, int s, int num_sms) {
    return n > 0 && s <= fused_grid(n, num_sms) * kWarps - 1;  // one block per apply warp (the block cache)
}

FusedPlan plan_fused(int n, int s, int dmax, int num_sms, int m, bool has_long, const int* brp, bool rows) {
    FusedPlan F;
    if (m > kMaxRestart || n <= 0 || dmax > kIdx16MaxDim || rows || !brp) return F;
    if (has_long) return F;  // hub rows: the per-kernel path gives them whole CTAs
    if (!fused_possible(n, s, num_sms)) return F;
    const int npad = (n + 1) & ~1;
    const int ystride = ((dmax + 31) / 32) * 32;
    const int grid = fused_grid(n, num_sms);
    int slice = (npad + grid - 1) / grid;
    slice = (slice + 1) & ~1;
    int nnz_cap = 0;  // largest matrix slice
    for (int c = 0; c < grid && c * slice < n; ++c)
        nnz_cap = std::max(nnz_cap, brp[std::min(n, (c + 1) * slice)] - brp[c * slice]);
    nnz_cap = (nnz_cap + 1) & ~1;
    const size_t smem = (size_t)2 * slice * sizeof(double) + (size_t)(m + 1) * (m + 1) * sizeof(double) +
                        (size_t)nnz_cap * (sizeof(double) + sizeof(int)) + (size_t)(((slice + 2) & ~1) + 2) * sizeof(int) +
                        16 + (size_t)kWarps * apply_warp_bytes(ystride, rows);
    const size_t static_smem = sizeof(double) * (2 * (2 * kMaxRestart + 4) + 2 * (kMaxRestart + 1) + kWarps) +
                               sizeof(GivensSmem) + 1024;
    if (smem + static_smem > kSmemMax) return F;
    F.ok = true;
    F.grid = grid;
    F.slice = slice;
    F.ystride = ystride;
    F.nnz_cap = nnz_cap;
    F.smem = smem;
    F.rows = rows;
    return F;
}

void launch_arnoldi_cycle(const FusedPlan& F, const SpkView& pc, const DevCsr& a, const SpmvPlan& plan,
                          const KrylovBufs& kb, double* gram, SolveState* sst, GridBarrier* gb, float* z32,
                          unsigned long long* prof, cudaStream_t st, int64_t* launches) {
    FusedArgs args{pc, a, plan.group, plan.long_thresh, plan.n_long, plan.long_rows, kb, gram, sst, gb, z32,
                   a.n, (a.n + 1) & ~1, F.slice, F.ystride, F.nnz_cap, prof};
    // The cycle kernel's apply runs from L2 (factors, basis and matrix of
    // the fused configs fit): its chain is latency bound, and the per-step
    // bulk L2 prefetches (a win for the HBM-streaming standalone apply)
    // queue behind each other in the SM's TMA unit: off (config 1: apply
    // phase 20.2 -> 16.6 us/step).
    args.pc.pf = 0;
    void (*fn)(FusedArgs) = k_arnoldi_cycle;
    HPBJ_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F.smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(F.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = F.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HPBJ_CUDA(cudaLaunchKernelEx(&cfg, fn, args));
    *launches += 1;
}

}  // namespace hpbj
