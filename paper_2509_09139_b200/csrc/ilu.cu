// ILU(0) preconditioner on the device — replaces ilu0
// (lu.cpp:227-312), Preconditioner::from_ilu0 (preconditioner.cpp:94-98) and
// its lu_solve<double> apply (lu.hpp:88-112, preconditioner.cpp:168-170).
//
// The factors live in place in a copy of A's values (original ordering, A's
// pattern): row i holds L (columns < i, unit diagonal implied), then U's
// diagonal, then U (columns > i) — exactly the reference's `vals` before it
// splits them into its lower/upper CSR (lu.cpp:273-298).
//
// Factorisation and both triangular solves are sync-free: rows are handed
// out in chunks of consecutive rows by an atomic ticket, in dependency order;
// a warp sweeps its chunk in order (dependencies inside the chunk — the i-1
// chains of ring and mesh orderings — resolve locally), waits on the per-chunk
// progress words of the rows it reads from other chunks (acquire) and
// publishes its own progress after every row (release). Every row depends only
// on rows with earlier tickets, all of which are held by running warps, so
// the scheme cannot deadlock, and no level schedule has to be built. Each
// row's floating-point operation sequence is the reference's (same order,
// separate multiply and subtract — no FMA), so the factors and the applies
// are bit-identical to the FP64 reference.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kIluWarps = 4;
constexpr int kIluMaxSleep = 256;
constexpr int kIluCtasPerSm = 4;  // warps in flight: enough for mesh wavefronts, few enough pollers
constexpr int kIluStage = 8;  // staged out-of-chunk products per row in the backward pass

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i32(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// position of column c in ci[lo, hi) (sorted), or -1
__device__ __forceinline__ int find_col(const int* ci, int lo, int hi, int c) {
    const int end = hi;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int v = __ldg(ci + mid);
        if (v < c) lo = mid + 1;
        else hi = mid;
    }
    return (lo < end && __ldg(ci + lo) == c) ? lo : -1;
}

__global__ void k_ilu_diag(int n, const int* __restrict__ rp, const int* __restrict__ ci, int* __restrict__ dpos,
                           int* __restrict__ first_bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int d = -1;
        for (int k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) d = k;
        dpos[i] = d;
        if (d < 0) atomicMin(first_bad, i);
    }
}

// first row whose factored diagonal is exactly zero (lu.cpp:266-269)
__global__ void k_ilu_zero_diag(int n, const int* __restrict__ dpos, const double* __restrict__ lu,
                                int* __restrict__ first_zero) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (lu[dpos[i]] == 0.0) atomicMin(first_zero, i);
}

// Value + epoch tag in one 16-byte slot {value, tag}. The producer stores the
// value, then publishes the tag with st.release; a consumer ld.acquire's the
// tag and only then reads the value. (A single v2 access is not single-copy
// atomic in the PTX memory model, so the tag alone may not vouch for the
// value without this release/acquire pair.) The epoch comes from a monotone
// ticket, so no reset is needed between applies.
__device__ __forceinline__ void st_tagged(double2* p, double v, double tag) {
    double* q = reinterpret_cast<double*>(p);
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(q), "d"(v) : "memory");
    asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(q + 1), "d"(tag) : "memory");
}
__device__ __forceinline__ double ld_tag_acquire(const double2* p) {
    double t;
    asm volatile("ld.acquire.gpu.global.f64 %0, [%1];" : "=d"(t) : "l"(reinterpret_cast<const double*>(p) + 1)
                 : "memory");
    return t;
}
__device__ __forceinline__ double ld_value_relaxed(const double2* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(reinterpret_cast<const double*>(p))
                 : "memory");
    return v;
}
// Spinning lanes back off exponentially (32 ns .. kIluMaxSleep): thousands of
// waiters polling the same few L2 lines at full rate would queue the very
// stores they wait for behind their loads.
__device__ __forceinline__ double wait_tagged(const double2* p, double tag) {
    unsigned ns = 32;
    while (ld_tag_acquire(p) != tag) {
        __nanosleep(ns);
        ns = min(2 * ns, (unsigned)kIluMaxSleep);
    }
    return ld_value_relaxed(p);
}
__device__ __forceinline__ void wait_flag(const int* f) {
    unsigned ns = 32;
    while (ld_acquire_i32(f) == 0) {
        __nanosleep(ns);
        ns = min(2 * ns, (unsigned)kIluMaxSleep);
    }
}

// Row-wise i-k-j elimination restricted to A's pattern (lu.cpp:243-265), one
// warp per row (rows ticketed in order): the earlier pivot rows of row i are
// eliminated while the latest ones (the i-1 chain) are still in flight.
// Matching row i against pivot row k iterates the shorter of the two tails
// and binary-searches the other (hub rows of 10^4 entries stay cheap); every
// matched entry is updated once per k, in the reference's k order.
// err: min over (i << 32 | k) of the first zero pivot row k met by row i —
// the reference throws at the first one in its sequential order.
__global__ void __launch_bounds__(kIluWarps * 32) k_ilu0_factor(IluParams p, unsigned long long* err) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(p.ticket32, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= p.n) return;
        const int e = __ldg(p.rp + i + 1), dp = __ldg(p.dpos + i);
        bool reported = false;
        for (int q0 = __ldg(p.rp + i); q0 < dp; ++q0) {
            const int k = __ldg(p.ci + q0);
            if (lane == 0) wait_flag(p.flags + k);
            __syncwarp();
            const int dk = __ldg(p.dpos + k), ek = __ldg(p.rp + k + 1);
            const double ukk = __ldcg(p.lu + dk);
            if (ukk == 0.0 && !reported) {
                reported = true;
                if (lane == 0) atomicMin(err, ((unsigned long long)i << 32) | (unsigned)k);
            }
            const double lik = __ddiv_rn(__ldcg(p.lu + q0), ukk);
            __syncwarp();
            if (lane == 0) __stcg(p.lu + q0, lik);
            if (e - (q0 + 1) <= ek - (dk + 1)) {  // row i's tail is shorter: search row k
                for (int r = q0 + 1 + lane; r < e; r += 32) {
                    const int q = find_col(p.ci, dk + 1, ek, __ldg(p.ci + r));
                    if (q >= 0) __stcg(p.lu + r, __dsub_rn(__ldcg(p.lu + r), __dmul_rn(lik, __ldcg(p.lu + q))));
                }
            } else {
                for (int q = dk + 1 + lane; q < ek; q += 32) {
                    const int r = find_col(p.ci, q0 + 1, e, __ldg(p.ci + q));
                    if (r >= 0) __stcg(p.lu + r, __dsub_rn(__ldcg(p.lu + r), __dmul_rn(lik, __ldcg(p.lu + q))));
                }
            }
            __syncwarp();
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();  // the row's values, written by all lanes
            st_release_i32(p.flags + i, 1);
        }
    }
}

// z = U^-1 L^-1 v (lu_solve, lu.hpp:101-111) as one ticketed pass over
// chunks of 32 rows: tickets [0, nch) are the forward chunks ascending,
// [nch, 2 nch) the backward chunks descending. Per chunk, phase A runs one
// lane per row over the row's dependencies in other chunks — in the forward
// pass those are a prefix of the row's subtraction chain (columns < r0), so
// the lane folds them into a partial sum; in the backward pass they are a
// suffix (columns >= r1), so the lane stages their products — and phase B
// (lane 0) runs the in-chunk chain in row order from shared memory. Results
// are published as (value, epoch) pairs; the epoch comes from the monotone
// ticket counter, so nothing is reset between applies (CUDA-graph friendly).
__global__ void __launch_bounds__(kIluWarps * 32)
    k_ilu0_apply(IluParams p, const double* __restrict__ vin, const double* __restrict__ V, int ldv,
                 const SolveState* sst, int early_exit, double* zout, double* xadd) {
    if (early_exit && sst->done) return;
    __shared__ double pre[kIluWarps][32];
    __shared__ double cb[kIluWarps][32];
    __shared__ double stage[kIluWarps][32][kIluStage];
    __shared__ int qa[kIluWarps][32], qb[kIluWarps][32], ns[kIluWarps][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double* src = V ? V + (size_t)sst->j * ldv : vin;
    const unsigned long long stride = 2ull * p.nch + (unsigned long long)gridDim.x * kIluWarps;
    unsigned long long tbase = 0;
    double tag = 0.0;
    bool first = true;
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(p.ticket64, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (first) {  // every warp's first ticket lies in [tbase, tbase + stride) of this launch
            tbase = t - t % stride;
            tag = (double)(t / stride + 1);
            first = false;
        }
        const long long rel = (long long)(t - tbase);
        if (rel >= 2ll * p.nch) return;
        const bool fwd = rel < p.nch;
        const int ch = fwd ? (int)rel : (int)(2ll * p.nch - 1 - rel);
        const int r0 = ch * 32, cnt = min(p.n - r0, 32), r1 = r0 + cnt;
        if (fwd) {
            if (lane < cnt) {  // A: s = v_i - sum_{c < r0} L_ic y_c, in column order
                const int i = r0 + lane, dp = __ldg(p.dpos + i);
                int q = __ldg(p.rp + i);
                double s = src[i];
                for (; q < dp; ++q) {
                    const int c = __ldg(p.ci + q);
                    if (c >= r0) break;
                    s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), wait_tagged(p.ytag + c, tag)));
                }
                pre[wid][lane] = s;
                qa[wid][lane] = q;
                qb[wid][lane] = dp;
            }
            __syncwarp();
            if (lane == 0) {  // B: the in-chunk tail, rows in order
                for (int l = 0; l < cnt; ++l) {
                    double s = pre[wid][l];
                    const int qe = qb[wid][l];
                    for (int q = qa[wid][l]; q < qe; ++q)
                        s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), cb[wid][__ldg(p.ci + q) - r0]));
                    cb[wid][l] = s;
                    st_tagged(p.ytag + r0 + l, s, tag);
                }
            }
            __syncwarp();
        } else {
            if (lane < cnt) {  // A: y_i, and the products of the columns >= r1 (staged)
                const int i = r0 + lane, dp = __ldg(p.dpos + i), e = __ldg(p.rp + i + 1);
                pre[wid][lane] = wait_tagged(p.ytag + i, tag);
                int q = dp + 1;
                while (q < e && __ldg(p.ci + q) < r1) ++q;
                qa[wid][lane] = q;  // in-chunk part: (dp, q)
                int k = 0;
                for (int qq = q; qq < e && k < kIluStage; ++qq, ++k)
                    stage[wid][lane][k] = __dmul_rn(__ldg(p.lu + qq), wait_tagged(p.ztag + __ldg(p.ci + qq), tag));
                ns[wid][lane] = k;
            }
            __syncwarp();
            if (lane == 0) {  // B: rows descending; in-chunk columns first, then the staged ones
                for (int l = cnt - 1; l >= 0; --l) {
                    const int i = r0 + l, dp = __ldg(p.dpos + i), e = __ldg(p.rp + i + 1), qs = qa[wid][l];
                    double s = pre[wid][l];
                    for (int q = dp + 1; q < qs; ++q)
                        s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), cb[wid][__ldg(p.ci + q) - r0]));
                    const int k = ns[wid][l];
                    for (int j = 0; j < k; ++j) s = __dsub_rn(s, stage[wid][l][j]);
                    for (int q = qs + k; q < e; ++q)  // beyond the stage: read directly
                        s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), wait_tagged(p.ztag + __ldg(p.ci + q), tag)));
                    const double zi = __ddiv_rn(s, __ldg(p.lu + dp));
                    cb[wid][l] = zi;
                    st_tagged(p.ztag + i, zi, tag);
                    if (zout) zout[i] = zi;
                    if (xadd) xadd[i] = xadd[i] + zi;
                }
            }
            __syncwarp();
        }
    }
}

// The same substitution swept by one warp over all chunks in order: no
// waiting and no publishing — every dependency was computed earlier by this
// warp (visible across its lanes after __syncwarp). For the deep dependency
// graphs of ring and via orderings (depth ~ n/4 .. n) this beats the ticketed
// pass, whose cross-chunk hand-offs then sit on the critical path; the setup
// times both and keeps the faster (IluParams::seq).
__global__ void __launch_bounds__(32)
    k_ilu0_apply_seq(IluParams p, const double* __restrict__ vin, const double* __restrict__ V, int ldv,
                     const SolveState* sst, int early_exit, double* zout, double* xadd) {
    if (early_exit && sst->done) return;
    __shared__ double pre[32], cb[32];
    __shared__ int qa[32], qb[32];
    const int lane = threadIdx.x;
    const double* src = V ? V + (size_t)sst->j * ldv : vin;
    double* y = reinterpret_cast<double*>(p.ytag);  // plain scratch here: y in the first n, z in the next n
    double* z = y + p.n;
    for (int ch = 0; ch < p.nch; ++ch) {  // forward, chunks ascending
        const int r0 = ch * 32, cnt = min(p.n - r0, 32);
        if (lane < cnt) {
            const int i = r0 + lane, dp = __ldg(p.dpos + i);
            int q = __ldg(p.rp + i);
            double s = src[i];
            for (; q < dp; ++q) {
                const int c = __ldg(p.ci + q);
                if (c >= r0) break;
                s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), y[c]));
            }
            pre[lane] = s;
            qa[lane] = q;
            qb[lane] = dp;
        }
        __syncwarp();
        if (lane == 0) {
            for (int l = 0; l < cnt; ++l) {
                double s = pre[l];
                for (int q = qa[l]; q < qb[l]; ++q) s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), cb[__ldg(p.ci + q) - r0]));
                cb[l] = s;
                y[r0 + l] = s;
            }
        }
        __syncwarp();
    }
    for (int ch = p.nch - 1; ch >= 0; --ch) {  // backward, chunks descending
        const int r0 = ch * 32, cnt = min(p.n - r0, 32), r1 = r0 + cnt;
        if (lane < cnt) {  // the in-chunk columns come first in the chain: only locate them here
            const int i = r0 + lane, dp = __ldg(p.dpos + i), e = __ldg(p.rp + i + 1);
            int q = dp + 1;
            while (q < e && __ldg(p.ci + q) < r1) ++q;
            qa[lane] = q;
            pre[lane] = y[i];
        }
        __syncwarp();
        if (lane == 0) {
            for (int l = cnt - 1; l >= 0; --l) {
                const int i = r0 + l, dp = __ldg(p.dpos + i), e = __ldg(p.rp + i + 1), qs = qa[l];
                double s = pre[l];
                for (int q = dp + 1; q < qs; ++q) s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), cb[__ldg(p.ci + q) - r0]));
                for (int q = qs; q < e; ++q) s = __dsub_rn(s, __dmul_rn(__ldg(p.lu + q), z[__ldg(p.ci + q)]));
                const double zi = __ddiv_rn(s, __ldg(p.lu + dp));
                cb[l] = zi;
                z[i] = zi;
                if (zout) zout[i] = zi;
                if (xadd) xadd[i] = xadd[i] + zi;
            }
        }
        __syncwarp();
    }
}

// u = sum_{i < st->j} y_i V_i (gmres.cpp:152-157, FP64, i ascending); xadd: x += u
__global__ void k_basis_combine(const double* __restrict__ V, int ldv, const double* __restrict__ y,
                                const SolveState* sst, int n, double* __restrict__ u, double* xadd) {
    const int steps = sst->j;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < steps; ++i) s = fma(y[i], __ldg(V + (size_t)i * ldv + r), s);
        if (xadd) xadd[r] = xadd[r] + s;
        else u[r] = s;
    }
}

// z = V[:, st->j] (identity preconditioner step)
__global__ void k_copy_column(const double* __restrict__ V, int ldv, const SolveState* sst, int n,
                              double* __restrict__ z) {
    if (sst->done) return;
    const double* src = V + (size_t)sst->j * ldv;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) z[r] = src[r];
}

int ilu_grid(int n, int num_sms) {
    int per_sm = 0;
    HPBJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilu0_apply, kIluWarps * 32, 0));
    const int nch = (n + 31) / 32;
    return std::max(1, std::min((nch + kIluWarps - 1) / kIluWarps, num_sms * std::min(kIluCtasPerSm, std::max(1, per_sm))));
}

}  // namespace

int launch_ilu0_diag(int n, const int* rp, const int* ci, int* dpos, int* scratch, cudaStream_t st,
                     int64_t* launches) {
    const int big = 0x7fffffff;
    HPBJ_CUDA(cudaMemcpyAsync(scratch, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    k_ilu_diag<<<std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st>>>(n, rp, ci, dpos, scratch);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
    int bad = big;
    HPBJ_CUDA(cudaMemcpyAsync(&bad, scratch, sizeof(int), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaStreamSynchronize(st));
    return bad == big ? -1 : bad;
}

int launch_ilu0_zero_diag(const IluParams& p, int* scratch, cudaStream_t st, int64_t* launches) {
    const int big = 0x7fffffff;
    HPBJ_CUDA(cudaMemcpyAsync(scratch, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    k_ilu_zero_diag<<<std::max(1, std::min((p.n + 255) / 256, 148 * 8)), 256, 0, st>>>(p.n, p.dpos, p.lu, scratch);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
    int bad = big;
    HPBJ_CUDA(cudaMemcpyAsync(&bad, scratch, sizeof(int), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaStreamSynchronize(st));
    return bad == big ? -1 : bad;
}

void launch_ilu0_factor(const IluParams& p, unsigned long long* err, int num_sms, cudaStream_t st,
                        int64_t* launches) {
    HPBJ_CUDA(cudaMemsetAsync(p.flags, 0, sizeof(int) * (size_t)p.n, st));
    HPBJ_CUDA(cudaMemsetAsync(p.ticket32, 0, sizeof(int), st));
    int per_sm = 0;
    HPBJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilu0_factor, kIluWarps * 32, 0));
    const int grid = std::max(1, std::min((p.n + kIluWarps - 1) / kIluWarps, num_sms * std::max(1, per_sm)));
    k_ilu0_factor<<<grid, kIluWarps * 32, 0, st>>>(p, err);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
    // the applies tag their results with epochs from 1 on a fresh ticket counter
    HPBJ_CUDA(cudaMemsetAsync(p.ytag, 0, sizeof(double2) * (size_t)p.n, st));
    HPBJ_CUDA(cudaMemsetAsync(p.ztag, 0, sizeof(double2) * (size_t)p.n, st));
    HPBJ_CUDA(cudaMemsetAsync(p.ticket64, 0, sizeof(unsigned long long), st));
}

void launch_ilu0_apply(const IluParams& p, const double* vin, const double* V, int ldv, const SolveState* sst,
                       double* z, double* xadd, cudaStream_t st, int64_t* launches) {
    if (p.seq) {
        k_ilu0_apply_seq<<<1, 32, 0, st>>>(p, vin, V, ldv, sst, V != nullptr ? 1 : 0, z, xadd);
    } else {
        // the grid must be the same for every launch on this ticket counter (the epoch stride depends on it)
        k_ilu0_apply<<<p.apply_grid, kIluWarps * 32, 0, st>>>(p, vin, V, ldv, sst, V != nullptr ? 1 : 0, z, xadd);
    }
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

int ilu0_apply_grid(int n, int num_sms) { return ilu_grid(n, num_sms); }

void ilu0_choose_apply(IluParams& p, double* vin, double* z, cudaStream_t st, int64_t* launches) {
    HPBJ_CUDA(cudaMemsetAsync(vin, 0, sizeof(double) * (size_t)p.n, st));
    cudaEvent_t e[3];
    for (auto& ev : e) HPBJ_CUDA(cudaEventCreate(&ev));
    HPBJ_CUDA(cudaEventRecord(e[0], st));
    p.seq = 0;
    launch_ilu0_apply(p, vin, nullptr, 0, nullptr, z, nullptr, st, launches);
    HPBJ_CUDA(cudaEventRecord(e[1], st));
    p.seq = 1;
    launch_ilu0_apply(p, vin, nullptr, 0, nullptr, z, nullptr, st, launches);
    HPBJ_CUDA(cudaEventRecord(e[2], st));
    HPBJ_CUDA(cudaEventSynchronize(e[2]));
    float t_par = 0.f, t_seq = 0.f;
    HPBJ_CUDA(cudaEventElapsedTime(&t_par, e[0], e[1]));
    HPBJ_CUDA(cudaEventElapsedTime(&t_seq, e[1], e[2]));
    for (auto& ev : e) cudaEventDestroy(ev);
    p.seq = t_seq < t_par ? 1 : 0;
    if (const char* f = getenv("HPBJ_ILU_APPLY")) p.seq = f[0] == 's' ? 1 : f[0] == 't' ? 0 : p.seq;  // sweep / ticketed
    // the sweep used the tag arrays as plain scratch: restart the epochs
    HPBJ_CUDA(cudaMemsetAsync(p.ytag, 0, sizeof(double2) * (size_t)p.n, st));
    HPBJ_CUDA(cudaMemsetAsync(p.ztag, 0, sizeof(double2) * (size_t)p.n, st));
    HPBJ_CUDA(cudaMemsetAsync(p.ticket64, 0, sizeof(unsigned long long), st));
    if (getenv("HPBJ_DEBUG"))
        fprintf(stderr, "[hpbj] ilu0 apply: ticketed %.3f ms, one-warp sweep %.3f ms -> %s\n", t_par, t_seq,
                p.seq ? "sweep" : "ticketed");
}
int ilu0_chunks(int n) { return (n + 31) / 32; }

void launch_basis_combine(const KrylovBufs& kb, const SolveState* sst, int n, double* u, double* xadd,
                          cudaStream_t st, int64_t* launches) {
    k_basis_combine<<<std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st>>>(kb.V, kb.ldv, kb.y, sst, n,
                                                                                    u, xadd);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_copy_column(const KrylovBufs& kb, const SolveState* sst, int n, double* z, cudaStream_t st,
                        int64_t* launches) {
    k_copy_column<<<std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, st>>>(kb.V, kb.ldv, sst, n, z);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
