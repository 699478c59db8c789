// FP64 CSR SpMV — replaces spmv<T> (spmv.hpp:31-47) and residual_vector
// (gmres.cpp:75-81), on the permuted matrix Q A Q^T.
//
// Rows are processed by groups of G lanes (G = 1..32 by mean row length:
// coalesced, vectorised row access); each lane strides the row and the group
// reduces with G-wide shuffles in a fixed order. Rows longer than
// plan.long_thresh (supply-rail hubs, ~1e4 nnz in config 2) get a whole CTA
// each, appended to the same grid so they run concurrently with the ordinary
// rows. The epilogue is a plain store, or r = b - A x with a deterministic
// grid-wide norm (per-CTA partials summed in CTA order by the last CTA).

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kSpmvThreads = 256;

template <class XT>
__device__ __forceinline__ double ldx(const XT* x, int c) {
    return (double)__ldg(x + c);
}

// MODE 0: y = A x.  MODE 1: y = b - A x, st->rnorm = ||y||_2.
// CTAs [0, n_long) take one hub row each (dispatched first: they are the
// longest), CTAs [n_long, n_long + main_grid) sweep the ordinary rows (G lanes
// per row, hub rows skipped) concurrently.
template <int G, class XT, int MODE>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv(DevCsr a, const XT* __restrict__ x,
                                                       double* __restrict__ y, const double* __restrict__ bvec,
                                                       const int* __restrict__ long_rows, int long_thresh,
                                                       int n_long, SolveState* sst, double* __restrict__ partials) {
    if (MODE == 0 && sst && sst->done) return;
    __shared__ double sh[kSpmvThreads / 32];
    double ss = 0.0;
    if ((int)blockIdx.x < n_long) {
        const int row = long_rows[blockIdx.x];
        const int b = __ldg(a.rp + row), e = __ldg(a.rp + row + 1);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // four chains: loads of four strides in flight
        int k = b + threadIdx.x;
        for (; k + 3 * kSpmvThreads < e; k += 4 * kSpmvThreads) {
            s0 = fma(__ldg(a.val + k), ldx(x, __ldg(a.ci + k)), s0);
            s1 = fma(__ldg(a.val + k + kSpmvThreads), ldx(x, __ldg(a.ci + k + kSpmvThreads)), s1);
            s2 = fma(__ldg(a.val + k + 2 * kSpmvThreads), ldx(x, __ldg(a.ci + k + 2 * kSpmvThreads)), s2);
            s3 = fma(__ldg(a.val + k + 3 * kSpmvThreads), ldx(x, __ldg(a.ci + k + 3 * kSpmvThreads)), s3);
        }
        for (; k < e; k += kSpmvThreads) s0 = fma(__ldg(a.val + k), ldx(x, __ldg(a.ci + k)), s0);
        double s = block_sum<kSpmvThreads>((s0 + s1) + (s2 + s3), sh);
        if (threadIdx.x == 0) {
            if (MODE == 0) {
                y[row] = s;
            } else {
                const double r = bvec[row] - s;
                y[row] = r;
                ss = r * r;
            }
        }
    } else {
        const int gl = threadIdx.x & (G - 1);
        const int group = ((blockIdx.x - n_long) * kSpmvThreads + threadIdx.x) / G;
        const int ngroups = (gridDim.x - n_long) * (kSpmvThreads / G);
        const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
        auto finish = [&](int row, double sum) {
            if (MODE == 0) {
                y[row] = sum;
            } else {
                const double r = bvec[row] - sum;
                y[row] = r;
                ss = fma(r, r, ss);
            }
        };
        {
            for (int row = group; row < a.n; row += ngroups) {
                const int b = __ldg(a.rp + row), e = __ldg(a.rp + row + 1);
                if (e - b > long_thresh) continue;  // uniform within the group
                double sum = 0.0;
                // four strides per round: their index/value loads, then their x
                // gathers, are in flight together (same summation order as a plain loop)
                for (int k0 = b + gl; k0 < e; k0 += 4 * G) {
                    int c[4];
                    double v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int k = k0 + u * G;
                        c[u] = k < e ? __ldg(a.ci + k) : 0;
                        v[u] = k < e ? __ldg(a.val + k) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (k0 + u * G < e) sum = fma(v[u], ldx(x, c[u]), sum);
                }
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(gmask, sum, o, G);
                if (gl == 0) finish(row, sum);
            }
        }
    }
    if (MODE == 1) {
        __shared__ bool last;
        ss = block_sum<kSpmvThreads>(ss, sh);
        if (threadIdx.x == 0) {
            partials[blockIdx.x] = ss;
            __threadfence();
            const unsigned t = atomicAdd(&sst->ticket, 1u);
            last = (t == gridDim.x - 1);
        }
        __syncthreads();
        if (last && threadIdx.x < 32) {
            __threadfence();
            const double tot = warp_sum_partials(partials, gridDim.x);
            if (threadIdx.x == 0) {
                sst->rnorm = sqrt(tot);
                sst->ticket = 0;
            }
        }
    }
}

__global__ void __launch_bounds__(kSpmvThreads) k_norm(const double* __restrict__ x, int n, SolveState* sst,
                                                       double* __restrict__ partials) {
    __shared__ double sh[kSpmvThreads / 32];
    __shared__ bool last;
    double ss = 0.0;
    for (int i = blockIdx.x * kSpmvThreads + threadIdx.x; i < n; i += gridDim.x * kSpmvThreads) {
        const double v = x[i];
        ss = fma(v, v, ss);
    }
    ss = block_sum<kSpmvThreads>(ss, sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = ss;
        __threadfence();
        const unsigned t = atomicAdd(&sst->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {
        __threadfence();
        const double tot = warp_sum_partials(partials, gridDim.x);
        if (threadIdx.x == 0) {
            sst->scratch = sqrt(tot);
            sst->ticket = 0;
        }
    }
}

constexpr int kMaxRedBlocks = 148 * 8;

int spmv_grid(int n, int G) {
    const int rows_per_cta = kSpmvThreads / G;
    return std::max(1, std::min((n + rows_per_cta - 1) / rows_per_cta, kMaxRedBlocks));
}

template <class XT, int MODE>
void run(const DevCsr& a, const SpmvPlan& plan, const XT* x, double* y, const double* b, SolveState* sst,
         double* partials, cudaStream_t st, int64_t* launches) {
    const int G = plan.group;
    // y = A x: one CTA per 256 / G rows, no grid stride — the hardware CTA
    // scheduler backfills the SMs the hub-row CTAs and slow CTAs hold (a
    // one-wave grid-stride launch waited on its last CTAs: config 2
    // 42.0 -> 38.2 us, config 3 79.0 -> 76.2 us). The residual keeps the
    // capped grid (one reduction partial per CTA).
    const int main_grid = MODE == 0 ? std::max(1, (a.n + kSpmvThreads / G - 1) / (kSpmvThreads / G))
                                    : spmv_grid(a.n, G);
    const int grid = main_grid + plan.n_long;
#define HPBJ_SPMV_CASE(GG)                                                                              \
    case GG:                                                                                            \
        k_spmv<GG, XT, MODE><<<grid, kSpmvThreads, 0, st>>>(a, x, y, b, plan.long_rows, plan.long_thresh, \
                                                            plan.n_long, sst, partials);                \
        break;
    switch (G) {
        HPBJ_SPMV_CASE(1)
        HPBJ_SPMV_CASE(2)
        HPBJ_SPMV_CASE(4)
        HPBJ_SPMV_CASE(8)
        HPBJ_SPMV_CASE(16)
        HPBJ_SPMV_CASE(32)
        default:
            fail(HPBJ_EINVAL, "spmv: bad group size");
    }
#undef HPBJ_SPMV_CASE
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace

void launch_spmv_f32x(const DevCsr& a, const SpmvPlan& plan, const float* x, double* y, const SolveState* sst,
                      cudaStream_t st, int64_t* launches) {
    run<float, 0>(a, plan, x, y, nullptr, const_cast<SolveState*>(sst), nullptr, st, launches);
}

void launch_spmv_f64x(const DevCsr& a, const SpmvPlan& plan, const double* x, double* y, cudaStream_t st,
                      int64_t* launches, const SolveState* sst) {
    run<double, 0>(a, plan, x, y, nullptr, const_cast<SolveState*>(sst), nullptr, st, launches);
}

void launch_residual(const DevCsr& a, const SpmvPlan& plan, const double* x, const double* b, double* r,
                     SolveState* sst, double* partials, cudaStream_t st, int64_t* launches) {
    run<double, 1>(a, plan, x, r, b, sst, partials, st, launches);
}

void launch_norm(const double* x, int n, SolveState* sst, double* partials, cudaStream_t st,
                 int64_t* launches) {
    const int grid = std::max(1, std::min((n + kSpmvThreads - 1) / kSpmvThreads, kMaxRedBlocks));
    k_norm<<<grid, kSpmvThreads, 0, st>>>(x, n, sst, partials);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
