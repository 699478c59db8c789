// FP64 CSR SpMV — replaces spmv<T> (spmv.hpp:31-47) and residual_vector
// (gmres.cpp:75-81), on the permuted matrix Q A Q^T.
//
// Rows are processed by groups of G lanes (G = 4/8/16/32 by mean row length:
// coalesced, vectorised row access); each lane strides the row and the group
// reduces with G-wide shuffles in a fixed order. Rows longer than
// plan.long_thresh (supply-rail hubs, ~1e4 nnz in config 2) are split across
// a whole CTA by a separate kernel that runs first and parks the row sum in
// ylong[row]; the main kernel then treats the row like any other, so the
// epilogue (plain store, or r = b - A x with a deterministic grid-wide norm)
// stays uniform.

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kSpmvThreads = 256;
constexpr int kLongThreads = 512;

template <class XT>
__device__ __forceinline__ double ldx(const XT* x, int c) {
    return (double)__ldg(x + c);
}

template <class XT>
__global__ void __launch_bounds__(kLongThreads) k_spmv_long(const int* __restrict__ rows, DevCsr a,
                                                            const XT* __restrict__ x,
                                                            double* __restrict__ ylong, const SolveState* sst) {
    if (sst && sst->done) return;
    __shared__ double sh[kLongThreads / 32];
    const int row = rows[blockIdx.x];
    const int b = a.rp[row], e = a.rp[row + 1];
    double s = 0.0;
    for (int k = b + threadIdx.x; k < e; k += kLongThreads) s = fma(a.val[k], ldx(x, a.ci[k]), s);
    s = block_sum<kLongThreads>(s, sh);
    if (threadIdx.x == 0) ylong[row] = s;
}

// MODE 0: y = A x.  MODE 1: y = b - A x, st->rnorm = ||y||_2.
template <int G, class XT, int MODE>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv(DevCsr a, const XT* __restrict__ x,
                                                       double* __restrict__ y, const double* __restrict__ bvec,
                                                       const double* __restrict__ ylong, int long_thresh,
                                                       SolveState* sst, double* __restrict__ partials) {
    if (MODE == 0 && sst && sst->done) return;
    const int gl = threadIdx.x & (G - 1);
    const int group = (blockIdx.x * kSpmvThreads + threadIdx.x) / G;
    const int ngroups = gridDim.x * (kSpmvThreads / G);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    double ss = 0.0;
    for (int row = group; row < a.n; row += ngroups) {
        const int b = __ldg(a.rp + row), e = __ldg(a.rp + row + 1);
        double sum;
        if (e - b > long_thresh) {
            sum = ylong[row];
        } else {
            sum = 0.0;
            for (int k = b + gl; k < e; k += G) sum = fma(__ldg(a.val + k), ldx(x, __ldg(a.ci + k)), sum);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(gmask, sum, o, G);
        }
        if (gl == 0) {
            if (MODE == 0) {
                y[row] = sum;
            } else {
                const double r = bvec[row] - sum;
                y[row] = r;
                ss = fma(r, r, ss);
            }
        }
    }
    if (MODE == 1) {
        __shared__ double sh[kSpmvThreads / 32];
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
    if (plan.n_long > 0) {
        k_spmv_long<XT><<<plan.n_long, kLongThreads, 0, st>>>(plan.long_rows, a, x, plan.ylong,
                                                              MODE == 0 ? sst : nullptr);
        *launches += 1;
    }
    const int G = plan.group;
    const int grid = spmv_grid(a.n, G);
#define HPBJ_SPMV_CASE(GG)                                                                          \
    case GG:                                                                                        \
        k_spmv<GG, XT, MODE><<<grid, kSpmvThreads, 0, st>>>(a, x, y, b, plan.ylong, plan.long_thresh, \
                                                            sst, partials);                         \
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
                      int64_t* launches) {
    run<double, 0>(a, plan, x, y, nullptr, nullptr, nullptr, st, launches);
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
