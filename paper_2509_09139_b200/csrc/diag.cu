// Preconditioner diagnostics on the device — replaces
// cond_estimate_block + block_error_bound (preconditioner.cpp:13-88) and the
// block-stats fill of block_jacobi (:127-136).
//
// Per block, one warp:
//  * ||A_b||_1: column sums of |a_ij| over the block's entries of Q A Q^T, in
//    the reference's order (rows ascending; matrix_one_norm,
//    sparse_matrix.cpp:168-176);
//  * ||A_b^-1||_1: exact for d <= 64 (max over the columns of A^-1, one solve
//    per unit vector — inverse_one_norm_dense), otherwise Hager's estimator
//    with at most 8 iterations (inverse_one_norm_hager: x = 1/n, solve,
//    sign vector, transpose solve, stop when max|z_j| <= z^T x);
//  * cond = ||A_b||_1 ||A_b^-1||_1 and the bound (cond*u_high + u_low)*cond
//    with u_low = 2^-24 (FP32 preconditioner), u_high = 2^-53.
// Solves run in FP64 on the FP32 factors in the dense panels the LU wrote
// (the reference uses its FP64 factors: the estimates agree to the factor
// rounding). Row-oriented substitutions with the lanes over the row's columns
// and a warp reduction per row; the solution vectors live in shared memory.
#include <cstdint>

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kDiagWarps = 4;

__device__ __forceinline__ float fac_at(const float* F, int dp4, int k, int c) {
    return F[(size_t)(k >> 5) * 32 * dp4 + (c >> 2) * 128 + (k & 31) * 4 + (c & 3)];
}

// x = A^-1 r with P A = L U (row k of L\U = original row piv[k]): y = L^-1 (P r), x = U^-1 y.
__device__ void lu_solve_warp(const float* F, int dp4, const int* piv, int d, const double* r, double* y,
                              double* x, int lane) {
    for (int k = 0; k < d; ++k) {
        double s = 0.0;
        for (int c = lane; c < k; c += 32) s = fma((double)fac_at(F, dp4, k, c), y[c], s);
        s = warp_sum(s);
        if (lane == 0) y[k] = r[piv[k]] - s;
        __syncwarp();
    }
    for (int k = d - 1; k >= 0; --k) {
        double s = 0.0;
        for (int c = k + 1 + lane; c < d; c += 32) s = fma((double)fac_at(F, dp4, k, c), x[c], s);
        s = warp_sum(s);
        if (lane == 0) x[k] = (y[k] - s) / (double)fac_at(F, dp4, k, k);
        __syncwarp();
    }
}

// x = A^-T r: w = U^-T r, y = L^-T w, x[piv[k]] = y[k] (lu_solve_transpose, lu.cpp:314-339).
__device__ void lu_solve_t_warp(const float* F, int dp4, const int* piv, int d, const double* r, double* w,
                                double* x, int lane) {
    for (int k = 0; k < d; ++k) {  // U^T lower: w_k = (r_k - sum_{c<k} U_ck w_c) / U_kk
        double s = 0.0;
        for (int c = lane; c < k; c += 32) s = fma((double)fac_at(F, dp4, c, k), w[c], s);
        s = warp_sum(s);
        if (lane == 0) w[k] = (r[k] - s) / (double)fac_at(F, dp4, k, k);
        __syncwarp();
    }
    for (int k = d - 1; k >= 0; --k) {  // L^T unit upper: y_k = w_k - sum_{c>k} L_ck y_c (in place)
        double s = 0.0;
        for (int c = k + 1 + lane; c < d; c += 32) s = fma((double)fac_at(F, dp4, c, k), w[c], s);
        s = warp_sum(s);
        if (lane == 0) w[k] -= s;
        __syncwarp();
    }
    for (int k = lane; k < d; k += 32) x[piv[k]] = w[k];
    __syncwarp();
}

__global__ void __launch_bounds__(kDiagWarps * 32) k_block_cond(DiagParams p) {
    extern __shared__ double dsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double* base = dsm + (size_t)wid * 4 * p.dmax;
    double* v0 = base;               // rhs / x
    double* v1 = base + p.dmax;      // y / w
    double* v2 = base + 2 * p.dmax;  // solution
    double* v3 = base + 3 * p.dmax;  // sign vector / column sums
    for (int b = blockIdx.x * kDiagWarps + wid; b < p.s; b += gridDim.x * kDiagWarps) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        const int dp4 = (d + 3) & ~3;  // panel row stride (padded to a quad)
        const float* F = p.fac + p.fac_off[b];
        const int* piv = p.piv + o;
        // ||A_b||_1: column sums in row order
        for (int c = lane; c < d; c += 32) v3[c] = 0.0;
        __syncwarp();
        for (int r = 0; r < d; ++r) {
            const int kb = p.a.rp[o + r], ke = p.a.rp[o + r + 1];
            for (int k = kb + lane; k < ke; k += 32) {
                const int c = p.a.ci[k] - o;
                if (c >= 0 && c < d) v3[c] += fabs(p.a.val[k]);  // one lane per column within a row
            }
            __syncwarp();
        }
        double nm = 0.0;
        for (int c = lane; c < d; c += 32) nm = fmax(nm, v3[c]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) nm = fmax(nm, __shfl_xor_sync(0xffffffffu, nm, off));
        double ninv = 0.0;
        if (d <= 64) {  // inverse_one_norm_dense
            for (int j = 0; j < d; ++j) {
                for (int c = lane; c < d; c += 32) v0[c] = (c == j) ? 1.0 : 0.0;
                __syncwarp();
                lu_solve_warp(F, dp4, piv, d, v0, v1, v2, lane);
                double sm = 0.0;
                for (int c = lane; c < d; c += 32) sm += fabs(v2[c]);
                sm = warp_sum(sm);
                ninv = fmax(ninv, sm);
            }
        } else {  // inverse_one_norm_hager
            for (int c = lane; c < d; c += 32) v0[c] = 1.0 / (double)d;
            __syncwarp();
            for (int it = 0; it < 8; ++it) {
                lu_solve_warp(F, dp4, piv, d, v0, v1, v2, lane);
                double est = 0.0;
                for (int c = lane; c < d; c += 32) est += fabs(v2[c]);
                ninv = warp_sum(est);
                for (int c = lane; c < d; c += 32) v3[c] = v2[c] >= 0.0 ? 1.0 : -1.0;
                __syncwarp();
                lu_solve_t_warp(F, dp4, piv, d, v3, v1, v2, lane);  // z in v2
                // jmax = argmax |z_i| (first on ties), z^T x
                double best = -1.0, ztx = 0.0;
                int jmax = 0;
                for (int c = lane; c < d; c += 32) {
                    const double az = fabs(v2[c]);
                    if (az > best) {
                        best = az;
                        jmax = c;
                    }
                    ztx = fma(v2[c], v0[c], ztx);
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                    const int oj = __shfl_xor_sync(0xffffffffu, jmax, off);
                    if (ob > best || (ob == best && oj < jmax)) {
                        best = ob;
                        jmax = oj;
                    }
                }
                ztx = warp_sum(ztx);
                if (best <= ztx) break;
                for (int c = lane; c < d; c += 32) v0[c] = (c == jmax) ? 1.0 : 0.0;
                __syncwarp();
            }
        }
        if (lane == 0) {
            const double cond = d == 0 ? 1.0 : nm * ninv;
            p.cond[b] = cond;
            p.ebound[b] = (cond * 0x1p-53 + 0x1p-24) * cond;  // block_error_bound(cond, 2^-24, 2^-53)
        }
        __syncwarp();
    }
}

}  // namespace

void launch_block_cond(const DiagParams& p, int num_sms, cudaStream_t st, int64_t* launches) {
    const size_t smem = sizeof(double) * 4 * (size_t)p.dmax * kDiagWarps;
    if (smem > 48 * 1024)
        HPBJ_CUDA(cudaFuncSetAttribute(k_block_cond, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = std::max(1, std::min((p.s + kDiagWarps - 1) / kDiagWarps, num_sms * 8));
    k_block_cond<<<grid, kDiagWarps * 32, smem, st>>>(p);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
