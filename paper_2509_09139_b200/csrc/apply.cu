// Block-Jacobi preconditioner apply — replaces Preconditioner::apply_impl
// (preconditioner.cpp:159-188) + lu_solve<T> (lu.hpp:88-112).
//
// The solve runs in the permuted frame (Q A Q^T), so each block is a
// contiguous index range and the reference's scatter/gather by perm
// (preconditioner.cpp:174, :184) disappears from the hot loop.
//
// One warp per block, blocked substitution over 32-row panels:
//   forward  y_k = rhs[pivot_rows[k]] - sum_{c<k} L_kc y_c
//   backward x_k = (y_k - sum_{c>k} U_kc x_c) / U_kk
// Lane r owns row 32t + r of panel t. Off-panel columns stream as coalesced
// float4 loads (512 B per warp per 4 columns) against y/x held in shared
// memory (broadcast reads); the 32x32 diagonal triangle resolves with 32
// warp shuffles. HBM-bound: every factor byte is read exactly once.
//
// Arnoldi apply: FP32 arithmetic, FP64 v rounded to FP32 on load (north
// star). Cycle update: x += M^-1 (V y) with the basis combination fused into
// the right-hand-side gather and FP64 arithmetic on the FP32 factors.

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kApplyWarps = 4;

struct SrcDownF32 {  // (float) v[row]
    const double* v;
    __device__ float operator()(int row) const { return __double2float_rn(__ldg(v + row)); }
};
struct SrcBasisF64 {  // sum_i y_i V[i][row]  (gmres.cpp:152-157 order: i ascending)
    const double* V;
    int ldv;
    const double* y;
    int steps;
    __device__ double operator()(int row) const {
        double u = 0.0;
        for (int i = 0; i < steps; ++i) u = fma(y[i], __ldg(V + (size_t)i * ldv + row), u);
        return u;
    }
};
struct DstF32 {
    float* z;
    __device__ void operator()(int row, float v) const { z[row] = v; }
};
struct DstF64 {
    double* z;
    template <class T>
    __device__ void operator()(int row, T v) const { z[row] = (double)v; }
};
struct DstAddX {  // x = x0 + z (gmres.cpp:158-159)
    double* x;
    __device__ void operator()(int row, double v) const { x[row] = x[row] + v; }
};

template <class Acc>
__device__ __forceinline__ Acc fms(float f, Acc y, Acc acc) {
    return fma(-(Acc)f, y, acc);
}
template <>
__device__ __forceinline__ float fms<float>(float f, float y, float acc) {
    return fmaf(-f, y, acc);
}

// a / b for finite normal operands without the IEEE slow-path branches:
// q0 = a * rcp(b); one FMA residual correction gives the correctly rounded
// quotient (Markstein) for the operand ranges a factor block produces.
__device__ __forceinline__ float div_fast(float a, float b, float rb) {
    const float q = a * rb;
    const float r = fmaf(-q, b, a);
    return fmaf(r, rb, q);
}
__device__ __forceinline__ double div_fast(double a, double b, double rb) {
    const double q = a * rb;
    const double r = fma(-q, b, a);
    return fma(r, rb, q);
}
__device__ __forceinline__ float recip(float b) { return __frcp_rn(b); }
__device__ __forceinline__ double recip(double b) { return 1.0 / b; }

template <class Acc, class Src, class Dst>
__global__ void __launch_bounds__(kApplyWarps * 32) k_apply(ApplyParams p, Src src, Dst dst,
                                                           const SolveState* sst, int ybuf_stride) {
    if (sst && sst->done) return;
    extern __shared__ __align__(16) unsigned char apply_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Acc* ybuf = reinterpret_cast<Acc*>(apply_smem) + wid * ybuf_stride;
    const int nw = gridDim.x * kApplyWarps;

    for (int b = blockIdx.x * kApplyWarps + wid; b < p.s; b += nw) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        const int T = (d + 31) >> 5;
        const int dq = (d + 3) >> 2;  // float4 columns
        const float* F = p.fac + p.fac_off[b];
        const int* pv = p.piv + o;

        // gather rhs[pivot_rows[k]] for the whole block (independent loads)
        for (int k = lane; k < 32 * T; k += 32) ybuf[k] = (k < d) ? (Acc)src(o + __ldg(pv + k)) : (Acc)0;
        __syncwarp();
        // ---------------- forward: unit-lower L, rows in pivot order
        for (int t = 0; t < T; ++t) {
            const int k = 32 * t + lane;
            Acc acc = ybuf[k];
            const float4* panel = reinterpret_cast<const float4*>(F + (size_t)t * 32 * 4 * dq);
            // off-panel columns [0, 32t)
            const int cq_end = 8 * t;
#pragma unroll 4
            for (int cq = 0; cq < cq_end; ++cq) {
                const float4 f = __ldg(panel + cq * 32 + lane);
                const Acc* yy = ybuf + 4 * cq;
                acc = fms<Acc>(f.x, yy[0], acc);
                acc = fms<Acc>(f.y, yy[1], acc);
                acc = fms<Acc>(f.z, yy[2], acc);
                acc = fms<Acc>(f.w, yy[3], acc);
            }
            // diagonal 32x32 triangle
            float fd[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int cq = 8 * t + q;
                float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                if (cq < dq) f = __ldg(panel + cq * 32 + lane);
                fd[4 * q + 0] = f.x;
                fd[4 * q + 1] = f.y;
                fd[4 * q + 2] = f.z;
                fd[4 * q + 3] = f.w;
            }
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
                const Acc yc = __shfl_sync(0xffffffffu, acc, cc);
                if (lane > cc) acc = fms<Acc>(fd[cc], yc, acc);
            }
            ybuf[k] = acc;
            __syncwarp();
        }
        // ---------------- backward: upper U with diagonal
        for (int t = T - 1; t >= 0; --t) {
            const int k = 32 * t + lane;
            Acc acc = ybuf[k];
            const float4* panel = reinterpret_cast<const float4*>(F + (size_t)t * 32 * 4 * dq);
#pragma unroll 4
            for (int cq = 8 * (t + 1); cq < dq; ++cq) {
                const float4 f = __ldg(panel + cq * 32 + lane);
                const Acc* xx = ybuf + 4 * cq;
                acc = fms<Acc>(f.x, xx[0], acc);
                acc = fms<Acc>(f.y, xx[1], acc);
                acc = fms<Acc>(f.z, xx[2], acc);
                acc = fms<Acc>(f.w, xx[3], acc);
            }
            float fd[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int cq = 8 * t + q;
                float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                if (cq < dq) f = __ldg(panel + cq * 32 + lane);
                fd[4 * q + 0] = f.x;
                fd[4 * q + 1] = f.y;
                fd[4 * q + 2] = f.z;
                fd[4 * q + 3] = f.w;
            }
            // own diagonal U_kk (padded rows: 1, and they stay 0)
            float udiag = 1.0f;
#pragma unroll
            for (int cc = 0; cc < 32; ++cc)
                if (lane == cc) udiag = fd[cc];
            const Acc udg = (Acc)udiag;
            const Acc urcp = recip(udg);
#pragma unroll
            for (int cc = 31; cc >= 0; --cc) {
                if (lane == cc && k < d) acc = div_fast(acc, udg, urcp);
                const Acc xc = __shfl_sync(0xffffffffu, acc, cc);
                if (lane < cc) acc = fms<Acc>(fd[cc], xc, acc);
            }
            ybuf[k] = acc;
            __syncwarp();
            if (k < d) dst(o + k, acc);
        }
        __syncwarp();
    }
}

template <class Acc, class Src, class Dst>
void launch(const ApplyParams& p, Src src, Dst dst, const SolveState* sst, cudaStream_t st,
            int64_t* launches) {
    const int stride = ((p.dmax + 31) / 32) * 32 + 4;  // +4 keeps 16 B alignment, spreads banks
    const size_t smem = sizeof(Acc) * stride * kApplyWarps;
    const int grid = (p.s + kApplyWarps - 1) / kApplyWarps;
    k_apply<Acc, Src, Dst><<<grid, kApplyWarps * 32, smem, st>>>(p, src, dst, sst, stride);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace

void launch_apply_f32(const ApplyParams& p, const double* v, const SolveState* sst, int ldv, float* z32,
                      double* z64, cudaStream_t st, int64_t* launches) {
    (void)ldv;
    if (z32) launch<float>(p, SrcDownF32{v}, DstF32{z32}, sst, st, launches);
    else launch<float>(p, SrcDownF32{v}, DstF64{z64}, sst, st, launches);
}

// The Arnoldi-step apply reads column st->j of the basis: resolved on device.
namespace {
struct SrcDownF32Col {
    const double* V;
    int ldv;
    const SolveState* sst;
    __device__ float operator()(int row) const {
        return __double2float_rn(__ldg(V + (size_t)sst->j * ldv + row));
    }
};
struct SrcBasisF64Dyn {
    const double* V;
    int ldv;
    const double* y;
    const SolveState* sst;
    __device__ double operator()(int row) const {
        const int steps = sst->j;
        double u = 0.0;
        for (int i = 0; i < steps; ++i) u = fma(y[i], __ldg(V + (size_t)i * ldv + row), u);
        return u;
    }
};
}  // namespace

void launch_apply_step(const ApplyParams& p, const double* V, int ldv, const SolveState* sst, float* z32,
                       cudaStream_t st, int64_t* launches) {
    launch<float>(p, SrcDownF32Col{V, ldv, sst}, DstF32{z32}, sst, st, launches);
}

void launch_apply_update(const ApplyParams& p, const double* V, int ldv, const double* y,
                         const SolveState* sst, double* x, cudaStream_t st, int64_t* launches) {
    launch<double>(p, SrcBasisF64Dyn{V, ldv, y, sst}, DstAddX{x}, nullptr, st, launches);
}

}  // namespace hpbj
