// Device-side shared definitions for libhpbj.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "hpbj_common.hpp"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libhpbj targets sm_100a (B200) only"
#endif

namespace hpbj {

inline const char* src_base(const char* f) {
    const char* b = f;
    for (const char* p = f; *p; ++p)
        if (*p == '/') b = p + 1;
    return b;
}

#define HPBJ_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            ::hpbj::fail(e_ == cudaErrorMemoryAllocation ? HPBJ_ENOMEM : HPBJ_ECUDA,      \
                         std::string(#call) + " [" + ::hpbj::src_base(__FILE__) + ":" +   \
                             std::to_string(__LINE__) + "]: " + cudaGetErrorString(e_));  \
    } while (0)

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Solver control block, resident in device memory for the whole solve. The
// Arnoldi kernels read/write it so no host round-trip happens per iteration;
// the host reads it once per restart cycle.
struct SolveState {
    // configuration (written once per solve)
    int64_t n;
    int32_t m;             // restart length
    int32_t ldv;           // leading dimension of the basis (doubles)
    double thr;            // tol * ||b|| (or tol if absolute)
    double bnorm;
    double breakdown_factor;   // 1e2 * 2^-53 (FP64 basis)
    double floor_roundoff;     // 2^-24 (FP32 preconditioner)
    // per cycle
    double beta;           // ||r0||
    double attainable;     // 10 * floor_roundoff * beta
    int32_t j;             // Arnoldi steps completed in this cycle
    int32_t done;          // cycle finished (converged / breakdown / floor / m)
    int32_t converged_est;
    int32_t breakdown;
    int32_t rank_deficient;
    int32_t pad;
    double pre_norm;       // last ||w|| before orthogonalisation
    double last_est;
    // reductions
    double rnorm;          // true residual norm from the last residual kernel
    double scratch;
    uint32_t ticket;       // last-block-done counter
    uint32_t pad2;
    // restart driver bookkeeping (hybrid_restart_gmres, gmres.cpp:236-258),
    // advanced on the device by k_cycle_end when the solve runs as a graph
    int32_t max_restarts;
    int32_t cycles;
    int32_t total_iterations;
    int32_t hist_len;      // device history rows written (excluding row 0)
    int32_t converged;
    int32_t breakdown_any;
    int32_t rank_any;
    int32_t last_steps;
};

// Generation barrier of one cooperative launch (zero-initialised).
constexpr int kFlagSlots = 4;      // reductions of the pipelined MGS that may be in flight at once (+ reuse distance)
constexpr int kFlagMaxCtas = 160;  // CTAs of its all-gather (one per SM; larger grids use the barrier kernel)
struct GridBarrier {
    unsigned int count;
    unsigned int gen;
    // All-gather of k_mgs_pipe (arnoldi.cu): seq counts its launches (CTA 0
    // bumps it after the last collect); ll[slot][cta] carries that CTA's two
    // partial sums as four 64-bit words (32 payload bits << 32 | epoch): a
    // word is single-copy atomic, so data and flag arrive together and the
    // exchange needs no fence.
    unsigned long long seq;
    alignas(32) unsigned long long ll[kFlagSlots][kFlagMaxCtas][4];
    alignas(32) unsigned long long tot[kFlagSlots][4];  // the totals, from CTA 0, same encoding
};

// Grid-wide deterministic reduction: each CTA deposits a partial; the last
// CTA to arrive sums them in CTA order (fixed, run-to-run reproducible).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum with a fixed order; every thread gets the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* NT/32 */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (wid == 0) {
        t = lane < NT / 32 ? sh[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) sh[0] = t;
    }
    __syncthreads();
    t = sh[0];
    return t;
}

// Sums partials[0..count) in a fixed order (lane-strided then xor tree).
// Lane l's share: s = ((0 + p[l]) + p[l + 32]) + ... . The loads go out in
// batches of eight independent L2 reads (one round trip per 256 partials
// instead of one per 32: with the loop-carried sum the compiler waited on
// each load before issuing the next), summed in the same order.
__device__ __forceinline__ double lane_sum_partials(const double* partials, int count) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int i0 = lane; i0 < count; i0 += 8 * 32) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = i0 + 32 * k < count ? __ldcg(partials + i0 + 32 * k) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (i0 + 32 * k < count) s += v[k];
    }
    return s;
}

__device__ __forceinline__ double warp_sum_partials(const double* partials, int count) {
    return warp_sum(lane_sum_partials(partials, count));
}

}  // namespace hpbj
