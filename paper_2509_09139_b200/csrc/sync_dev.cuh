// Grid-wide synchronisation and warp reductions shared by the cooperative
// Krylov kernels (arnoldi.cu, fused.cu).
#pragma once

#include "device.cuh"

namespace hpbj {
namespace sync {

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense-free generation barrier over all CTAs of a cooperative launch.
// Data published before it must be read after it through L2 (ld.cg /
// __ldcg): L1 is not coherent across SMs.
__device__ __forceinline__ void grid_barrier(GridBarrier* gb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(&gb->gen);
        __threadfence();
        const unsigned prev = atomicAdd(&gb->count, 1u);
        if (prev == gridDim.x - 1) {
            gb->count = 0;
            __threadfence();
            st_release(&gb->gen, g + 1);
        } else {
            while (ld_acquire(&gb->gen) == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// NV per-lane accumulators -> lane l holds the warp total of slot l % NV
// (butterfly transpose-reduction: NV - 1 shuffles for NV partial dots, then
// log2(32 / NV) to fold the lane groups). Fixed order: deterministic.
template <int NV>
__device__ __forceinline__ double transpose_reduce(double (&v)[NV], int lane) {
#pragma unroll
    for (int off = NV / 2; off >= 1; off >>= 1) {
#pragma unroll
        for (int q = 0; q < off; ++q) {
            const bool hi = (lane & off) != 0;
            const double send = hi ? v[q] : v[q + off];
            const double keep = hi ? v[q + off] : v[q];
            v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    double r = v[0];
#pragma unroll
    for (int off = NV; off < 32; off <<= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
    return r;
}

}  // namespace sync
}  // namespace hpbj
