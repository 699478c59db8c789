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

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void ld_relaxed_v2u64(const unsigned long long* p, unsigned long long& x,
                                                 unsigned long long& y) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed_v2u64(unsigned long long* p, unsigned long long x, unsigned long long y) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}

// Sense-free generation barrier over all CTAs of a cooperative launch, with
// release/acquire atomics instead of full fences (0.5 us cheaper per barrier
// on B200, scripts/micro/barrier.cu): bar.sync orders the CTA's writes before
// thread 0's acq_rel arrival; the last arriver's release of the generation is
// acquired by every spinner, and bar.sync hands it to the rest of the CTA.
// Data published before it must be read after it through L2 (ld.cg /
// __ldcg) or plain loads (the gpu-scope acquire invalidates L1).
__device__ __forceinline__ void grid_barrier(GridBarrier* gb) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_relaxed(&gb->gen);
        if (atom_add_acq_rel(&gb->count, 1u) == gridDim.x - 1) {
            gb->count = 0;  // ordered before the release below
            st_release(&gb->gen, g + 1);
        } else {
            while (ld_acquire(&gb->gen) == g) {
            }
        }
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
