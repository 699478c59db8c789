// Micro-benchmark: grid-barrier variants for the persistent Arnoldi kernel
// (148 CTAs x 1024 threads, cooperative launch). nvcc -O3 -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
struct Bar {
    unsigned count, gen, pad[30];
    unsigned group[32 * 32];
    unsigned flags[1024];
};

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// MODE 5: per-CTA arrival flags (no same-address atomics): CTA c stores the
// epoch to flags[c], warp 0 of CTA 0 polls all flags, then releases gen.
template <int MODE>
__device__ __forceinline__ void barrier(Bar* b, unsigned epoch = 0) {
    if (MODE == 5) {
        __syncthreads();
        if (blockIdx.x == 0) {
            if (threadIdx.x < 32) {
                for (int c = 1 + threadIdx.x; c < (int)gridDim.x; c += 32)
                    while (ld_acquire(&b->flags[c]) != epoch) {
                    }
                __syncwarp();
                if (threadIdx.x == 0) st_release(&b->gen, epoch);
            }
        } else if (threadIdx.x == 0) {
            st_release(&b->flags[blockIdx.x], epoch);
            while (ld_acquire(&b->gen) != epoch) {
            }
        }
        __syncthreads();
        return;
    }
    if (MODE == 4) {  // CUTLASS-style: release/acquire atomics, no full fences
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned g = ld_relaxed(&b->gen);
            if (atom_add_acqrel(&b->count, 1u) == gridDim.x - 1) {
                b->count = 0;
                st_release(&b->gen, g + 1);
            } else {
                while (ld_acquire(&b->gen) == g) {
                }
            }
        }
        __syncthreads();
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(&b->gen);
        __threadfence();
        bool last = false;
        if (MODE == 0 || MODE == 2) {
            last = atomicAdd(&b->count, 1u) == gridDim.x - 1;
        } else {
            const int GS = MODE == 1 ? 16 : 8;
            const int grp = blockIdx.x / GS, ng = (gridDim.x + GS - 1) / GS;
            const int gsz = min(GS, (int)gridDim.x - grp * GS);
            if (atomicAdd(&b->group[grp * 32], 1u) == (unsigned)gsz - 1) {
                b->group[grp * 32] = 0;
                __threadfence();
                last = atomicAdd(&b->count, 1u) == (unsigned)ng - 1;
            }
        }
        if (last) {
            b->count = 0;
            __threadfence();
            st_release(&b->gen, g + 1);
        } else {
            while (ld_acquire(&b->gen) == g) {
                if (MODE == 2) __nanosleep(20);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(Bar* b, int iters, unsigned long long* out) {
    const unsigned long long t0 = clock64();
    const unsigned base = ld_relaxed(&b->gen);
    for (int i = 0; i < iters; ++i) barrier<MODE>(b, base + 1 + i);
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

template <int MODE>
void run(Bar* b, unsigned long long* out, int grid) {
    cudaMemset(b, 0, sizeof(Bar));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(1024);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k<MODE>, b, 10, out);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k<MODE>, b, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("mode %d grid %d: %.3f us per barrier (%s)\n", MODE, grid, ms * 1e3 / iters,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    Bar* b;
    unsigned long long* out;
    cudaMalloc(&b, sizeof(Bar));
    cudaMalloc(&out, 8);
    for (int grid : {148, 101, 51}) {
        run<0>(b, out, grid);
        run<1>(b, out, grid);
        run<3>(b, out, grid);
        run<2>(b, out, grid);
        run<4>(b, out, grid);
        run<5>(b, out, grid);
    }
    return 0;
}
