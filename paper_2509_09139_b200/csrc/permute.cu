// Q A Q^T on the device: replaces permute_symmetric (sparse_matrix.cpp:113-153).
// B[perm[i], perm[j]] = A[i, j], each permuted row sorted by column, plus a
// position map src[p] (permuted position -> original position) so a new set
// of values with the same pattern (config 4) is re-permuted by one gather.
//
// Integer/index work, HBM-bound: rows are scattered with one thread per row,
// short rows sorted in registers by their owning thread, long rows (hub
// rails, > kShortRow entries) by one CTA each with a shared-memory bitonic
// sort (global-memory bitonic above kSmemSortMax entries).

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// Exclusive scan of one tile; writes tile total to sums[blockIdx.x].
__global__ void __launch_bounds__(kScanThreads) k_scan_tile(const int* __restrict__ in, int* __restrict__ out,
                                                            int n, int* __restrict__ sums) {
    __shared__ int wsum[kScanThreads / 32];
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    int v[kScanItems];
    int t = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        t += v[k];
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int s = wsum[lane];
        int si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += y;
        }
        wsum[lane] = si - s;  // exclusive warp offsets
        if (lane == 31 && sums) sums[blockIdx.x] = si;
    }
    __syncthreads();
    int run = wsum[wid] + incl - t;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

__global__ void k_scan_add(int* __restrict__ out, int n, const int* __restrict__ offs) {
    const int i = blockIdx.x * kScanTile + threadIdx.x;
    const int off = offs[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int idx = i + k * kScanThreads;
        if (idx < n) out[idx] += off;
    }
}

__global__ void k_perm_rowlen(int n, const int* __restrict__ rp, const int* __restrict__ perm,
                              int* __restrict__ newlen) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        newlen[perm[i]] = rp[i + 1] - rp[i];
}

// Each target claimed once: a second claim of a bit is a repeated target.
__global__ void k_perm_check(int n, const int* __restrict__ perm, unsigned* __restrict__ bits, int* __restrict__ bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int p = perm[i];
        const unsigned bit = 1u << (p & 31);
        if (atomicOr(&bits[p >> 5], bit) & bit) *bad = 1;
    }
}

__global__ void k_set_total(int* out, int n, const int* in_last, const int* out_last) {
    out[n] = *out_last + *in_last;
}

// One thread per original row: scatter entries into the permuted row and,
// for short rows, insertion-sort them by new column in place.
__global__ void k_perm_fill(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                            const int* __restrict__ perm, const int* __restrict__ nrp,
                            int* __restrict__ nci, int* __restrict__ src, int short_max) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int b = rp[i], e = rp[i + 1];
        const int d = nrp[perm[i]];
        const int len = e - b;
        if (len <= short_max) {
            int kc[kShortRow], ks[kShortRow];
#pragma unroll 1
            for (int k = 0; k < len; ++k) {
                const int c = perm[ci[b + k]];
                int p = k;
                while (p > 0 && kc[p - 1] > c) {
                    kc[p] = kc[p - 1];
                    ks[p] = ks[p - 1];
                    --p;
                }
                kc[p] = c;
                ks[p] = b + k;
            }
            for (int k = 0; k < len; ++k) {
                nci[d + k] = kc[k];
                src[d + k] = ks[k];
            }
        } else {
            for (int k = 0; k < len; ++k) {
                nci[d + k] = perm[ci[b + k]];
                src[d + k] = b + k;
            }
        }
    }
}

// Bitonic sort of (key, payload) pairs of one long row; keys are distinct.
template <bool SMEM>
__global__ void k_sort_long_rows(const int* __restrict__ rows, const int* __restrict__ nrp,
                                 int* __restrict__ nci, int* __restrict__ src, int* __restrict__ gscratch,
                                 int scratch_stride) {
    extern __shared__ int sh[];
    const int row = rows[blockIdx.x];
    const int b = nrp[row], len = nrp[row + 1] - b;
    int pw = 1;
    while (pw < len) pw <<= 1;
    int* key = SMEM ? sh : gscratch + (size_t)blockIdx.x * 2 * scratch_stride;
    int* val = key + pw;
    for (int k = threadIdx.x; k < pw; k += blockDim.x) {
        key[k] = k < len ? nci[b + k] : INT_MAX;
        val[k] = k < len ? src[b + k] : -1;
    }
    __syncthreads();
    for (int size = 2; size <= pw; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < pw / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const int a = key[lo], c = key[hi];
                if ((a > c) == up) {
                    key[lo] = c;
                    key[hi] = a;
                    const int va = val[lo];
                    val[lo] = val[hi];
                    val[hi] = va;
                }
            }
            __syncthreads();
        }
    }
    for (int k = threadIdx.x; k < len; k += blockDim.x) {
        nci[b + k] = key[k];
        src[b + k] = val[k];
    }
}

__global__ void k_gather_vals(int nnz, const int* __restrict__ src, const double* __restrict__ val,
                              double* __restrict__ nval) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += gridDim.x * blockDim.x)
        nval[p] = __ldg(val + src[p]);
}

__global__ void k_permute_vec(int n, const int* __restrict__ perm, const double* __restrict__ x,
                              double* __restrict__ y, int inverse) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (inverse) y[i] = x[perm[i]];  // y (original) <- x (permuted)
        else y[perm[i]] = x[i];          // y (permuted) <- x (original)
    }
}

}  // namespace

void scan_exclusive(const int* in, int* out, int n, int* tmp, cudaStream_t st, int64_t* launches) {
    // out[0..n]: exclusive prefix sums, out[n] = total. tmp >= 2 * tiles ints.
    const int tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles > kScanTile) fail(HPBJ_EINVAL, "scan: n too large");
    int* sums = tmp;
    int* soffs = tmp + tiles;
    k_scan_tile<<<tiles, kScanThreads, 0, st>>>(in, out, n, sums);
    k_scan_tile<<<1, kScanThreads, 0, st>>>(sums, soffs, tiles, nullptr);
    k_scan_add<<<tiles, kScanThreads, 0, st>>>(out, n, soffs);
    k_set_total<<<1, 1, 0, st>>>(out, n, in + n - 1, out + n - 1);
    *launches += 4;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_permute_pattern(const DevCsr& a, const int* perm, DevCsr& b, int* src, int* tmp,
                            const int* long_rows_new, int n_long, int max_long, cudaStream_t st,
                            int64_t* launches) {
    const int n = a.n;
    const int grid = std::min((n + 255) / 256, 148 * 16);
    k_perm_rowlen<<<grid, 256, 0, st>>>(n, a.rp, perm, tmp);
    scan_exclusive(tmp, b.rp, n, tmp + n, st, launches);
    k_perm_fill<<<grid, 256, 0, st>>>(n, a.rp, a.ci, perm, b.rp, b.ci, src, kShortRow);
    *launches += 2;
    if (n_long > 0) {
        int pw = 1;
        while (pw < max_long) pw <<= 1;
        const size_t smem = sizeof(int) * 2 * pw;
        if (smem <= kSmemSortMax) {
            HPBJ_CUDA(cudaFuncSetAttribute(k_sort_long_rows<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemSortMax));
            k_sort_long_rows<true><<<n_long, 1024, smem, st>>>(long_rows_new, b.rp, b.ci, src, nullptr, 0);
        } else {
            // rare: rows with > kSmemSortMax/8 entries sort in global scratch
            int* scratch = nullptr;
            HPBJ_CUDA(cudaMallocAsync(&scratch, sizeof(int) * 2 * (size_t)pw * n_long, st));
            k_sort_long_rows<false><<<n_long, 1024, 0, st>>>(long_rows_new, b.rp, b.ci, src, scratch, pw);
            HPBJ_CUDA(cudaFreeAsync(scratch, st));
        }
        *launches += 1;
    }
    HPBJ_CUDA(cudaGetLastError());
}

void launch_perm_check(int n, const int* perm, unsigned* bits, int* bad, cudaStream_t st, int64_t* launches) {
    HPBJ_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned) * (((size_t)n + 31) / 32), st));
    HPBJ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    const int grid = std::max(1, std::min((n + 255) / 256, 148 * 16));
    k_perm_check<<<grid, 256, 0, st>>>(n, perm, bits, bad);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_gather_values(const int* src, const double* val, double* nval, int nnz, cudaStream_t st,
                          int64_t* launches) {
    const int grid = std::min((nnz + 255) / 256, 148 * 16);
    k_gather_vals<<<std::max(grid, 1), 256, 0, st>>>(nnz, src, val, nval);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_permute_vec(int n, const int* perm, const double* x, double* y, bool inverse, cudaStream_t st,
                        int64_t* launches) {
    const int grid = std::min((n + 255) / 256, 148 * 16);
    k_permute_vec<<<std::max(grid, 1), 256, 0, st>>>(n, perm, x, y, inverse ? 1 : 0);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
