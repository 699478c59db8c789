// Sparse-panel ("SPK") storage of the block factors and the block-Jacobi
// apply on it — replaces Preconditioner::apply_impl (preconditioner.cpp:
// 159-188) + lu_solve<T> (lu.hpp:88-112).
//
// The batched LU (block_lu.cu) leaves F = L\U of every block in dense 32-row
// panels. Fill-in is sparse (5-22% of d^2 on the BASELINE configs), so for
// the hot apply each panel is repacked (once per factorisation):
//   * off-panel entries of the panel's 32 rows — the L part (columns left of
//     the panel) and the U part (columns right of it) — as a row-sorted
//     coordinate list: FP32 value, uint16 block-local column, uint8 panel row;
//   * the 32x32 diagonal tile dense, in a lane-quad layout so each lane
//     fetches its row segment as coalesced float4 loads (the forward pass
//     reads only the strictly-lower quads, the backward pass the upper ones).
// Per block one warp runs the blocked substitution: off-panel products are
// streamed 32 entries per warp step (coalesced) and folded per row with a
// deterministic segmented warp scan; the in-panel triangle resolves through
// 32 register shuffles (forward: unit-lower L; backward: U with diagonal).
// Stored bytes are what HBM streams: ~6 B per factor nonzero + 4 B per row
// of masks, instead of 4 B per dense entry.

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kMaxPanels = 9;  // pivots of up to 288 rows gathered with full ILP

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x - v;
}

// Dense panel element (k, c) of a block (see kernels.cuh panel layout).
__device__ __forceinline__ float dense_at(const float* F, int dq, int k, int c) {
    const int t = k >> 5;
    return F[(size_t)t * 32 * 4 * dq + (c >> 2) * 128 + (k & 31) * 4 + (c & 3)];
}

// Pass 1 (count) / pass 2 (pack); warp per panel.
template <bool PACK>
__global__ void k_spk_build(SpkBuild p) {
    extern __shared__ double inv_smem[];
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int P = gw; P < p.num_panels; P += nw) {
        const int b = p.panel_block[P];
        const int t = P - p.pstart[b];
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        const int dq = (d + 3) >> 2;
        const float* F = p.dense + p.fac_off[b];
        const int k = 32 * t + lane;
        const int c0 = 32 * t, c1 = min(d, 32 * t + 32);
        int nl = 0, nu = 0;
        unsigned mask = 0u;
        if (k < d) {
            for (int c = 0; c < c0; ++c) nl += dense_at(F, dq, k, c) != 0.0f;
            for (int c = c1; c < d; ++c) nu += dense_at(F, dq, k, c) != 0.0f;
            for (int c = c0; c < c1; ++c)
                if (dense_at(F, dq, k, c) != 0.0f || c == k) mask |= 1u << (c - c0);
        } else {
            mask = 1u << lane;  // padded row: unit diagonal
        }
        (void)mask;
        if (!PACK) {
            int tl = nl, tu = nu;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                tl += __shfl_xor_sync(0xffffffffu, tl, off);
                tu += __shfl_xor_sync(0xffffffffu, tu, off);
            }
            if (lane == 0) p.ent_count[P] = tl + tu;
            continue;
        }
        const int tl_tot = __shfl_sync(0xffffffffu, warp_excl_scan(nl, lane) + nl, 31);
        const int base = p.ent_off[P];
        const int ol = base + warp_excl_scan(nl, lane);
        const int ou = base + tl_tot + warp_excl_scan(nu, lane);
        int tu = nu;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) tu += __shfl_xor_sync(0xffffffffu, tu, off);
        if (lane == 0) p.desc[P] = SpkPanel{base, tl_tot, tu, 0};
        // Inverse of the 32x32 diagonal triangle, in FP64 from the FP32
        // factors: Linv (unit lower, strictly-lower part stored) and Uinv
        // (upper incl. diagonal) packed like L\U, written in a lane-quad
        // layout [q][lane][4] so each lane fetches its row as float4 loads.
        {
            double* Tt = inv_smem + (size_t)(threadIdx.x >> 5) * (2 * 32 * 33);
            double* X = Tt + 32 * 33;
            for (int c = 0; c < 32; ++c) {
                const int cc = c0 + c;
                double v;
                if (k < d && cc < c1) v = (double)dense_at(F, dq, k, cc);
                else v = (c == lane) ? 1.0 : 0.0;  // padded rows/columns: identity
                Tt[lane * 33 + c] = v;
            }
            __syncwarp();
            // lane = column c of the inverses
            const int c = lane;
            for (int i = 0; i < 32; ++i) {  // L x = e_c, unit lower
                double sum = (i == c) ? 1.0 : 0.0;
                for (int j = 0; j < i; ++j) sum -= Tt[i * 33 + j] * X[j * 33 + c];
                X[i * 33 + c] = (i < c) ? 0.0 : sum;
            }
            __syncwarp();
            float linv[32];
            for (int j = 0; j < 32; ++j) linv[j] = (float)X[lane * 33 + j];  // row `lane` of Linv
            __syncwarp();
            for (int i = 31; i >= 0; --i) {  // U x = e_c, upper with diagonal
                double sum = (i == c) ? 1.0 : 0.0;
                for (int j = i + 1; j < 32; ++j) sum -= Tt[i * 33 + j] * X[j * 33 + c];
                X[i * 33 + c] = (i > c) ? 0.0 : sum / Tt[i * 33 + i];
            }
            __syncwarp();
            float* tile = p.dtile + (size_t)P * 1024;
            for (int q = 0; q < 8; ++q) {
                float4 v4;
                float* w4 = &v4.x;
                for (int u = 0; u < 4; ++u) {
                    const int j = 4 * q + u;
                    w4[u] = (j < lane) ? linv[j] : (float)X[lane * 33 + j];
                }
                reinterpret_cast<float4*>(tile)[q * 32 + lane] = v4;
            }
            __syncwarp();
        }
        if (k < d) {
            int q = ol;
            for (int c = 0; c < c0; ++c) {
                const float v = dense_at(F, dq, k, c);
                if (v != 0.0f) {
                    p.eval[q] = v;
                    p.ecol[q] = (uint16_t)c;
                    p.erow[q] = (uint8_t)lane;
                    ++q;
                }
            }
            q = ou;
            for (int c = c1; c < d; ++c) {
                const float v = dense_at(F, dq, k, c);
                if (v != 0.0f) {
                    p.eval[q] = v;
                    p.ecol[q] = (uint16_t)c;
                    p.erow[q] = (uint8_t)lane;
                    ++q;
                }
            }
        }
    }
}

__global__ void k_panel_owner(const int* __restrict__ pstart, int s, int* __restrict__ panel_block) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < s; b += gridDim.x * blockDim.x)
        for (int P = pstart[b]; P < pstart[b + 1]; ++P) panel_block[P] = b;
}

// ----------------------------------------------------------------------------
struct SrcDown {  // (float) V[:, st->j][row]  (Arnoldi step)
    const double* V;
    int ldv;
    const SolveState* sst;
    __device__ float operator()(int row) const { return __double2float_rn(__ldg(V + (size_t)sst->j * ldv + row)); }
};
struct SrcVec {  // (float) v[row]
    const double* v;
    __device__ float operator()(int row) const { return __double2float_rn(__ldg(v + row)); }
};
struct SrcBasis {  // sum_i y_i V[i][row], i ascending (gmres.cpp:152-157), FP64
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
// a / b without IEEE slow-path branches (Markstein-corrected reciprocal)
__device__ __forceinline__ float div_fast(float a, float b, float rb) {
    const float q = a * rb;
    return fmaf(fmaf(-q, b, a), rb, q);
}
__device__ __forceinline__ double div_fast(double a, double b, double rb) {
    const double q = a * rb;
    return fma(fma(-q, b, a), rb, q);
}
__device__ __forceinline__ float recip(float b) { return __frcp_rn(b); }
__device__ __forceinline__ double recip(double b) { return 1.0 / b; }

// Fold entries [e0, e0 + cnt) of a row-sorted coordinate list into
// acc[row] -= sum val * x[col]: 32 entries per step, segmented warp scan by
// row, the last lane of every row segment applies the segment sum. Loads of
// up to four steps are issued together (memory-level parallelism).
template <class Acc>
__device__ __forceinline__ void fold_entries(const float* __restrict__ eval, const uint16_t* __restrict__ ecol,
                                             const uint8_t* __restrict__ erow, int e0, int cnt,
                                             const Acc* xs, Acc* acc, int lane) {
    constexpr int U = 4;
    for (int base = 0; base < cnt; base += 32 * U) {
        float v[U];
        int c[U], rr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int idx = base + 32 * u + lane;
            const bool valid = idx < cnt;
            const int e = valid ? e0 + idx : e0;
            v[u] = valid ? __ldg(eval + e) : 0.0f;
            c[u] = valid ? (int)__ldg(ecol + e) : 0;
            rr[u] = valid ? (int)__ldg(erow + e) : 64 + lane;  // invalid: unique, never applied
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + 32 * u >= cnt) break;
            Acc pr = (Acc)v[u] * xs[c[u]];
            const int r = rr[u];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const Acc q = __shfl_up_sync(0xffffffffu, pr, off);
                const int rq = __shfl_up_sync(0xffffffffu, r, off);
                if (lane >= off && rq == r) pr += q;
            }
            const int rn = __shfl_down_sync(0xffffffffu, r, 1);
            if (r < 32 && (lane == 31 || rn != r)) acc[r] -= pr;
            __syncwarp();
        }
    }
}

// L2 bulk prefetch of [p, p + bytes) (TMA engine; no registers, no smem).
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
    const uintptr_t a = (uintptr_t)p & ~(uintptr_t)15;
    const uintptr_t e = ((uintptr_t)p + bytes + 15) & ~(uintptr_t)15;
    if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

// Next block's head: descriptors, pivots and its first panel's data.
__device__ __forceinline__ void prefetch_block_head(const SpkView& p, int b) {
    const int P0 = p.pstart[b], P1 = p.pstart[b + 1];
    prefetch_l2(p.desc + P0, sizeof(SpkPanel) * (P1 - P0));
    const int o = p.bstart[b], d = p.bstart[b + 1] - o;
    prefetch_l2(p.piv + o, sizeof(int) * d);
    const int e0 = p.ent_off[P0], e1 = p.ent_off[P0 + 1];
    prefetch_l2(p.eval + e0, sizeof(float) * (e1 - e0));
    prefetch_l2(p.ecol + e0, sizeof(uint16_t) * (e1 - e0));
    prefetch_l2(p.erow + e0, (size_t)(e1 - e0));
    prefetch_l2(p.dtile + (size_t)P0 * 1024, sizeof(float) * 1024);
}

// One substitution step's data: entries [e0, e0 + cnt) and panel P's tile.
__device__ __forceinline__ void prefetch_step(const SpkView& p, int P, int e0, int cnt) {
    prefetch_l2(p.eval + e0, sizeof(float) * cnt);
    prefetch_l2(p.ecol + e0, sizeof(uint16_t) * cnt);
    prefetch_l2(p.erow + e0, (size_t)cnt);
    prefetch_l2(p.dtile + (size_t)P * 1024, sizeof(float) * 1024);
}


template <class Acc, class Src, class Dst>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_apply_spk(SpkView p, Src src, Dst dst,
                                                                 const SolveState* sst, int ystride) {
    if (sst && sst->done) return;
    extern __shared__ __align__(16) unsigned char spk_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int tmax = ystride / 32;
    // per warp: y/x buffer (Acc[ystride]), panel descriptors, row masks
    unsigned char* wbase = spk_smem + (size_t)wid * (sizeof(Acc) * ystride + sizeof(SpkPanel) * tmax);
    Acc* ybuf = reinterpret_cast<Acc*>(wbase);
    SpkPanel* dsh = reinterpret_cast<SpkPanel*>(wbase + sizeof(Acc) * ystride);
    const int nw = gridDim.x * kWarpsPerCta;
    const int b_first = blockIdx.x * kWarpsPerCta + wid;
    if (lane == 0 && b_first < p.s) prefetch_block_head(p, b_first);
    for (int b = b_first; b < p.s; b += nw) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        const int T = (d + 31) >> 5;
        const int P0 = p.pstart[b];
        if (lane < T) dsh[lane] = p.desc[P0 + lane];
        __syncwarp();
        // rhs[pivot_rows[k]] for the whole block: all pivot loads first, then
        // all gathers (two latency rounds, not 2T)
        {
            int pv[kMaxPanels];
#pragma unroll
            for (int t = 0; t < kMaxPanels; ++t) {
                const int k = 32 * t + lane;
                pv[t] = (t < T && k < d) ? __ldg(p.piv + o + k) : -1;
            }
#pragma unroll
            for (int t = 0; t < kMaxPanels; ++t)
                if (t < T) ybuf[32 * t + lane] = pv[t] >= 0 ? (Acc)src(o + pv[t]) : (Acc)0;
            for (int t = kMaxPanels; t < T; ++t) {
                const int k = 32 * t + lane;
                ybuf[k] = (k < d) ? (Acc)src(o + __ldg(p.piv + o + k)) : (Acc)0;
            }
        }
        __syncwarp();
        // ---- forward: y_k = rhs_k - sum_{c<k} L_kc y_c
        for (int t = 0; t < T; ++t) {
            const SpkPanel ds = dsh[t];
            if (lane == 0) {  // next step's data into L2 while this one computes
                if (t + 1 < T) prefetch_step(p, P0 + t + 1, dsh[t + 1].off, dsh[t + 1].nl);
                else prefetch_step(p, P0 + t, ds.off + ds.nl, ds.nu);
            }
            fold_entries<Acc>(p.eval, p.ecol, p.erow, ds.off, ds.nl, ybuf, ybuf + 32 * t, lane);
            // y_t = Linv_tt r_t: row `lane` of the strictly-lower inverse, r from smem
            {
                const float4* tile = reinterpret_cast<const float4*>(p.dtile + (size_t)(P0 + t) * 1024);
                float4 f4[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    f4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (4 * q < lane) f4[q] = __ldg(tile + q * 32 + lane);
                }
                const Acc* r = ybuf + 32 * t;
                Acc a0 = r[lane], a1 = (Acc)0, a2 = (Acc)0, a3 = (Acc)0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float* f = &f4[q].x;
                    // entries on/right of the diagonal belong to Uinv: masked out
                    a0 = fma((Acc)((4 * q + 0 < lane) ? f[0] : 0.f), r[4 * q + 0], a0);
                    a1 = fma((Acc)((4 * q + 1 < lane) ? f[1] : 0.f), r[4 * q + 1], a1);
                    a2 = fma((Acc)((4 * q + 2 < lane) ? f[2] : 0.f), r[4 * q + 2], a2);
                    a3 = fma((Acc)((4 * q + 3 < lane) ? f[3] : 0.f), r[4 * q + 3], a3);
                }
                const Acc yv = (a0 + a1) + (a2 + a3);
                __syncwarp();
                ybuf[32 * t + lane] = yv;
                __syncwarp();
            }
        }
        // ---- backward: x_k = (y_k - sum_{c>k} U_kc x_c) / U_kk
        for (int t = T - 1; t >= 0; --t) {
            const SpkPanel ds = dsh[t];
            if (lane == 0) {
                if (t > 0) prefetch_step(p, P0 + t - 1, dsh[t - 1].off + dsh[t - 1].nl, dsh[t - 1].nu);
                else if (b + nw < p.s) prefetch_block_head(p, b + nw);
            }
            fold_entries<Acc>(p.eval, p.ecol, p.erow, ds.off + ds.nl, ds.nu, ybuf, ybuf + 32 * t, lane);
            // x_t = Uinv_tt y'_t: row `lane` of the upper inverse (incl. diagonal)
            const int k = 32 * t + lane;
            {
                const float4* tile = reinterpret_cast<const float4*>(p.dtile + (size_t)(P0 + t) * 1024);
                float4 f4[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    f4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (4 * q + 3 >= lane) f4[q] = __ldg(tile + q * 32 + lane);
                }
                const Acc* r = ybuf + 32 * t;
                Acc a0 = (Acc)0, a1 = (Acc)0, a2 = (Acc)0, a3 = (Acc)0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float* f = &f4[q].x;
                    // entries left of the diagonal are zero in the upper inverse rows
                    a0 = fma((Acc)((4 * q + 0 >= lane) ? f[0] : 0.f), r[4 * q + 0], a0);
                    a1 = fma((Acc)((4 * q + 1 >= lane) ? f[1] : 0.f), r[4 * q + 1], a1);
                    a2 = fma((Acc)((4 * q + 2 >= lane) ? f[2] : 0.f), r[4 * q + 2], a2);
                    a3 = fma((Acc)((4 * q + 3 >= lane) ? f[3] : 0.f), r[4 * q + 3], a3);
                }
                const Acc xv = (a0 + a1) + (a2 + a3);
                __syncwarp();
                ybuf[k] = xv;
                __syncwarp();
                if (k < d) dst(o + k, xv);
            }
        }
        __syncwarp();
    }
}

template <class Acc, class Src, class Dst>
void launch(const SpkView& v, Src src, Dst dst, const SolveState* sst, cudaStream_t st, int64_t* launches) {
    const int ystride = ((v.dmax + 31) / 32) * 32;
    const size_t smem = (sizeof(Acc) * ystride + sizeof(SpkPanel) * (ystride / 32)) * kWarpsPerCta;
    const int grid = (v.s + kWarpsPerCta - 1) / kWarpsPerCta;
    k_apply_spk<Acc, Src, Dst><<<grid, kWarpsPerCta * 32, smem, st>>>(v, src, dst, sst, ystride);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace

void launch_spk_count(const SpkBuild& p, cudaStream_t st, int64_t* launches) {
    k_panel_owner<<<std::max(1, std::min((p.s + 255) / 256, 1184)), 256, 0, st>>>(p.pstart, p.s, p.panel_block);
    const int grid = std::max(1, std::min((p.num_panels * 32 + 255) / 256, 148 * 16));
    k_spk_build<false><<<grid, 256, 0, st>>>(p);
    *launches += 2;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_spk_pack(const SpkBuild& p, cudaStream_t st, int64_t* launches) {
    const int grid = std::max(1, std::min((p.num_panels * 32 + 127) / 128, 148 * 16));
    const int smem = 4 * 2 * 32 * 33 * sizeof(double);
    HPBJ_CUDA(cudaFuncSetAttribute(k_spk_build<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_spk_build<true><<<grid, 128, smem, st>>>(p);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_apply_step(const SpkView& v, const double* V, int ldv, const SolveState* sst, float* z32,
                       cudaStream_t st, int64_t* launches) {
    launch<float>(v, SrcDown{V, ldv, sst}, DstF32{z32}, sst, st, launches);
}

void launch_apply_vec(const SpkView& v, const double* vin, double* z64, cudaStream_t st, int64_t* launches) {
    launch<float>(v, SrcVec{vin}, DstF64{z64}, nullptr, st, launches);
}

void launch_apply_update(const SpkView& v, const double* V, int ldv, const double* y, const SolveState* sst,
                         double* x, cudaStream_t st, int64_t* launches) {
    launch<double>(v, SrcBasis{V, ldv, y, sst}, DstAddX{x}, nullptr, st, launches);
}

}  // namespace hpbj
