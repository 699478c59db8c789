// Sparse-panel ("SPK") storage of the block factors and the block-Jacobi
// apply on it — replaces Preconditioner::apply_impl (preconditioner.cpp:
// 159-188) + lu_solve<T> (lu.hpp:88-112).
//
// The batched LU (block_lu.cu) leaves F = L\U of every block in dense 32-row
// panels. Fill-in is sparse (5-22% of d^2 on the BASELINE configs), so for
// the hot apply each panel is repacked (once per factorisation):
//   * off-panel entries of the panel's 32 rows — the L part (columns left of
//     the panel) and the U part (columns right of it) — in slot-major
//     ("jagged diagonal") order in chunks of four: slot k holds entries
//     4k..4k+3 of every row that has more than 4k entries, rows ascending,
//     zero padded; FP32 value + uint16 block-local column (6 B), plus the 32
//     row lengths of each part;
//   * the inverse of the 32x32 diagonal tile (unit-lower Linv and upper
//     Uinv, FP64-inverted, stored FP32) in a lane-quad layout so each lane
//     fetches its row segment as coalesced float4 loads (the forward pass
//     reads only the strictly-lower quads, the backward pass the upper ones).
// Per block one warp runs the blocked substitution (spk_dev.cuh): lane r owns
// panel row r, walks its own entries one 4-entry slot per step (each slot
// one coalesced float4 + ushort4 load; position by ballot/popc) and
// accumulates in a register;
// the in-panel triangle is a 32-wide mat-vec with the inverse tile.

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "kernels.cuh"
#include "spk_dev.cuh"

namespace hpbj {

namespace {

using namespace spk;

constexpr int kWarpsPerCta = 4;
// tile pass, per warp: the tile as FP64 [32][kTdLd] (even stride: 16-byte
// aligned pairs) + an FP32 [32][33] transpose buffer
constexpr int kTdLd = 34;
constexpr int kTileWarpDoubles = 32 * kTdLd + (32 * 33 + 1) / 2;
// pack pass, per warp: the slot starts of the longest row-quad part
__host__ __device__ inline int pack_slot_ints(int dmax) { return ((dmax + 3) / 4 + 4) & ~3; }

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x - v;
}

// Quad qi (columns 4 qi .. 4 qi + 3) of row k: one aligned float4.
__device__ __forceinline__ float4 dense_quad(const float* F, int dq, int k, int qi) {
    const int t = k >> 5;
    return __ldg(reinterpret_cast<const float4*>(F + (size_t)t * 32 * 4 * dq + qi * 128 + (k & 31) * 4));
}
__device__ __forceinline__ int nnz4(float4 v) {
    return (v.x != 0.0f) + (v.y != 0.0f) + (v.z != 0.0f) + (v.w != 0.0f);
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Row-quad layout of one off-panel part (columns [lo, hi) of panel row k):
// each row's nonzeros in quads of four (zero padded), quad i of the row with
// rank r (rows ranked by quad count desc, then row asc) at quad slot
// S[i] + r, S[i] = number of quads in the slots before i. The active rows of
// slot i are then ranks 0..c_i-1: the apply's lane r reads one coalesced
// float4 + index quad per slot (spk_dev.cuh fold_rows). S (mq + 1 ints of
// the warp's shared memory) is built by one ballot per slot; each lane then
// scans its row once.
template <class IdxT>
__device__ void pack_row_quads(const SpkBuild& p, const float* F, int dq, int k, bool live, int lo, int hi, int q,
                               int rank, int mq, int base, int* S, int lane) {
    int run = 0;
    for (int i = 0; i < mq; ++i) {
        const int c = __popc(__ballot_sync(0xffffffffu, i < q));
        if (lane == 0) S[i] = run;
        run += c;
    }
    __syncwarp();
    int cnt = 0;
    IdxT* eidx = reinterpret_cast<IdxT*>(p.eidx);
    if (live) {
        const int qe = (hi + 3) >> 2;
        for (int q0 = lo >> 2; q0 < qe; q0 += 4) {
            float4 v4[4];  // four quads in flight per lane
#pragma unroll
            for (int g = 0; g < 4; ++g)
                v4[g] = q0 + g < qe ? dense_quad(F, dq, k, q0 + g) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const float fv[4] = {v4[g].x, v4[g].y, v4[g].z, v4[g].w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = 4 * (q0 + g) + u;
                    if (fv[u] != 0.0f && c >= lo && c < hi) {
                        const int e = base + 4 * (S[cnt >> 2] + rank) + (cnt & 3);
                        p.eval[e] = fv[u];
                        eidx[e] = (IdxT)c;
                        ++cnt;
                    }
                }
            }
        }
    }
    for (; cnt & 3; ++cnt) {  // zero padding of the last quad
        const int e = base + 4 * (S[cnt >> 2] + rank) + (cnt & 3);
        p.eval[e] = 0.0f;
        eidx[e] = (IdxT)0;
    }
    __syncwarp();
}

// Pass 3 for one panel: inverse of the 32x32 diagonal triangle.
__device__ __forceinline__ void spk_tile(const SpkBuild& p, const float* F, int dq, int k, int d, int c0, int c1, int P,
                                         bool last, int lane, double* inv_smem) {
    // Inverse of the 32x32 diagonal triangle, in FP64 from the FP32
    // factors: Linv (unit lower) and Uinv (upper incl. diagonal), written
    // as 9 float4 quads per row (see kernels.cuh SpkView::dtile). The
    // block's last panel stores the product Uinv Linv instead (8 quads):
    // its forward and backward in-panel solves are back to back (no U
    // entries right of it), so the apply does them as one mat-vec.
    {
        // tile (FP32 factor values, held as FP64 — exact — so the
        // substitutions read each operand with one broadcast load, two per
        // LDS.128, and no conversion) and an FP32 transpose buffer in shared
        // memory; the column of the inverse a lane computes stays in
        // registers (fully unrolled substitutions, two partial sums per row)
        double* Td = reinterpret_cast<double*>(inv_smem) + (size_t)(threadIdx.x >> 5) * kTileWarpDoubles;
        float* W = reinterpret_cast<float*>(Td + 32 * kTdLd);
        for (int q = 0; q < 8; ++q) {
            const float4 v4 = (k < d && c0 + 4 * q < c1) ? dense_quad(F, dq, k, (c0 >> 2) + q)
                                                         : make_float4(0.f, 0.f, 0.f, 0.f);
            const float fv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = 4 * q + u;
                // padded rows/columns: identity
                Td[lane * kTdLd + c] = (k < d && c0 + c < c1) ? (double)fv[u] : ((c == lane) ? 1.0 : 0.0);
            }
        }
        __syncwarp();
        // lane = column c of the inverses
        const int c = lane;
        double x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {  // L x = e_c, unit lower
            double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
            for (int j = 0; j + 1 < i; j += 2) {
                const double2 t = *reinterpret_cast<const double2*>(Td + i * kTdLd + j);
                s0 -= t.x * x[j];
                s1 -= t.y * x[j + 1];
            }
            if (i & 1) s0 -= Td[i * kTdLd + i - 1] * x[i - 1];
            x[i] = (i < c) ? 0.0 : s0 + s1;
        }
        float4* tile = reinterpret_cast<float4*>(p.dtile + (size_t)P * kTileFloats);
        const int qd = lane >> 2;  // the quad holding the diagonal
        if (!last) {  // quads 0..qd of row `lane`: strictly lower Linv (through the transpose buffer)
#pragma unroll
            for (int i = 0; i < 32; ++i) W[i * 33 + c] = (float)x[i];
            __syncwarp();
            for (int q = 0; q <= qd; ++q) {
                float4 v4;
                float* w4 = &v4.x;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = 4 * q + u;
                    w4[u] = (j < lane) ? W[lane * 33 + j] : 0.0f;
                }
                tile[q * 32 + lane] = v4;
            }
            __syncwarp();
        }
        // U x = e_c (Uinv, upper with diagonal); last panel: U x = Linv e_c
        // in place (x = Uinv Linv = (L U)^-1 of the diagonal tile)
#pragma unroll
        for (int i = 31; i >= 0; --i) {
            double s0 = last ? x[i] : ((i == c) ? 1.0 : 0.0), s1 = 0.0;
            int j = i + 1;
            if (j & 1) {
                if (j < 32) s0 -= Td[i * kTdLd + j] * x[j];
                ++j;
            }
#pragma unroll
            for (; j + 1 < 32; j += 2) {
                const double2 t = *reinterpret_cast<const double2*>(Td + i * kTdLd + j);
                s0 -= t.x * x[j];
                s1 -= t.y * x[j + 1];
            }
            x[i] = (!last && i > c) ? 0.0 : (s0 + s1) / Td[i * kTdLd + i];
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) W[i * 33 + c] = (float)x[i];  // row `lane`: W[lane * 33 + j]
        __syncwarp();
        if (last) {  // row `lane` of Uinv Linv
            for (int q = 0; q < 9; ++q) {
                float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
                if (q < 8) v4 = make_float4(W[lane * 33 + 4 * q], W[lane * 33 + 4 * q + 1], W[lane * 33 + 4 * q + 2],
                                            W[lane * 33 + 4 * q + 3]);
                tile[q * 32 + lane] = v4;
            }
        } else {  // quads qd+1..7 and quad 8 (the diagonal quad's part) of row `lane`: upper Uinv
            for (int q = qd + 1; q < 10; ++q) {
                const int qq = q == 9 ? qd : q;
                if (q == 8) continue;
                float4 v4;
                float* w4 = &v4.x;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = 4 * qq + u;
                    w4[u] = (j >= lane) ? W[lane * 33 + j] : 0.0f;
                }
                tile[(q == 9 ? 8 : q) * 32 + lane] = v4;
            }
        }
        __syncwarp();
    }
}

// Pass 1 (count), pass 2 (pack the off-panel entries), pass 3 (invert the
// diagonal tiles); warp per panel, lane = panel row. The pack pass streams the
// dense panels (HBM bound: few registers, many warps, four quads in flight per
// lane); the tile pass holds an FP64 column of the inverse in registers (168)
// but reads only the 32x32 tiles.
enum { kSpkCount = 0, kSpkPack = 1, kSpkTile = 2 };
template <int MODE, class IdxT, bool ROWS = false>
__global__ void __launch_bounds__(MODE == kSpkTile ? 128 : 256, MODE == kSpkTile ? 3 : 4) k_spk_build(SpkBuild p) {
    constexpr bool PACK = MODE != kSpkCount;
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
        if (MODE == kSpkTile) {
            spk_tile(p, F, dq, k, d, c0, c1, P, 32 * (t + 1) >= d, lane, inv_smem);
            continue;
        }
        int nl = 0, nu = 0;
        if (!PACK) {
            if (k < d) {  // whole quads: c0 and c1 < d are multiples of 4, columns >= d are zero
                for (int qi = 0; qi < (c0 >> 2); ++qi) nl += nnz4(dense_quad(F, dq, k, qi));
                if (c1 < d)
                    for (int qi = c1 >> 2; qi < dq; ++qi) nu += nnz4(dense_quad(F, dq, k, qi));
            }
            p.rowcnt[(size_t)P * 64 + lane] = (uint16_t)nl;
            p.rowcnt[(size_t)P * 64 + 32 + lane] = (uint16_t)nu;
        } else {
            nl = p.rowcnt[(size_t)P * 64 + lane];
            nu = p.rowcnt[(size_t)P * 64 + 32 + lane];
        }
        const int el = warp_excl_scan(nl, lane), eu = warp_excl_scan(nu, lane);
        const int tl = __shfl_sync(0xffffffffu, el + nl, 31);
        const int tu = __shfl_sync(0xffffffffu, eu + nu, 31);
        const int pl = (tl + 3) & ~3, pu = (tu + 3) & ~3;  // parts start 16-byte aligned
        const int ql = (nl + 3) >> 2, qu = (nu + 3) >> 2;  // row quads
        const int sl = warp_sum_int(ql), su = warp_sum_int(qu);
        if (!PACK) {
            if (lane == 0) {
                p.ent_count[P] = pl + pu;
                p.ent_count_rows[P] = 4 * (sl + su);
                atomicAdd(p.totals, (unsigned long long)(pl + pu));
                atomicAdd(p.totals + 1, (unsigned long long)(4 * (sl + su)));
            }
            continue;
        }
        const int base = p.ent_off[P];
        int rl = 0, ru = 0, mql = 0, mqu = 0;  // row-quad layout: ranks, longest rows
        if (ROWS) {
            for (int j = 0; j < 32; ++j) {
                const int a = __shfl_sync(0xffffffffu, ql, j), b = __shfl_sync(0xffffffffu, qu, j);
                rl += (a > ql) || (a == ql && j < lane);
                ru += (b > qu) || (b == qu && j < lane);
                mql = max(mql, a);
                mqu = max(mqu, b);
            }
            if (lane == 0)
                p.desc[P] = SpkPanel{base, mql | (sl << kRowQuadBits), mqu | (su << kRowQuadBits), base + 4 * sl};
            p.rmeta[(size_t)(2 * P) * 32 + rl] = (uint16_t)(lane | (ql << 5));
            p.rmeta[(size_t)(2 * P + 1) * 32 + ru] = (uint16_t)(lane | (qu << 5));
        } else {
            if (lane == 0) p.desc[P] = SpkPanel{base, tl, tu, base + pl};
            // the folds read whole quads: the padding up to each part's end is (0, col 0, row 0)
            if (lane < pl - tl) {
                p.eval[base + tl + lane] = 0.0f;
                reinterpret_cast<IdxT*>(p.eidx)[base + tl + lane] = (IdxT)0;
            } else if (lane >= 4 && lane - 4 < pu - tu) {
                p.eval[base + pl + tu + lane - 4] = 0.0f;
                reinterpret_cast<IdxT*>(p.eidx)[base + pl + tu + lane - 4] = (IdxT)0;
            }
        }
        if (ROWS) {
            int* S = reinterpret_cast<int*>(inv_smem) + (size_t)(threadIdx.x >> 5) * pack_slot_ints(p.dmax);
            pack_row_quads<IdxT>(p, F, dq, k, k < d, 0, c0, ql, rl, mql, base, S, lane);
            pack_row_quads<IdxT>(p, F, dq, k, k < d, c1, d, qu, ru, mqu, base + 4 * sl, S, lane);
            continue;
        }
        // off-panel entries, row-sorted: value + packed (column << 5 | row)
        if (k < d) {
            auto emit = [&](int qlo, int qhi, int q) {
                for (int qi = qlo; qi < qhi; ++qi) {
                    const float4 v4 = dense_quad(F, dq, k, qi);
                    const float fv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (fv[u] != 0.0f) {
                            p.eval[q] = fv[u];
                            reinterpret_cast<IdxT*>(p.eidx)[q] = (IdxT)(((unsigned)(4 * qi + u) << 5) | lane);
                            ++q;
                        }
                }
            };
            emit(0, c0 >> 2, base + el);
            if (c1 < d) emit(c1 >> 2, dq, base + pl + eu);
        }
    }
}

__global__ void k_panel_owner(const int* __restrict__ pstart, int s, int* __restrict__ panel_block) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < s; b += gridDim.x * blockDim.x)
        for (int P = pstart[b]; P < pstart[b + 1]; ++P) panel_block[P] = b;
}

// STAGE: tile quads staged through shared memory by cp.async so their
// latency overlaps the fold — a win for shallow blocks (few, short folds),
// a loss for deep ones (long folds already hide it; fewer resident warps).
constexpr int kStageMaxDim = 160;

template <class Acc, class IdxT, bool STAGE, bool ROWS, class Src, class Dst>
__global__ void __launch_bounds__(kWarpsPerCta * 32, ROWS ? 7 : 8) k_apply_spk(SpkView p, Src src, Dst dst,
                                                                 const SolveState* sst, int ystride) {
    if (sst && sst->done) return;
    extern __shared__ __align__(16) unsigned char spk_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int tmax = ystride / 32;
    constexpr int TB = STAGE ? 4096 : 0;
    // per warp: [tile staging (8 x 32 float4)], y/x buffer (Acc[ystride]), panel descriptors,
    // [row-quad metadata (2 x 32 uint16 per panel)]
    const size_t per = TB + sizeof(Acc) * ystride + sizeof(SpkPanel) * tmax + (ROWS ? 128 * tmax : 0);
    unsigned char* wbase = spk_smem + (size_t)wid * per;
    float4* tbuf = reinterpret_cast<float4*>(wbase);
    Acc* ybuf = reinterpret_cast<Acc*>(wbase + TB);
    SpkPanel* dsh = reinterpret_cast<SpkPanel*>(wbase + TB + sizeof(Acc) * ystride);
    uint16_t* msh = reinterpret_cast<uint16_t*>(wbase + TB + sizeof(Acc) * ystride + sizeof(SpkPanel) * tmax);
    const int nw = gridDim.x * kWarpsPerCta;
    const int b_first = blockIdx.x * kWarpsPerCta + wid;
    if (b_first < p.s) {
        prefetch_block_head<IdxT>(p, b_first, lane);
        if (p.pf) src.prefetch(p.bstart[b_first], p.bstart[b_first + 1] - p.bstart[b_first], lane);
    }
    for (int b = b_first; b < p.s; b += nw)
        spk_solve_block<Acc, IdxT, STAGE, ROWS>(p, b, b + nw < p.s ? b + nw : -1, src, dst, ybuf, dsh, lane, tbuf,
                                                msh);
}

template <class Acc, class Src, class Dst>
void launch(const SpkView& v, Src src, Dst dst, const SolveState* sst, cudaStream_t st, int64_t* launches) {
    const int ystride = ((v.dmax + 31) / 32) * 32;
    const bool stage = v.dmax <= kStageMaxDim;
    const size_t smem = ((stage ? 4096 : 0) + sizeof(Acc) * ystride + sizeof(SpkPanel) * (ystride / 32) +
                         (v.rows ? 128 * (ystride / 32) : 0)) *
                        kWarpsPerCta;
    const int grid = (v.s + kWarpsPerCta - 1) / kWarpsPerCta;
#define HPBJ_APPLY(IDX, STG, RW) k_apply_spk<Acc, IDX, STG, RW, Src, Dst><<<grid, kWarpsPerCta * 32, smem, st>>>(v, src, dst, sst, ystride)
    if (v.rows) {
        if (v.idx32) HPBJ_APPLY(uint32_t, false, true);
        else HPBJ_APPLY(uint16_t, false, true);
    } else if (v.idx32) {
        if (stage) HPBJ_APPLY(uint32_t, true, false);
        else HPBJ_APPLY(uint32_t, false, false);
    } else {
        if (stage) HPBJ_APPLY(uint16_t, true, false);
        else HPBJ_APPLY(uint16_t, false, false);
    }
#undef HPBJ_APPLY
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace

void launch_spk_count(const SpkBuild& p, cudaStream_t st, int64_t* launches) {
    k_panel_owner<<<std::max(1, std::min((p.s + 255) / 256, 1184)), 256, 0, st>>>(p.pstart, p.s, p.panel_block);
    const int grid = std::max(1, std::min((p.num_panels * 32 + 255) / 256, 148 * 16));
    HPBJ_CUDA(cudaMemsetAsync(p.totals, 0, 2 * sizeof(unsigned long long), st));
    k_spk_build<kSpkCount, uint16_t><<<grid, 256, 0, st>>>(p);
    *launches += 2;
    HPBJ_CUDA(cudaGetLastError());
}

// The diagonal-tile inverses: depend on the dense panels and the panel
// owners only (launch after launch_spk_count, possibly on another stream).
void launch_spk_tile(const SpkBuild& p, cudaStream_t st, int64_t* launches) {
    const int tgrid = std::max(1, std::min((p.num_panels * 32 + 127) / 128, 148 * 16));
    const int tsmem = 4 * kTileWarpDoubles * sizeof(double);
    HPBJ_CUDA(cudaFuncSetAttribute(k_spk_build<kSpkTile, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem));
    k_spk_build<kSpkTile, uint16_t><<<tgrid, 128, tsmem, st>>>(p);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

void launch_spk_pack(const SpkBuild& p, cudaStream_t st, int64_t* launches) {
    const int grid = std::max(1, std::min((p.num_panels * 32 + 255) / 256, 148 * 16));
    const int smem = 8 * pack_slot_ints(p.dmax) * sizeof(int);
    auto fn = p.rows ? (p.idx32 ? k_spk_build<kSpkPack, uint32_t, true> : k_spk_build<kSpkPack, uint16_t, true>)
                     : (p.idx32 ? k_spk_build<kSpkPack, uint32_t> : k_spk_build<kSpkPack, uint16_t>);
    if (smem > 48 * 1024) HPBJ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    fn<<<grid, 256, smem, st>>>(p);
    *launches += 1;
    HPBJ_CUDA(cudaGetLastError());
}

namespace {

// Truncated Neumann series z = sum_{i=0..k} (I - Phi^-1 A)^i Phi^-1 v
// (apply_neumann, preconditioner.cpp:200-220): the first apply seeds term and
// acc, each later apply (of A term) folds "term -= corr; acc += term" into its
// store, in T like the reference's vectors; xadd (optional) receives x += acc.
template <class T>
struct DstNeumann {
    T* term;
    T* acc;
    double* xadd;
    double* out;
    int init;
    template <class V>
    __device__ void operator()(int row, V v) const {
        T a;
        if (init) {
            term[row] = (T)v;
            a = (T)v;
        } else {
            const T t = term[row] - (T)v;
            term[row] = t;
            a = acc[row] + t;
        }
        acc[row] = a;
        if (xadd) xadd[row] = xadd[row] + (double)a;
        if (out) out[row] = (double)a;
    }
};
struct SrcVec64 {
    const double* v;
    __device__ double operator()(int row) const { return __ldg(v + row); }
    __device__ void prefetch(int o, int d, int lane) const { prefetch_rows_l2(v, o, d, lane); }
};

}  // namespace

void launch_apply_neumann_f32(const SpkView& v, const double* vin, const double* V, int ldv, float* term,
                              float* acc, double* out, int init, const SolveState* sst, cudaStream_t st,
                              int64_t* launches) {
    const DstNeumann<float> dst{term, acc, nullptr, out, init};
    if (V) launch<float>(v, SrcDown{V, ldv, sst}, dst, sst, st, launches);
    else launch<float>(v, SrcVec{vin}, dst, sst, st, launches);
}

void launch_apply_neumann_f64(const SpkView& v, const double* vin, const double* V, int ldv, const double* y,
                              double* term, double* acc, double* xadd, int init, const SolveState* sst,
                              cudaStream_t st, int64_t* launches) {
    const DstNeumann<double> dst{term, acc, xadd, nullptr, init};
    if (V) launch<double>(v, SrcBasis{V, ldv, y, sst}, dst, nullptr, st, launches);
    else launch<double>(v, SrcVec64{vin}, dst, nullptr, st, launches);
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
