// Batched FP32 LU of the block-Jacobi diagonal blocks — replaces gp_lu
// (lu.cpp:134-225) + slice_diag_block (preconditioner.cpp:20-40) +
// matrix_inf_norm (sparse_matrix.cpp:155-166) + materialize_low.
//
// One CTA per block (persistent over blocks). The block is gathered from the
// permuted CSR straight into a dense FP32 tile (FP64 -> FP32 RNE on load),
// held in shared memory when it fits (dim <= smem_dim, ~223) and in a
// per-CTA global scratch tile otherwise (L1/L2 resident).
//
// Pivoting semantics match the reference:
//  * pivot of column k = argmax |x_i| over not-yet-pivotal rows, ties to the
//    smallest (original, local) row index (lu.cpp:171-181). Rows are never
//    physically swapped ("logical" pivoting), so the row index used for the
//    tie break is the reference's.
//  * an all-zero candidate column picks the smallest unused row, as the
//    empty-column fallback (lu.cpp:182-186) does; see DESIGN.md for the one
//    structurally-zero corner where the reference restricts to its reach set.
//  * regularize_pivot in FP64 against the FP64 block inf-norm (lu.cpp:10-20,
//    :188-197); a zero regularised pivot is SingularBlockError(column).
//
// Output: F = L_strict + U in pivot order, packed in 32-row panels (see
// kernels.cuh panel_floats) for the coalesced apply kernel; pivot_rows.

#include <cfloat>
#include <cstdlib>

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {

namespace {

constexpr int kLuThreads = 256;
constexpr int kLuMaxDim = 2048;          // act/prow arrays in static shared memory
constexpr size_t kLuSmemTile = 200 * 1024;

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
    return a > b ? a : b;
}

// x / pv, IEEE round-to-nearest (the multiplier of lu.cpp:207). A zero
// numerator over a finite nonzero pivot is the signed zero: returned without
// the division, whose range check (FCHK) sends zero numerators — most
// entries of a sparse block — down the slow software path.
__device__ __forceinline__ float div_mult(float x, float pv) {
    if (x == 0.0f && pv != 0.0f && isfinite(pv))
        return __int_as_float((__float_as_int(x) ^ __float_as_int(pv)) & (int)0x80000000);
    return x / pv;
}

// regularize_pivot's keep test (lu.cpp:10-20): norm == 0 ? p != 0 :
// RN(|p| / norm) >= eps. A product bracket decides it without the FP64
// division whenever |p| is not within 2^-48 (relative) of eps*norm: with
// t = RN(eps*norm) normal, |p| >= RN(t*(1+2^-48)) implies the exact quotient
// exceeds eps*(1+2^-49), so its rounding is >= eps; |p| <= RN(t*(1-2^-48))
// implies it is below eps*(1-2^-49), so its rounding is < eps. Otherwise (and
// for eps = 0, NaN, or t out of the normal range) the quotient is formed.
__device__ __forceinline__ bool pivot_keep(double pvd, double norm, double eps) {
    if (norm == 0.0) return pvd != 0.0;
    const double a = fabs(pvd);
    const double t = eps * norm;
    if (t >= DBL_MIN && t <= DBL_MAX * 0.5) {
        if (a >= t * (1.0 + 0x1p-48)) return true;
        if (a <= t * (1.0 - 0x1p-48)) return false;
    }
    return a / norm >= eps;
}

// pivot_keep's brackets as FP32 thresholds, once per block: for a float
// |p|, |p| >= RN(t (1 + 2^-48)) iff |p| >= its float ceiling, |p| <=
// RN(t (1 - 2^-48)) iff |p| <= its float floor; ok = 0 when the brackets do
// not apply (norm == 0, t outside the normal range) and the FP64 test runs.
struct KeepBrackets {
    float hi, lo;
    int ok;
};
__device__ __forceinline__ KeepBrackets keep_brackets(double norm, double eps) {
    KeepBrackets k{0.f, 0.f, 0};
    const double t = eps * norm;
    if (norm != 0.0 && t >= DBL_MIN && t <= DBL_MAX * 0.5) {
        k.hi = __double2float_ru(t * (1.0 + 0x1p-48));
        k.lo = __double2float_rd(t * (1.0 - 0x1p-48));
        k.ok = 1;
    }
    return k;
}
// pivot_keep(p, norm, eps) for a float pivot: the FP32 bracket decides it
// except within 2^-48 of the threshold
__device__ __forceinline__ bool pivot_keep_f(float p, const KeepBrackets& kb, double norm, double eps) {
    const float a = fabsf(p);
    if (kb.ok) {
        if (a >= kb.hi) return true;
        if (a <= kb.lo) return false;
    }
    return pivot_keep((double)p, norm, eps);
}

// Warp argmax of |x| with ties to the smallest row: returns the winning row
// (value key = float bits + 1 so that "no candidate" = 0; NaN keys win, as in
// the 64-bit (value, ~row) key max).
__device__ __forceinline__ int warp_pivot_row(unsigned key, int row, unsigned* kmax) {
    const unsigned mx = __reduce_max_sync(0xffffffffu, key);
    const unsigned pr = __reduce_min_sync(0xffffffffu, key == mx ? (unsigned)row : 0xFFFFFFFFu);
    *kmax = mx;
    return (int)pr;
}

// mode 0: blocks with d <= smem_dim (tile in shared memory)
// mode 1: blocks with d >  smem_dim (tile in global scratch)
__global__ void __launch_bounds__(kLuThreads) k_block_lu(LuParams p, int mode) {
    extern __shared__ float smem_tile[];
    __shared__ int act[kLuMaxDim];
    __shared__ int prow[kLuMaxDim];
    __shared__ unsigned long long red[kLuThreads / 32];
    __shared__ double redd[kLuThreads / 32];
    __shared__ int sh_p, sh_abort;
    __shared__ float sh_pv;
    __shared__ double sh_norm;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = kLuThreads / 32;

    for (int b = blockIdx.x; b < p.s; b += gridDim.x) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        if (d <= p.warp_dim) continue;  // warp-per-block kernel
        const bool in_smem = d <= p.smem_dim;
        if ((mode == 0) != in_smem) continue;
        const int ld = d | 1;  // odd stride: conflict-free column walks
        float* A = in_smem ? smem_tile : p.scratch + (size_t)blockIdx.x * p.scratch_ld * p.scratch_ld;

        for (int e = tid; e < d * ld; e += kLuThreads) A[e] = 0.0f;
        for (int r = tid; r < d; r += kLuThreads) act[r] = r;
        __syncthreads();

        // Gather the diagonal block (FP64 -> FP32) and its inf-norm. The row
        // sum runs sequentially in column order like matrix_inf_norm, so the
        // FP64 norm is bit-identical to the reference's.
        double wmax = 0.0;
        for (int r = tid; r < d; r += kLuThreads) {  // thread per row
            const int kb = __ldg(p.a.rp + o + r), ke = __ldg(p.a.rp + o + r + 1);
            double rs = 0.0;
            for (int k = kb; k < ke; ++k) {
                const int c = __ldg(p.a.ci + k) - o;
                if (c >= 0 && c < d) {
                    const double v = __ldg(p.a.val + k);
                    A[r * ld + c] = __double2float_rn(v);
                    rs = __dadd_rn(rs, fabs(v));
                }
            }
            wmax = fmax(wmax, rs);
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o2));
        if (lane == 0) redd[wid] = wmax;
        if (tid == 0) sh_abort = 0;
        __syncthreads();
        if (tid == 0) {
            double nm = 0.0;
            for (int w = 0; w < NW; ++w) nm = fmax(nm, redd[w]);
            sh_norm = nm;
        }
        __syncthreads();
        const double norm = sh_norm;

        int na = d;
        int nperturb = 0;
        for (int k = 0; k < d; ++k) {
            // ---- pivot search: max |a_rk|, ties -> smallest row r
            unsigned long long best = 0ull;
            for (int a = tid; a < na; a += kLuThreads) {
                const int r = act[a];
                const float v = fabsf(A[r * ld + k]);
                const unsigned long long key =
                    ((unsigned long long)(__float_as_uint(v) + 1u) << 32) |
                    ((unsigned long long)(0xFFFFu - (unsigned)r) << 16) | (unsigned)a;
                best = umax64(best, key);
            }
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) best = umax64(best, __shfl_xor_sync(0xffffffffu, best, o2));
            if (lane == 0) red[wid] = best;
            __syncthreads();
            if (tid == 0) {
                unsigned long long f = red[0];
                for (int w = 1; w < NW; ++w) f = umax64(f, red[w]);
                const int apos = (int)(f & 0xFFFFu);
                const int pr = act[apos];
                const float xp = A[pr * ld + k];
                // regularize_pivot (lu.cpp:10-20), FP64
                const double pvd = (double)xp;
                const bool keep = norm == 0.0 ? (pvd != 0.0) : (fabs(pvd) / norm >= p.eps);
                const double val = keep ? pvd : ((pvd < 0.0 ? -1.0 : 1.0) * p.eps * norm);
                if (val == 0.0) {
                    atomicMin(p.singular, ((unsigned long long)b << 32) | (unsigned)k);
                    sh_abort = 1;
                } else if (!keep) {
                    ++nperturb;
                    const int slot = atomicAdd(p.pert_n, 1);
                    if (slot < p.pert_cap) p.pert[slot] = PertRecord{b, k, pvd, val};
                }
                const float fv = (float)val;
                A[pr * ld + k] = fv;
                prow[k] = pr;
                act[apos] = act[na - 1];
                sh_pv = fv;
                sh_p = pr;
            }
            __syncthreads();
            if (sh_abort) break;
            --na;
            // ---- multipliers and rank-1 update of the active rows
            const float pv = sh_pv;
            const float* urow = A + sh_p * ld;
            for (int a = wid; a < na; a += NW) {
                const int r = act[a];
                float* arow = A + r * ld;
                const float l = div_mult(arow[k], pv);
                for (int j = k + 1 + lane; j < d; j += 32) arow[j] = fmaf(-l, urow[j], arow[j]);
                __syncwarp();
                if (lane == 0) arow[k] = l;
            }
            __syncthreads();
        }
        if (tid == 0) p.pert_count[b] = nperturb;
        if (!sh_abort) {
            // ---- write F = L\U in pivot order into packed 32-row panels
            const int T = (d + 31) / 32;
            const int dp4 = (d + 3) & ~3;
            const int total = T * 32 * dp4;
            float* F = p.fac + p.fac_off[b];
            for (int e = tid; e < total; e += kLuThreads) {
                const int t = e / (32 * dp4);
                const int rem = e - t * 32 * dp4;
                const int c = ((rem >> 7) << 2) | (rem & 3);
                const int k = 32 * t + ((rem >> 2) & 31);
                float v;
                if (k < d && c < d) v = A[prow[k] * ld + c];
                else v = (k == c) ? 1.0f : 0.0f;
                F[e] = v;
            }
            for (int k = tid; k < d; k += kLuThreads) p.piv[o + k] = prow[k];
        }
        __syncthreads();
    }
}


// ---------------------------------------------------------------------------
// Warp-per-block LU for blocks that fit a per-warp shared-memory tile
// (d <= kWarpLuMax): warp-synchronous right-looking elimination — lane l owns
// rows l, l+32, ... — so no CTA barrier sits on the per-column critical path.
// Same pivot rule, regularisation and output as k_block_lu.
constexpr int kWarpLuMax = 96;  // measured: above this the blocked kernel is faster

template <int kWarpLuRowsPerLane>  // rows per lane = ceil(max block dim / 32)
__global__ void __launch_bounds__(256) k_block_lu_warp(LuParams p, int dw, int ldw) {
    extern __shared__ float wsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nwc = blockDim.x >> 5;
    float* A = wsm + (size_t)wid * (dw * ldw + dw);  // tile + prow
    int* prow = reinterpret_cast<int*>(A + dw * ldw);
    const int gw = blockIdx.x * nwc + wid, nw = gridDim.x * nwc;
    for (int b = gw; b < p.s; b += nw) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        if (d > dw) continue;
        const int ld = d | 1;
        for (int e = lane; e < d * ld; e += 32) A[e] = 0.0f;
        __syncwarp();
        // gather + FP64 inf-norm (row sums sequential in column order, as
        // matrix_inf_norm sparse_matrix.cpp:155-166)
        double nrm = 0.0;
        for (int r = lane; r < d; r += 32) {  // lane per row: all rows' loads in flight
            const int kb = __ldg(p.a.rp + o + r), ke = __ldg(p.a.rp + o + r + 1);
            double rs = 0.0;
            for (int k = kb; k < ke; ++k) {
                const int c = __ldg(p.a.ci + k) - o;
                if (c >= 0 && c < d) {
                    const double v = __ldg(p.a.val + k);
                    A[r * ld + c] = __double2float_rn(v);
                    rs = __dadd_rn(rs, fabs(v));
                }
            }
            nrm = fmax(nrm, rs);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, off));
        __syncwarp();
        unsigned pivoted = 0u;  // bit q: row lane + 32 q already pivotal
        int nperturb = 0;
        bool abort = false;
        for (int k = 0; k < d; ++k) {
            // pivot: max |a_rk| over unpivoted rows, ties -> smallest row
            unsigned bk = 0u;
            int brow = 0x7fffffff;
#pragma unroll
            for (int q = 0; q < kWarpLuRowsPerLane; ++q) {
                const int r = lane + 32 * q;
                if (r < d && !((pivoted >> q) & 1u)) {
                    const unsigned key = __float_as_uint(fabsf(A[r * ld + k])) + 1u;
                    if (key > bk) {  // rows ascend with q: an equal key keeps the smaller row
                        bk = key;
                        brow = r;
                    }
                }
            }
            unsigned kmx;
            const int pr = warp_pivot_row(bk, brow, &kmx);
            const float xp = A[pr * ld + k];
            // regularize_pivot (lu.cpp:10-20), FP64, identical in every lane
            const double pvd = (double)xp;
            const bool keep = pivot_keep(pvd, nrm, p.eps);
            const double val = keep ? pvd : ((pvd < 0.0 ? -1.0 : 1.0) * p.eps * nrm);
            if (val == 0.0) {
                if (lane == 0) atomicMin(p.singular, ((unsigned long long)b << 32) | (unsigned)k);
                abort = true;
                break;
            }
            if (!keep) {
                ++nperturb;
                if (lane == 0) {
                    const int slot = atomicAdd(p.pert_n, 1);
                    if (slot < p.pert_cap) p.pert[slot] = PertRecord{b, k, pvd, val};
                }
            }
            const float pv = (float)val;
            __syncwarp();
            if (lane == (pr & 31)) {
                A[pr * ld + k] = pv;
                pivoted |= 1u << (pr >> 5);
                prow[k] = pr;
            }
            __syncwarp();
            const float* urow = A + pr * ld;
            float lq[kWarpLuRowsPerLane];
#pragma unroll
            for (int q = 0; q < kWarpLuRowsPerLane; ++q) {
                const int r = lane + 32 * q;
                lq[q] = 0.0f;
                if (r < d && !((pivoted >> q) & 1u)) {
                    lq[q] = div_mult(A[r * ld + k], pv);  // L(i,k) = x_i / pivot (lu.cpp:207)
                    A[r * ld + k] = lq[q];
                }
            }
            // rank-1 update with lanes over columns (j = k+1+lane+32c): the live
            // rows (unpivoted, l != 0; a uniform ballot mask) are walked four at a
            // time — their multipliers are shared-memory broadcasts and every
            // lane updates its own columns, so there is no divergence and the
            // loads of four rows are in flight together. Rows with l == 0 are
            // left bit-unchanged.
            unsigned lmask[kWarpLuRowsPerLane];
#pragma unroll
            for (int q = 0; q < kWarpLuRowsPerLane; ++q) lmask[q] = __ballot_sync(0xffffffffu, lq[q] != 0.0f);
            constexpr int C = kWarpLuRowsPerLane;  // column groups (d <= 32 C)
            float ucol[C];
            bool cj[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int j = k + 1 + lane + 32 * c;
                cj[c] = j < d;
                ucol[c] = cj[c] ? urow[j] : 0.0f;
            }
            float* Aj = A + k + 1 + lane;
#pragma unroll
            for (int q = 0; q < kWarpLuRowsPerLane; ++q) {
                unsigned m = lmask[q];
                while (m) {
                    int rr[4];
                    int nr = 0;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        rr[t] = m ? 32 * q + __ffs(m) - 1 : -1;
                        if (m) {
                            m &= m - 1;
                            ++nr;
                        }
                    }
                    float l[4], a[4][C];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        l[t] = rr[t] >= 0 ? A[rr[t] * ld + k] : 0.0f;
#pragma unroll
                        for (int c = 0; c < C; ++c) a[t][c] = (rr[t] >= 0 && cj[c]) ? Aj[rr[t] * ld + 32 * c] : 0.0f;
                    }
#pragma unroll
                    for (int t = 0; t < 4; ++t)
#pragma unroll
                        for (int c = 0; c < C; ++c)
                            if (rr[t] >= 0 && cj[c]) Aj[rr[t] * ld + 32 * c] = fmaf(-l[t], ucol[c], a[t][c]);
                    (void)nr;
                }
            }
            __syncwarp();
        }
        if (lane == 0) p.pert_count[b] = nperturb;
        if (!abort) {
            const int T = (d + 31) / 32;
            const int dp4 = (d + 3) & ~3;
            float* F = p.fac + p.fac_off[b];
            // panel t, element rem = (c >> 2) * 128 + (k & 31) * 4 + (c & 3):
            // lane-contiguous stores, the row index fixed per lane and panel
            for (int t = 0; t < T; ++t) {
                float* Ft = F + (size_t)t * 32 * dp4;
                const int k = 32 * t + (lane >> 2);  // rows of rem = lane + 32 i: (lane >> 2) + 8 (i & 3)
                for (int rem = lane; rem < 32 * dp4; rem += 32) {
                    const int c = ((rem >> 7) << 2) | (rem & 3);
                    const int kk = k + (((rem >> 5) & 3) << 3);
                    float v;
                    if (kk < d && c < d) v = A[prow[kk] * ld + c];
                    else v = (kk == c) ? 1.0f : 0.0f;
                    Ft[rem] = v;
                }
            }
            for (int k = lane; k < d; k += 32) p.piv[o + k] = prow[k];
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Two warps per block (d <= kWarpLuMax): the same elimination as
// k_block_lu_warp with the rows split between the warps (warp w owns rows
// lane + 32 (2q + w)), so each warp walks half of the live rows per column;
// the per-warp pivot candidates meet in shared memory behind one 64-thread
// barrier per column (double-buffered slots). Twice the resident warps per
// block's shared-memory tile and half the per-column chain: same pivots,
// same FMA sequence per element, bit-identical factors.
template <int C>  // column groups: d <= 32 C
__global__ void __launch_bounds__(64) k_block_lu_pair(LuParams p, int dw, int ldw) {
    extern __shared__ float wsm[];
    __shared__ unsigned sk[2][2];
    __shared__ int sr[2][2];
    __shared__ float sv[2][2];  // the candidates' values (read before the owner overwrites the pivot)
    __shared__ double snrm[2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, tid = threadIdx.x;
    float* A = wsm;
    int* prow = reinterpret_cast<int*>(A + dw * ldw);
    constexpr int R = 2;  // rows per lane and warp: lane + 32 (2q + w), q < 2 (d <= 128)
    for (int b = blockIdx.x; b < p.s; b += gridDim.x) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        if (d > dw) continue;
        const int ld = d | 1;
        for (int e = tid; e < d * ld; e += 64) A[e] = 0.0f;
        __syncthreads();
        // gather + FP64 inf-norm (row sums sequential in column order)
        double nrm = 0.0;
        for (int r = tid; r < d; r += 64) {
            const int kb = __ldg(p.a.rp + o + r), ke = __ldg(p.a.rp + o + r + 1);
            double rs = 0.0;
            for (int k = kb; k < ke; ++k) {
                const int c = __ldg(p.a.ci + k) - o;
                if (c >= 0 && c < d) {
                    const double v = __ldg(p.a.val + k);
                    A[r * ld + c] = __double2float_rn(v);
                    rs = __dadd_rn(rs, fabs(v));
                }
            }
            nrm = fmax(nrm, rs);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, off));
        if (lane == 0) snrm[w] = nrm;
        __syncthreads();
        nrm = fmax(snrm[0], snrm[1]);
        unsigned pivoted = 0u;  // bit q: row lane + 32 (2q + w) already pivotal
        int nperturb = 0;
        bool abort = false;
        for (int k = 0; k < d; ++k) {
            const int par = k & 1;
            unsigned bk = 0u;
            int brow = 0x7fffffff;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int r = lane + 32 * (2 * q + w);
                if (r < d && !((pivoted >> q) & 1u)) {
                    const unsigned key = __float_as_uint(fabsf(A[r * ld + k])) + 1u;
                    if (key > bk) {  // rows ascend with q: an equal key keeps the smaller row
                        bk = key;
                        brow = r;
                    }
                }
            }
            unsigned kmx;
            const int prw = warp_pivot_row(bk, brow, &kmx);
            const float xw = (kmx != 0u) ? A[prw * ld + k] : 0.0f;
            if (lane == 0) {
                sk[par][w] = kmx;
                sr[par][w] = prw;
                sv[par][w] = xw;
            }
            __syncthreads();
            const unsigned k0 = sk[par][0], k1 = sk[par][1];
            const int r0 = sr[par][0], r1 = sr[par][1];
            const bool first = k0 > k1 || (k0 == k1 && r0 < r1);  // max key, ties -> smaller row
            const int pr = first ? r0 : r1;
            const float xp = first ? sv[par][0] : sv[par][1];
            const double pvd = (double)xp;
            const bool keep = pivot_keep(pvd, nrm, p.eps);
            const double val = keep ? pvd : ((pvd < 0.0 ? -1.0 : 1.0) * p.eps * nrm);
            if (val == 0.0) {
                if (tid == 0) atomicMin(p.singular, ((unsigned long long)b << 32) | (unsigned)k);
                abort = true;
                break;
            }
            if (!keep) {
                ++nperturb;
                if (tid == 0) {
                    const int slot = atomicAdd(p.pert_n, 1);
                    if (slot < p.pert_cap) p.pert[slot] = PertRecord{b, k, pvd, val};
                }
            }
            const float pv = (float)val;
            const bool own = ((pr >> 5) & 1) == w;  // warp owning the pivot row
            __syncwarp();
            if (own && lane == (pr & 31)) {
                A[pr * ld + k] = pv;
                pivoted |= 1u << (pr >> 6);
                prow[k] = pr;
            }
            __syncwarp();
            const float* urow = A + pr * ld;
            float lq[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int r = lane + 32 * (2 * q + w);
                lq[q] = 0.0f;
                if (r < d && !((pivoted >> q) & 1u)) {
                    lq[q] = div_mult(A[r * ld + k], pv);  // L(i,k) = x_i / pivot (lu.cpp:207)
                    A[r * ld + k] = lq[q];
                }
            }
            unsigned lmask[R];
#pragma unroll
            for (int q = 0; q < R; ++q) lmask[q] = __ballot_sync(0xffffffffu, lq[q] != 0.0f);
            float ucol[C];
            bool cj[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int j = k + 1 + lane + 32 * c;
                cj[c] = j < d;
                ucol[c] = cj[c] ? urow[j] : 0.0f;
            }
            float* Aj = A + k + 1 + lane;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                unsigned m = lmask[q];
                const int rbase = 32 * (2 * q + w);
                while (m) {
                    int rr[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        rr[t] = m ? rbase + __ffs(m) - 1 : -1;
                        if (m) m &= m - 1;
                    }
                    float l[4], a[4][C];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        l[t] = rr[t] >= 0 ? A[rr[t] * ld + k] : 0.0f;
#pragma unroll
                        for (int c = 0; c < C; ++c) a[t][c] = (rr[t] >= 0 && cj[c]) ? Aj[rr[t] * ld + 32 * c] : 0.0f;
                    }
#pragma unroll
                    for (int t = 0; t < 4; ++t)
#pragma unroll
                        for (int c = 0; c < C; ++c)
                            if (rr[t] >= 0 && cj[c]) Aj[rr[t] * ld + 32 * c] = fmaf(-l[t], ucol[c], a[t][c]);
                }
            }
        }
        __syncthreads();
        if (tid == 0) p.pert_count[b] = nperturb;
        if (!abort) {
            const int T = (d + 31) / 32;
            const int dp4 = (d + 3) & ~3;
            float* F = p.fac + p.fac_off[b];
            for (int t = w; t < T; t += 2) {  // panel t: rem = (c >> 2) * 128 + (k & 31) * 4 + (c & 3)
                float* Ft = F + (size_t)t * 32 * dp4;
                const int k = 32 * t + (lane >> 2);
                for (int rem = lane; rem < 32 * dp4; rem += 32) {
                    const int c = ((rem >> 7) << 2) | (rem & 3);
                    const int kk = k + (((rem >> 5) & 3) << 3);
                    float v;
                    if (kk < d && c < d) v = A[prow[kk] * ld + c];
                    else v = (kk == c) ? 1.0f : 0.0f;
                    Ft[rem] = v;
                }
            }
            for (int k = tid; k < d; k += 64) p.piv[o + k] = prow[k];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Blocked right-looking LU for mid-size blocks (kWarpLuMax < d <= kBlkMax),
// one CTA per block, the block in a per-CTA global scratch tile (L2 resident,
// 16-byte rows). Per 32-column panel:
//   (1) the panel of the not-yet-pivotal rows is factored with each thread
//       holding its (<= 2) rows' 32 panel entries in registers: per column a
//       CTA argmax, the pivot row broadcast through shared memory, and the
//       rank-1 update restricted to the panel, all register-resident;
//   (2) the 32 pivot rows' entries right of the panel (U12) by forward
//       substitution with the panel's unit-lower part, thread per column;
//   (3) the remaining rows' trailing entries take the rank-32 update, each
//       element a chain of 32 FMAs in column order (warp per 4 rows, lane per
//       column, the U12 column in registers, multipliers as float4 broadcasts).
// Every element receives exactly the fmaf(-l, u, a) sequence, in the same
// column order, that the column-by-column kernels apply, and the pivot rule
// is the same, so factors and pivots are bit-identical to k_block_lu.
constexpr int kBlkThreads = 256;
constexpr int kBlkMax = 512;  // two panel rows per thread

__host__ __device__ inline int blk_ld(int d) { return (d + 3) & ~3; }

size_t blk_smem_bytes(int dhi) {
    const int d4 = blk_ld(dhi);
    return (size_t)dhi * 32 * sizeof(float)     // multipliers of the panel, 16-byte rows
           + (size_t)32 * d4 * sizeof(float)    // U12 / output staging
           + (size_t)dhi * 2 * sizeof(int)      // act, prow
           + (size_t)dhi;                       // panel pivot flags
}

template <int NT, int RPT>  // threads, panel rows per thread (d <= NT * RPT)
__global__ void __launch_bounds__(NT, 2) k_block_lu_blk(LuParams p, int dlo, int dhi, int ldmax) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) float bsm[];
    const int d4hi = blk_ld(dhi);
    float* Lm = bsm;                                  // [dhi][32]
    float* U = Lm + (size_t)dhi * 32;                 // [32][d4hi]
    int* act = reinterpret_cast<int*>(U + (size_t)32 * d4hi);
    int* prow = act + dhi;
    unsigned char* pflag = reinterpret_cast<unsigned char*>(prow + dhi);
    __shared__ __align__(16) float Pv[32];            // pivot row of the current column
    __shared__ unsigned red_k[NW];
    __shared__ int red_r[NW], red_a[NW];
    __shared__ double redd[NW];
    __shared__ int pc[32];
    __shared__ int sh_na;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    float* A = p.scratch + (size_t)blockIdx.x * ldmax * ldmax;

    for (int b = blockIdx.x; b < p.s; b += gridDim.x) {
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        if (d <= dlo || d > dhi) continue;
        const int ld = blk_ld(d);
        for (int e = tid; e < d * ld; e += NT) A[e] = 0.0f;
        for (int r = tid; r < d; r += NT) act[r] = r;
        __syncthreads();
        // gather (FP64 -> FP32) + FP64 inf-norm, row sums in column order
        double wmax = 0.0;
        for (int r = tid; r < d; r += NT) {
            const int kb = __ldg(p.a.rp + o + r), ke = __ldg(p.a.rp + o + r + 1);
            double rs = 0.0;
            for (int k = kb; k < ke; ++k) {
                const int c = __ldg(p.a.ci + k) - o;
                if (c >= 0 && c < d) {
                    const double v = __ldg(p.a.val + k);
                    A[r * ld + c] = __double2float_rn(v);
                    rs = __dadd_rn(rs, fabs(v));
                }
            }
            wmax = fmax(wmax, rs);
        }
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o2));
        if (lane == 0) redd[wid] = wmax;
        __syncthreads();
        double norm = 0.0;
        for (int w = 0; w < NW; ++w) norm = fmax(norm, redd[w]);

        int na = d;
        int nperturb = 0;
        bool abort = false;
        for (int k0 = 0; k0 < d; k0 += 32) {
            const int kw = min(32, d - k0);
            // (1) panel rows into registers: position a = tid + 256 i
            float rv[RPT][32];
            bool fl[RPT];
            int arow[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int a = tid + NT * i;
                fl[i] = a >= na;  // no row: treated as already pivotal
                arow[i] = a < na ? act[a] : 0;
                const float4* src = reinterpret_cast<const float4*>(A + arow[i] * ld + k0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (!fl[i] && 4 * q < kw) v = src[q];  // columns >= d: zero
                    rv[i][4 * q + 0] = v.x;
                    rv[i][4 * q + 1] = v.y;
                    rv[i][4 * q + 2] = v.z;
                    rv[i][4 * q + 3] = v.w;
                }
            }
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                if (c >= kw) break;
                const int k = k0 + c;
                // pivot: max |a_rk| over unpivoted rows, ties -> smallest row
                unsigned bk = 0u;
                int brow = 0x7fffffff, bpos = 0;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    if (fl[i]) continue;
                    const unsigned key = __float_as_uint(fabsf(rv[i][c])) + 1u;
                    if (key > bk || (key == bk && arow[i] < brow)) {
                        bk = key;
                        brow = arow[i];
                        bpos = tid + NT * i;
                    }
                }
                {
                    unsigned kmx;
                    const int wr = warp_pivot_row(bk, brow, &kmx);
                    const unsigned own_l = __ballot_sync(0xffffffffu, bk == kmx && brow == wr);
                    const int wpos = __shfl_sync(0xffffffffu, bpos, __ffs(own_l) - 1);
                    if (lane == 0) {
                        red_k[wid] = kmx;
                        red_r[wid] = wr;
                        red_a[wid] = wpos;
                    }
                }
                __syncthreads();
                unsigned fk = red_k[0];
                int frow = red_r[0], apos = red_a[0];
#pragma unroll
                for (int w = 1; w < NW; ++w)
                    if (red_k[w] > fk || (red_k[w] == fk && red_r[w] < frow)) {
                        fk = red_k[w];
                        frow = red_r[w];
                        apos = red_a[w];
                    }
                const int pr = act[apos];
                const int own = (apos - tid) % NT == 0 && apos >= tid ? (apos - tid) / NT : -1;
#pragma unroll
                for (int i = 0; i < RPT; ++i)  // broadcast the pivot row's panel entries
                    if (own == i)
#pragma unroll
                        for (int c2 = 0; c2 < 32; ++c2) Pv[c2] = rv[i][c2];
                __syncthreads();
                // regularize_pivot (lu.cpp:10-20), FP64, identical in every thread
                const double pvd = (double)Pv[c];
                const bool keep = pivot_keep(pvd, norm, p.eps);
                const double val = keep ? pvd : ((pvd < 0.0 ? -1.0 : 1.0) * p.eps * norm);
                if (val == 0.0) {
                    if (tid == 0) atomicMin(p.singular, ((unsigned long long)b << 32) | (unsigned)k);
                    abort = true;
                    break;
                }
                if (!keep) {
                    ++nperturb;
                    if (tid == 0) {
                        const int slot = atomicAdd(p.pert_n, 1);
                        if (slot < p.pert_cap) p.pert[slot] = PertRecord{b, k, pvd, val};
                    }
                }
                const float pv = (float)val;
                if (tid == 0) {
                    prow[k] = pr;
                    pc[c] = apos;
                }
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    if (fl[i]) continue;
                    if (own == i) {
                        rv[i][c] = pv;
                        fl[i] = true;
                        continue;
                    }
                    const float l = div_mult(rv[i][c], pv);  // L(i,k) = x_i / pivot (lu.cpp:207)
                    rv[i][c] = l;
#pragma unroll
                    for (int c2 = c + 1; c2 < 32; ++c2) rv[i][c2] = fmaf(-l, Pv[c2], rv[i][c2]);
                }
            }
            if (abort) break;
            // panel entries back to the tile (multipliers of every row, L11\U11 of
            // the pivot rows) and the multipliers to 16-byte shared rows; pivot flags
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int a = tid + NT * i;
                if (a >= na) continue;
                float4* dstg = reinterpret_cast<float4*>(A + arow[i] * ld + k0);
                float4* dsts = reinterpret_cast<float4*>(Lm + a * 32);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 v = make_float4(rv[i][4 * q], rv[i][4 * q + 1], rv[i][4 * q + 2], rv[i][4 * q + 3]);
                    if (4 * q < kw) dstg[q] = v;  // kw % 4 != 0 only for the last panel (d's own padding)
                    dsts[q] = v;
                }
            }
            // pivot flags from the (uniform) pivot positions of this panel
            for (int a = tid; a < na; a += NT) pflag[a] = 0;
            __syncthreads();
            if (tid < kw) pflag[pc[tid]] = 1;
            // (2) U12: pivot rows' entries right of the panel, forward substitution
            const int j0 = k0 + kw, nj = d - j0;
            for (int jj = tid; jj < nj; jj += NT) {
                float x[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) x[c] = c < kw ? A[act[pc[c]] * ld + j0 + jj] : 0.0f;
#pragma unroll
                for (int c = 1; c < 32; ++c) {
                    if (c >= kw) break;
                    const float* lrow = Lm + pc[c] * 32;
#pragma unroll
                    for (int m = 0; m < c; ++m) x[c] = fmaf(-lrow[m], x[m], x[c]);
                }
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    if (c < kw) {
                        U[c * d4hi + jj] = x[c];
                        A[act[pc[c]] * ld + j0 + jj] = x[c];
                    }
                }
            }
            __syncthreads();
            // (3) trailing rank-32 update (kw < 32 only in the last panel, which
            // has no trailing part)
            if (nj > 0) {
                for (int jc = 0; jc < nj; jc += 32) {
                    const int jj = jc + lane;
                    const bool colok = jj < nj;
                    float u[32];
#pragma unroll
                    for (int m = 0; m < 32; ++m) u[m] = colok ? U[m * d4hi + jj] : 0.0f;
                    for (int a0 = wid; a0 < na; a0 += 4 * NW) {
                        float v[4];
                        bool ok[4];
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int a = a0 + r * NW;
                            ok[r] = colok && a < na && !pflag[a];
                            v[r] = ok[r] ? A[act[a] * ld + j0 + jj] : 0.0f;
                        }
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const int a = min(a0 + r * NW, na - 1);
                                const float4 l4 = reinterpret_cast<const float4*>(Lm + a * 32)[q];
                                v[r] = fmaf(-l4.x, u[4 * q + 0], v[r]);
                                v[r] = fmaf(-l4.y, u[4 * q + 1], v[r]);
                                v[r] = fmaf(-l4.z, u[4 * q + 2], v[r]);
                                v[r] = fmaf(-l4.w, u[4 * q + 3], v[r]);
                            }
                        }
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            if (ok[r]) A[act[a0 + r * NW] * ld + j0 + jj] = v[r];
                    }
                }
            }
            __syncthreads();
            // drop this panel's pivot rows from the active list (order is free:
            // the pivot rule breaks ties by row index, not list position)
            if (wid == 0) {
                int w = 0;
                for (int base = 0; base < na; base += 32) {
                    const int a = base + lane;
                    const bool keepr = a < na && !pflag[a];
                    const int r = a < na ? act[a] : 0;
                    const unsigned m = __ballot_sync(0xffffffffu, keepr);
                    __syncwarp();
                    if (keepr) act[w + __popc(m & ((1u << lane) - 1u))] = r;
                    w += __popc(m);
                    __syncwarp();
                }
                if (lane == 0) sh_na = w;
            }
            __syncthreads();
            na = sh_na;
        }
        if (tid == 0) p.pert_count[b] = nperturb;
        if (!abort) {
            // F = L\U in pivot order into packed 32-row panels: stage the 32 pivot
            // rows of a panel in shared memory (coalesced row reads), then write the
            // panel contiguously (streaming stores: F is read once, by the SPK build)
            const int T = (d + 31) / 32;
            const int dp4 = (d + 3) & ~3;
            float* F = p.fac + p.fac_off[b];
            for (int t = 0; t < T; ++t) {
                __syncthreads();
                for (int e = tid; e < 32 * dp4; e += NT) {
                    const int kk = e / dp4, c = e - kk * dp4;
                    const int k = 32 * t + kk;
                    U[kk * d4hi + c] = (k < d && c < d) ? A[prow[k] * ld + c] : ((k == c) ? 1.0f : 0.0f);
                }
                __syncthreads();
                float* Ft = F + (size_t)t * 32 * dp4;
                for (int e = tid; e < 32 * dp4; e += NT) {
                    const int c = ((e >> 7) << 2) | (e & 3);
                    const int kk = (e >> 2) & 31;
                    __stcs(Ft + e, U[kk * d4hi + c]);
                }
            }
            for (int k = tid; k < d; k += NT) p.piv[o + k] = prow[k];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Left-looking blocked LU for kWarpLuMax < d <= kLlMax, two CTAs of 256
// threads per SM so that one block's latency-bound column chain overlaps the
// other block's bulk updates. Per block, shared memory holds only the current
// column panel X of all d rows (swizzled FP32) and staging buffers; the L part
// of the factor — per 32-column panel Q the 32 pivot rows of Q in pivot order
// (L11\U11 rows), then the rows still active after Q (their 32 multipliers),
// L_Q — goes to a per-CTA scratch in global memory (L2-resident) and comes
// back by bulk copies (cp.async.bulk + mbarrier): L11 of the next panels
// double-buffered, the bulk of L_{Q-1} single-buffered. U leaves for HBM
// panel by panel. Per column panel P (columns c0 .. c0 + 31):
//   gather  the panel's columns from the permuted CSR (per-row cursors, FP64
//           -> FP32 RNE into a zero-filled X);
//   for each earlier panel Q, pipelined so that the one-warp triangular solve
//   of Q overlaps the bulk rank-32 update of Q - 1:
//     A_Q  every warp: (ii)_{Q-1} = X[r] -= L_{Q-1}[r] U_{Q-1} on Q's 32 pivot rows;
//     B_Q  warp 0: (i)_Q, Q's pivot rows x_k -= sum_{m<k} L11(k, m) x_m (lane
//          per column, float4 broadcasts); the other warps: (ii)_{Q-1} on the
//          remaining rows active after Q;
//   then every warp: (ii)_{P-1} on the rows still active;
//   factor  the panel's active rows (thread per row, RPT rows per thread, 32
//           entries each in registers; only the warps holding rows, named
//           barrier): per column each warp publishes its candidate (max |x|,
//           ties to the smaller row) with the candidate's row, ONE barrier, a
//           warp-wide argmax over the candidates, the regularisation test in
//           FP32 brackets, the rank-1 update in registers;
//   store   L_P to the scratch; the new pivot rows' L entries and the
//           finished U column panel to the packed output panels.
// Every element receives exactly the fmaf(-l, u, a) chain, in ascending
// column order, that the right-looking kernels apply (left- and right-looking
// only reorder independent chains), the divisions and the pivot rule are the
// same: factors and pivots are bit-identical to k_block_lu_blk / k_block_lu.
template <int N>
struct IntC {
    static constexpr int value = N;
};

constexpr int kLlMax = 288;
constexpr int kLlThreads = 256;
constexpr int kLlCtasPerSm = 2;
constexpr int kXld = 36;  // X row stride (floats), see xe()

__host__ __device__ inline int ll_lrows(int d) {  // L_Q rows kept: panels 0 .. T-2
    const int T = (d + 31) / 32;
    int r = 0;
    for (int q = 0; q + 1 < T; ++q) r += d - 32 * q;
    return r;
}

__host__ __device__ inline size_t ll_smem_bytes(int dhi) {
    constexpr int NW = kLlThreads / 32;
    const int T = (dhi + 31) / 32;
    const int lr = ll_lrows(dhi);
    return (size_t)dhi * kXld * sizeof(float)               // X: current column panel, all rows
           + (size_t)(dhi > 32 ? dhi - 32 : 1) * 32 * sizeof(float)  // Lb: rows 32.. of L_{Q-1}
           + (size_t)2 * 32 * 32 * sizeof(float)            // L11 of two panels
           + (size_t)2 * NW * 32 * sizeof(float)            // candidate rows (double buffered)
           + (size_t)lr * sizeof(short)                     // row id of every L_Q row
           + (size_t)(T > 1 ? T - 1 : 1) * dhi * sizeof(short)  // position of row r in L_Q
           + (size_t)3 * dhi * sizeof(short)                // ppos, act, prow
           + 64;
}

// X rows padded to kXld = 36 floats: a warp reading one row lane by lane
// (the updates) and eight threads reading their own rows quad by quad (the
// panel factorisation: row r's quads start in bank group 9r mod 8) are both
// conflict-free, and an element address is one multiply-add
__device__ __forceinline__ int xq(int r, int q) { return r * kXld + (q << 2); }
__device__ __forceinline__ int xe(int r, int c) { return r * kXld + c; }

__device__ __forceinline__ void bar_named(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* mb) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb)) : "memory");
}
// one elected thread: expect `bytes` on mb and copy them global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* mb) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mb))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(mb)),
        "r"(parity)
        : "memory");
}

// X[r][lane] -= sum_m L[pos][m] u[m], u = this lane's column of the 32 pivot
// rows of the panel behind L (ll_load_u), for the rows given by (pos, row)
// pairs; four rows in flight per warp. `rows(i)` yields {pos, row} or pos < 0.
__device__ __forceinline__ void ll_load_u(float (&u)[32], const float* X, const short* prv, int lane) {
#pragma unroll
    for (int m = 0; m < 32; ++m) u[m] = X[xe(prv[m], lane)];
}

template <class Rows>
__device__ __forceinline__ void ll_rank32(float* X, const float* L, const float (&u)[32], int lane, int i0, int i1,
                                          int step, Rows rows) {
    for (int i = i0; i < i1; i += 4 * step) {
        int pos[4], rr[4];
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int2 pr = (i + t * step < i1) ? rows(i + t * step) : make_int2(-1, 0);
            pos[t] = pr.x;
            rr[t] = pr.y;
            v[t] = pos[t] >= 0 ? X[xe(rr[t], lane)] : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float4 l4 = *reinterpret_cast<const float4*>(L + (size_t)max(pos[t], 0) * 32 + 4 * q);
                v[t] = fmaf(-l4.x, u[4 * q + 0], v[t]);
                v[t] = fmaf(-l4.y, u[4 * q + 1], v[t]);
                v[t] = fmaf(-l4.z, u[4 * q + 2], v[t]);
                v[t] = fmaf(-l4.w, u[4 * q + 3], v[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (pos[t] >= 0) X[xe(rr[t], lane)] = v[t];
    }
}

// x_k -= sum_{m<k} L11(k, m) x_m, m ascending per k (the fmaf chain of the
// right-looking U12 solve), four m per step: L11 row k at LQ + 32 k.
template <int M0>
__device__ __forceinline__ void ll_trsv(float (&x)[32], const float* LQ) {
#pragma unroll
    for (int mm = 1; mm < 4; ++mm)
#pragma unroll
        for (int m = 0; m < mm; ++m) x[M0 + mm] = fmaf(-LQ[(M0 + mm) * 32 + M0 + m], x[M0 + m], x[M0 + mm]);
#pragma unroll
    for (int k = M0 + 4; k < 32; ++k) {
        const float4 l4 = *reinterpret_cast<const float4*>(LQ + k * 32 + M0);
        x[k] = fmaf(-l4.x, x[M0 + 0], x[k]);
        x[k] = fmaf(-l4.y, x[M0 + 1], x[k]);
        x[k] = fmaf(-l4.z, x[M0 + 2], x[k]);
        x[k] = fmaf(-l4.w, x[M0 + 3], x[k]);
    }
    if constexpr (M0 + 4 < 32) ll_trsv<M0 + 4>(x, LQ);
}

template <int RPT>  // active rows per thread: d <= 256 RPT
__global__ void __launch_bounds__(kLlThreads, kLlCtasPerSm) k_block_lu_ll(LuParams p, int dlo, int dhi) {
    constexpr int NT = kLlThreads;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(128) float llsm[];
    const int lrmax = ll_lrows(dhi);
    const int Tmax = (dhi + 31) / 32;
    float* X = llsm;                                           // [dhi][kXld]
    float* Lb = X + (size_t)dhi * kXld;                        // [dhi-32][32]
    float* L11 = Lb + (size_t)(dhi > 32 ? dhi - 32 : 1) * 32;  // [2][32][32]
    float* cand_v = L11 + 2 * 32 * 32;                         // [2][NW][32]
    short* rowQ = reinterpret_cast<short*>(cand_v + 2 * NW * 32);  // [lrmax]
    short* posQ = rowQ + lrmax;                                // [Tmax-1][dhi]
    short* ppos = posQ + (size_t)(Tmax > 1 ? Tmax - 1 : 1) * dhi;  // pivot position of row r (or 0x7fff)
    short* act = ppos + dhi;                                   // active rows (stable order)
    short* prow = act + dhi;                                   // pivot row of position k
    __shared__ __align__(8) unsigned long long mbar[3];        // Lb, L11[0], L11[1]
    __shared__ double redd[NW];
    __shared__ int lofs[16];                                   // first L row of panel Q
    __shared__ int nact_sh;
    __shared__ unsigned long long piv_best[3];                  // column winners (panel factorisation)
    float* Lg = p.scratch + (size_t)blockIdx.x * lrmax * 32;   // this CTA's L_Q rows

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        mbar_init(&mbar[0]);
        mbar_init(&mbar[1]);
        mbar_init(&mbar[2]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned nb_issue = 0, n11_issue[2] = {0u, 0u};  // completed-phase counters (uniform)

    // dynamic schedule, largest blocks first: a CTA takes the next unclaimed
    // block (static striding left the CTAs with the most expensive block
    // mixes behind; the small blocks at the end even out the tail)
    __shared__ int next_b;
    for (;;) {
        __syncthreads();
        if (tid == 0) next_b = atomicAdd(p.next_block, 1);
        __syncthreads();
        if (next_b >= p.s) break;
        const int b = p.block_order ? p.block_order[next_b] : next_b;
        const int o = p.bstart[b];
        const int d = p.bstart[b + 1] - o;
        if (d <= dlo || d > dhi) continue;
        const int T = (d + 31) / 32;
        const int dp4 = (d + 3) & ~3;
        float* F = p.fac + p.fac_off[b];
        // per-row CSR cursors (thread tid owns rows tid + NT i for the
        // gathers) + FP64 inf-norm, row sums in column order (matrix_inf_norm)
        int cur[RPT], ke[RPT];
        double rs = 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = tid + NT * i;
            cur[i] = ke[i] = 0;
            if (r < d) {
                const int kb = __ldg(p.a.rp + o + r);
                ke[i] = __ldg(p.a.rp + o + r + 1);
                cur[i] = ke[i];
                double rsum = 0.0;
                for (int k = kb; k < ke[i]; ++k) {
                    const int c = __ldg(p.a.ci + k) - o;
                    if (c >= 0 && c < d) {
                        if (cur[i] == ke[i]) cur[i] = k;
                        rsum = __dadd_rn(rsum, fabs(__ldg(p.a.val + k)));
                    } else if (c >= d) {
                        break;
                    }
                }
                rs = fmax(rs, rsum);
                act[r] = (short)r;
                ppos[r] = 0x7fff;
            }
        }
        double wm = rs;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) wm = fmax(wm, __shfl_xor_sync(0xffffffffu, wm, off));
        if (lane == 0) redd[wid] = wm;
        if (tid == 0) {
            int acc = 0;
            for (int q = 0; q + 1 < T; ++q) {
                lofs[q] = acc;
                acc += d - 32 * q;
            }
        }
        if (tid < 3) piv_best[tid] = 0ull;
        __syncthreads();
        double norm = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) norm = fmax(norm, redd[w]);
        const KeepBrackets kbr = keep_brackets(norm, p.eps);

        int na = d;
        int nperturb = 0;
        bool abort = false;
        int buf = 0;
        int pb = 0;  // piv_best slot of the next column (warps that drop out of the
                     // panel factorisation do not return before the next block)
        for (int P = 0; P < T; ++P) {
            unsigned long long tp0 = 0;
            if (p.prof && tid == 0) tp0 = clock64();
            const int c0 = 32 * P;
            const int kw = min(32, d - c0);
            // ---- gather the column panel (rows in original order)
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = tid + NT * i;
                if (r < d) {
                    float4* xr = reinterpret_cast<float4*>(X + r * kXld);
#pragma unroll
                    for (int q = 0; q < 8; ++q) xr[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                    const int cend = o + c0 + kw;
                    while (cur[i] < ke[i]) {
                        const int c = __ldg(p.a.ci + cur[i]);
                        if (c >= cend) break;
                        const int lc = c - o - c0;
                        X[xe(r, lc)] = __double2float_rn(__ldg(p.a.val + cur[i]));
                        ++cur[i];
                    }
                }
            }
            // the first two L11 blocks of this panel's left-looking updates
            if (tid == 0)
                for (int q = 0; q < min(P, 2); ++q)
                    bulk_load(L11 + q * 1024, Lg + (size_t)lofs[q] * 32, 4096u, &mbar[1 + q]);
            __syncthreads();
            // ---- left-looking updates from the earlier panels
            for (int Q = 0; Q <= P; ++Q) {
                const int q0 = 32 * Q;
                const short* prv = prow + (Q > 0 ? q0 - 32 : 0);  // U_{Q-1}: pivot rows of Q - 1
                const int nprev = Q > 0 ? d - (q0 - 32) : 0;       // rows of L_{Q-1}
                float u[32];  // this lane's column of U_{Q-1} (A_Q, B_Q and the final step)
                if (Q > 0) {
                    ll_load_u(u, X, prv, lane);
                    mbar_wait(&mbar[0], (nb_issue - 1) & 1u);  // Lb = rows 32.. of L_{Q-1}
                }
                if (Q == P) {  // (ii)_{P-1} on the rows still active
                    if (Q > 0) {
                        const short* rP = rowQ + lofs[Q - 1];
                        ll_rank32(X, Lb - 32 * 32, u, lane, 32 + wid, nprev, NW,
                                  [&](int a) { return make_int2(a, (int)rP[a]); });
                        __syncthreads();
                    }
                    break;
                }
                if (Q > 0) {  // A_Q: (ii)_{Q-1} on Q's pivot rows
                    const short* posp = posQ + (size_t)(Q - 1) * dhi;
                    ll_rank32(X, Lb - 32 * 32, u, lane, wid, 32, NW, [&](int i) {
                        const int r = prow[q0 + i];
                        return make_int2((int)posp[r], r);
                    });
                    __syncthreads();
                }
                if (wid == 0) {  // B_Q, warp 0: (i)_Q with L11 of Q
                    const int sb = Q & 1;
                    mbar_wait(&mbar[1 + sb], n11_issue[sb] & 1u);
                    const float* LQ = L11 + sb * 1024;
                    float x[32];
#pragma unroll
                    for (int m = 0; m < 32; ++m) x[m] = X[xe(prow[q0 + m], lane)];
                    ll_trsv<0>(x, LQ);
#pragma unroll
                    for (int m = 0; m < 32; ++m) X[xe(prow[q0 + m], lane)] = x[m];
                } else if (Q > 0) {  // B_Q, other warps: (ii)_{Q-1} on the rows active after Q
                    const short* rP = rowQ + lofs[Q - 1];
                    const int qhi = q0 + 32;
                    ll_rank32(X, Lb - 32 * 32, u, lane, 32 + (wid - 1), nprev, NW - 1, [&](int a) {
                        const int r = rP[a];
                        return make_int2(ppos[r] >= qhi ? a : -1, r);  // Q's pivot rows: done in A_Q
                    });
                }
                n11_issue[Q & 1] += 1;  // L11 buffer Q & 1 consumed (phase counted in every thread)
                __syncthreads();
                // Lb and L11 buffer (Q & 1) are free: fetch L_Q's rows 32.. and L11 of Q + 2
                if (tid == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const int nq = d - q0;
                    bulk_load(Lb, Lg + ((size_t)lofs[Q] + 32) * 32, (unsigned)(nq - 32) * 128u, &mbar[0]);
                    if (Q + 2 < P) bulk_load(L11 + (Q & 1) * 1024, Lg + (size_t)lofs[Q + 2] * 32, 4096u, &mbar[1 + (Q & 1)]);
                }
                nb_issue += 1;
            }
            // ---- factor the panel: thread a owns active rows act[a + NT i];
            unsigned long long tp1 = 0;
            if (p.prof && tid == 0) tp1 = clock64();
            // only the warps holding rows take part (named barrier 1). A
            // rolled column loop over a shifting register window (rv[j] =
            // column c + j) keeps the code small: the rank-1 update writes
            // rv[j - 1] = fmaf(-l, Pv[j], rv[j]); each column's final entry
            // goes to X as it is produced (a pivot row stores its U row)
            const int nwa = (min(na, NT) + 31) >> 5;
            if (wid < nwa) {
                bool fl[RPT];
                int myrow[RPT];
                float rv[RPT][32];
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int a = tid + NT * i;
                    const bool has = a < na;
                    myrow[i] = has ? act[a] : 0;
                    fl[i] = !has;
                    const float4* xr = reinterpret_cast<const float4*>(X + myrow[i] * kXld);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 t4 = has ? xr[q] : make_float4(0.f, 0.f, 0.f, 0.f);
                        rv[i][4 * q + 0] = t4.x;
                        rv[i][4 * q + 1] = t4.y;
                        rv[i][4 * q + 2] = t4.z;
                        rv[i][4 * q + 3] = t4.w;
                    }
                }
                // The window shrinks by 8 every 8 columns (W = 32, 24, 16, 8):
                // column c + j for j >= W is past the panel, so the rank-1
                // update and the candidate copy only cover W columns (the
                // same fmaf chain per element as a constant 32-wide window,
                // 39% fewer update instructions)
                auto run_cols = [&](auto Wc, int cb, int ce) -> bool {
                    constexpr int W = decltype(Wc)::value;
#pragma unroll 1
                        for (int c = cb; c < ce; ++c) {
                        const int k = c0 + c;
                        // thread candidate, then warp candidate: max |x|, ties -> smaller row
                        unsigned key = 0u;
                        int brow = 0x7fffffff, bi = 0;
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            const unsigned ki = fl[i] ? 0u : __float_as_uint(fabsf(rv[i][0])) + 1u;
                            if (ki > key || (ki == key && ki != 0u && myrow[i] < brow)) {
                                key = ki;
                                brow = myrow[i];
                                bi = i;
                            }
                        }
                        unsigned kmx;
                        const int wr = warp_pivot_row(key, key ? brow : 0x7fffffff, &kmx);
                        const unsigned own = __ballot_sync(0xffffffffu, key != 0u && key == kmx && brow == wr);
                        float* cv = cand_v + (size_t)(buf * NW + wid) * 32;
                        // each warp's candidate meets the others in one 64-bit shared
                        // atomic max: key, then the smaller row (0xFFFF - row), then
                        // the owning thread slot (unique per row)
                        if (own && lane == __ffs(own) - 1) {
#pragma unroll
                            for (int i = 0; i < RPT; ++i)
                                if (i == bi)
#pragma unroll
                                    for (int q = 0; q < W / 4; ++q)
                                        reinterpret_cast<float4*>(cv)[q] = make_float4(rv[i][4 * q], rv[i][4 * q + 1],
                                                                                       rv[i][4 * q + 2], rv[i][4 * q + 3]);
                            atomicMax(&piv_best[pb], ((unsigned long long)kmx << 32) |
                                                         ((unsigned long long)(0xFFFF - wr) << 16) |
                                                         (unsigned long long)(tid + NT * bi));
                        }
                        bar_named(1, nwa * 32);
                        const unsigned long long wv = piv_best[pb];
                        // the previous column's slot is read by now: clear it for the
                        // column after next (three slots)
                        if (tid == 0) piv_best[pb == 0 ? 2 : pb - 1] = 0ull;
                        pb = pb == 2 ? 0 : pb + 1;
                        const int frow = 0xFFFF - (int)((wv >> 16) & 0xFFFFu);
                        const int owner = (int)(wv & 0xFFFFu);  // tid + NT * row slot
                        const int fw = (owner % NT) >> 5;
                        const float4* Pv4 = reinterpret_cast<const float4*>(cand_v + (size_t)(buf * NW + fw) * 32);
                        buf ^= 1;
                        // regularize_pivot (lu.cpp:10-20), identical in every thread;
                        // FP32 brackets, FP64 only near the threshold or to regularise
                        const float praw = Pv4[0].x;
                        float pv = praw;
                        if (!pivot_keep_f(praw, kbr, norm, p.eps)) {
                            const double pvd = (double)praw;
                            const double val = (pvd < 0.0 ? -1.0 : 1.0) * p.eps * norm;
                            if (val == 0.0) {
                                if (tid == 0) atomicMin(p.singular, ((unsigned long long)b << 32) | (unsigned)k);
                                return true;
                            }
                            ++nperturb;
                            if (tid == 0) {
                                const int slot = atomicAdd(p.pert_n, 1);
                                if (slot < p.pert_cap) p.pert[slot] = PertRecord{b, k, pvd, val};
                            }
                            pv = (float)val;
                        } else if (praw == 0.0f) {  // kept zero pivot (eps = 0)
                            if (tid == 0) atomicMin(p.singular, ((unsigned long long)b << 32) | (unsigned)k);
                            return true;
                        }
                        if (wid == 0 && c + lane < 32)  // the pivot row's U row (columns c..31) is final
                            X[xe(frow, c + lane)] = lane == 0 ? pv : reinterpret_cast<const float*>(Pv4)[lane];
#pragma unroll
                        for (int i = 0; i < RPT; ++i) {
                            if (owner == tid + NT * i) {  // the pivot row (its U row goes to X below)
                                fl[i] = true;
                                prow[k] = (short)myrow[i];
                                ppos[myrow[i]] = (short)k;
                            } else if (!fl[i]) {
                                const float l = div_mult(rv[i][0], pv);  // L(i,k) = x_i / pivot (lu.cpp:207)
                                X[xe(myrow[i], c)] = l;
                                // the pivot row's window quad by quad from the candidate
                                // slot (not held in registers: 128 per thread)
                                {
                                    const float4 w0 = Pv4[0];
                                    rv[i][0] = fmaf(-l, w0.y, rv[i][1]);
                                    rv[i][1] = fmaf(-l, w0.z, rv[i][2]);
                                    rv[i][2] = fmaf(-l, w0.w, rv[i][3]);
                                }
#pragma unroll
                                for (int q = 1; q < W / 4; ++q) {
                                    const float4 wq = Pv4[q];
                                    rv[i][4 * q - 1] = fmaf(-l, wq.x, rv[i][4 * q]);
                                    rv[i][4 * q + 0] = fmaf(-l, wq.y, rv[i][4 * q + 1]);
                                    rv[i][4 * q + 1] = fmaf(-l, wq.z, rv[i][4 * q + 2]);
                                    rv[i][4 * q + 2] = fmaf(-l, wq.w, rv[i][4 * q + 3]);
                                }
                            }
                        }
                    }
                    return false;
                };
                bool ab = run_cols(IntC<32>{}, 0, min(kw, 8));
                if (!ab && kw > 8) ab = run_cols(IntC<24>{}, 8, min(kw, 16));
                if (!ab && kw > 16) ab = run_cols(IntC<16>{}, 16, min(kw, 24));
                if (!ab && kw > 24) ab = run_cols(IntC<8>{}, 24, kw);
                abort = ab;
            }
            abort = __syncthreads_or(abort);
            if (abort) break;
            // ---- compact the active list (stable); L_P to the scratch: the 32
            if (p.prof && tid == 0) { const unsigned long long t2 = clock64(); atomicAdd(p.prof + 0, tp1 - tp0); atomicAdd(p.prof + 1, t2 - tp1); tp0 = t2; }
            // pivot rows first, in pivot order, then the rows still active
            if (wid == 0) {
                int w = 0;
                for (int base = 0; base < na; base += 32) {
                    const int a = base + lane;
                    const int r = a < na ? act[a] : 0;
                    const bool keepr = a < na && ppos[r] == 0x7fff;
                    const unsigned m = __ballot_sync(0xffffffffu, keepr);
                    __syncwarp();
                    if (keepr) act[w + __popc(m & ((1u << lane) - 1u))] = (short)r;
                    w += __popc(m);
                    __syncwarp();
                }
                if (lane == 0) nact_sh = w;
            }
            __syncthreads();
            const int nnew = nact_sh;
            if (P + 1 < T) {
                const int lo = lofs[P];
                for (int i = tid; i < 32 + nnew; i += NT) {
                    const int r = i < 32 ? prow[c0 + i] : act[i - 32];
                    const float4* xr = reinterpret_cast<const float4*>(X + r * kXld);
                    float4* lr = reinterpret_cast<float4*>(Lg + ((size_t)lo + i) * 32);
#pragma unroll
                    for (int q = 0; q < 8; ++q) lr[q] = xr[q];
                    rowQ[lo + i] = (short)r;
                    posQ[(size_t)P * dhi + r] = (short)i;
                }
                // the scratch rows are read back by the async proxy (bulk copies)
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            // ---- output: chunks (t, P) for t <= P (U / L11\U11 from X) and
            // (P, Q) for Q < P (the new pivot rows' L from L_Q); chunk (t, u)
            // = rows 32t.. of panel t, quads 8u .. 8u + nq(u), [quad][row][4]
            {
                const int nqP = min(8, dp4 / 4 - 8 * P);
                for (int e = tid; e < (P + 1) * 8 * 32; e += NT) {  // (t, P)
                    const int t = e >> 8, qi = (e >> 5) & 7, kr = e & 31;
                    if (qi >= nqP) continue;
                    const int k = 32 * t + kr;
                    const int cq = 4 * (8 * P + qi);
                    float4 v;
                    if (k < d) {
                        v = *reinterpret_cast<const float4*>(X + xq(prow[k], qi));
                        if (cq + 0 >= d) v.x = 0.f;
                        if (cq + 1 >= d) v.y = 0.f;
                        if (cq + 2 >= d) v.z = 0.f;
                        if (cq + 3 >= d) v.w = 0.f;
                    } else {
                        v = make_float4(k == cq ? 1.f : 0.f, k == cq + 1 ? 1.f : 0.f, k == cq + 2 ? 1.f : 0.f,
                                        k == cq + 3 ? 1.f : 0.f);
                    }
                    __stcs(reinterpret_cast<float4*>(F + (size_t)t * 32 * dp4 + (size_t)(8 * P + qi) * 128 + kr * 4),
                           v);
                }
                for (int e = tid; e < P * 8 * 32; e += NT) {  // (P, Q), Q < P
                    const int Q = e >> 8, qi = (e >> 5) & 7, kr = e & 31;
                    const int k = c0 + kr;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (k < d)
                        v = __ldcg(reinterpret_cast<const float4*>(
                            Lg + ((size_t)lofs[Q] + posQ[(size_t)Q * dhi + prow[k]]) * 32 + 4 * qi));
                    __stcs(reinterpret_cast<float4*>(F + (size_t)P * 32 * dp4 + (size_t)(8 * Q + qi) * 128 + kr * 4),
                           v);
                }
            }
            na = nnew;
            __syncthreads();
            if (p.prof && tid == 0) atomicAdd(p.prof + 2, clock64() - tp0);
        }
        if (tid == 0) p.pert_count[b] = nperturb;
        if (!abort)
            for (int k = tid; k < d; k += NT) p.piv[o + k] = prow[k];
        __syncthreads();
    }
}

int lu_smem_dim(int dmax) {
    int d = 1;
    while (d + 1 <= dmax && (size_t)(d + 1) * ((d + 1) | 1) * sizeof(float) <= kLuSmemTile) ++d;
    return d;
}

}  // namespace

// resident CTAs per SM of the blocked kernel (registers and shared memory):
// the grid is exactly one wave, and the scratch holds one tile per CTA
// (one instance per size range: one panel row per thread up to 256, two above)
using BlkFn = void (*)(LuParams, int, int, int);
BlkFn blk_fn(int dhi) { return dhi <= kBlkThreads ? k_block_lu_blk<kBlkThreads, 1> : k_block_lu_blk<kBlkThreads, 2>; }

int blk_ctas_per_sm(int dhi) {
    const size_t smem = blk_smem_bytes(dhi);
    const BlkFn fn = blk_fn(dhi);
    HPBJ_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    HPBJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kBlkThreads, smem));
    return std::max(occ, 1);
}

size_t block_lu_scratch_floats(int dmax, int num_sms, int* smem_dim, int* scratch_ld) {
    *smem_dim = lu_smem_dim(dmax);
    *scratch_ld = blk_ld(dmax | 1);  // odd-free 16-byte rows for the blocked kernel, >= dmax | 1
    size_t need = 0;
    const char* e = getenv("HPBJ_LU_LL");
    const bool ll = !(e && e[0] == '0');
    if (ll && dmax > kWarpLuMax)  // left-looking kernel: L_Q rows of one block per CTA
        need = (size_t)num_sms * kLlCtasPerSm * ll_lrows(std::min(dmax, kLlMax)) * 32;
    if (dmax > kWarpLuMax && (!ll || dmax > kLlMax)) {  // blocked kernels: one tile per resident CTA
        const int d1 = std::min(dmax, kBlkThreads);
        need = std::max(need, (size_t)num_sms * blk_ctas_per_sm(d1) * (*scratch_ld) * (*scratch_ld));
        if (dmax > kBlkThreads)
            need = std::max(need, (size_t)num_sms * blk_ctas_per_sm(std::min(dmax, kBlkMax)) * (*scratch_ld) *
                                      (*scratch_ld));
    }
    if (dmax > kBlkMax && dmax > *smem_dim)
        need = std::max(need, (size_t)num_sms * 4 * (*scratch_ld) * (*scratch_ld));
    return need;
}

void launch_block_lu(const LuParams& p_in, int dmax, int num_sms, cudaStream_t st, int64_t* launches) {
    if (dmax > kLuMaxDim) fail(HPBJ_EINVAL, "block_jacobi: block dimension exceeds 2048");
    LuParams p = p_in;
    // blocks up to kWarpLuMax: one warp each, tile in shared memory
    const int dw = std::min(dmax, kWarpLuMax);
    p.warp_dim = dw;
    {
        const int ldw = dw | 1;
        const size_t per_block = ((size_t)dw * ldw + dw) * sizeof(float);
        const char* e = getenv("HPBJ_LU_WARP");
        if (e && e[0] == '1') {  // one warp per block (k_block_lu_warp)
            const int wpc = (int)std::max<size_t>(1, std::min<size_t>(2, (200 * 1024) / per_block));
            const size_t smem = per_block * wpc;
            void (*fn)(LuParams, int, int) = nullptr;
            switch ((dw + 31) / 32) {
                case 1: fn = k_block_lu_warp<1>; break;
                case 2: fn = k_block_lu_warp<2>; break;
                default: fn = k_block_lu_warp<3>; break;
            }
            HPBJ_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int occ = 0;
            HPBJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * wpc, smem));
            occ = std::max(occ, 1);
            const int grid = std::max(1, std::min((p.s + wpc - 1) / wpc, num_sms * occ));
            fn<<<grid, 32 * wpc, smem, st>>>(p, dw, ldw);
        } else {  // two warps per block (k_block_lu_pair)
            void (*fn)(LuParams, int, int) = nullptr;
            switch ((dw + 31) / 32) {
                case 1: fn = k_block_lu_pair<1>; break;
                case 2: fn = k_block_lu_pair<2>; break;
                default: fn = k_block_lu_pair<3>; break;
            }
            HPBJ_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per_block));
            int occ = 0;
            HPBJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 64, per_block));
            occ = std::max(occ, 1);
            const int grid = std::max(1, std::min(p.s, num_sms * occ));
            fn<<<grid, 64, per_block, st>>>(p, dw, ldw);
        }
        *launches += 1;
    }
    if (dmax <= dw) {
        HPBJ_CUDA(cudaGetLastError());
        return;
    }
    // left-looking kernel for dw < d <= kLlMax (HPBJ_LU_LL=0: the L2-scratch
    // blocked kernel instead, for A/B runs and the bit-identity test)
    int dll = dw;
    {
        const char* e = getenv("HPBJ_LU_LL");
        if (!(e && e[0] == '0')) {
            // two row slots per thread for every size: measured faster than a
            // one-slot instance for d <= 256 too (config 2: 5.5 vs 7.6 ms,
            // config 3: 30.7 vs 44.4 ms with a separate one-slot launch)
            const int dhi = std::min(dmax, kLlMax);
            const size_t smem = ll_smem_bytes(dhi);
            void (*fn)(LuParams, int, int) = k_block_lu_ll<2>;
            HPBJ_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            const int grid = std::min(p.s, num_sms * kLlCtasPerSm);
            HPBJ_CUDA(cudaMemsetAsync(p.next_block, 0, sizeof(int), st));
            fn<<<grid, kLlThreads, smem, st>>>(p, dw, dhi);
            *launches += 1;
            dll = dhi;
        }
    }
    if (dmax <= dll) {
        HPBJ_CUDA(cudaGetLastError());
        return;
    }
    // blocked kernels for dll < d <= 256 and 256 < d <= kBlkMax
    for (int range = 0; range < 2; ++range) {
        const int dlo = std::max(dll, range == 0 ? dw : kBlkThreads);
        const int dhi = std::min(dmax, range == 0 ? kBlkThreads : kBlkMax);
        if (dhi <= dlo) continue;
        const size_t smem = blk_smem_bytes(dhi);
        const int grid = std::min(p.s, num_sms * blk_ctas_per_sm(dhi));  // sets the smem attribute
        blk_fn(dhi)<<<grid, kBlkThreads, smem, st>>>(p, dlo, dhi, p.scratch_ld);
        *launches += 1;
    }
    if (dmax <= kBlkMax) {
        HPBJ_CUDA(cudaGetLastError());
        return;
    }
    p.warp_dim = kBlkMax;  // the column-by-column kernels take only d > kBlkMax
    const int sd = p.smem_dim;
    const int dsm = std::min(dmax, sd);
    const size_t smem = (size_t)dsm * (dsm | 1) * sizeof(float);
    HPBJ_CUDA(cudaFuncSetAttribute(k_block_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLuSmemTile));
    int occ = 0;
    HPBJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_block_lu, kLuThreads, smem));
    occ = std::max(occ, 1);
    if (sd > kBlkMax) {
        const int grid0 = std::min(p.s, num_sms * occ);
        k_block_lu<<<grid0, kLuThreads, smem, st>>>(p, 0);
        *launches += 1;
    }
    if (dmax > sd) {
        const int grid1 = std::min(p.s, num_sms * 4);
        k_block_lu<<<grid1, kLuThreads, 0, st>>>(p, 1);
        *launches += 1;
    }
    HPBJ_CUDA(cudaGetLastError());
}

}  // namespace hpbj
