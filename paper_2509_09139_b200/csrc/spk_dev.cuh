// Device side of the sparse-panel block-Jacobi apply (spk.cu): the per-block
// substitution as a warp-level device function, shared by the standalone
// apply kernels (spk.cu) and the fused Arnoldi-cycle kernel (fused.cu).
#pragma once

#include <cstdint>
#include <type_traits>

#include "device.cuh"
#include "kernels.cuh"

namespace hpbj {
namespace spk {

constexpr int kMaxPanels = 9;  // pivots of up to 288 rows gathered with full ILP

// ----------------------------------------------------------------------------
// L2 prefetch of the 8-byte rows [o, o + d) of v (a block's source rows:
// pivoting permutes only within the block); warp-wide.
__device__ __forceinline__ void prefetch_rows_l2(const double* v, int o, int d, int lane) {
    const uintptr_t a = (uintptr_t)(v + o) & ~(uintptr_t)127;
    const uintptr_t e = (uintptr_t)(v + o + d);
    for (uintptr_t l = a + ((uintptr_t)lane << 7); l < e; l += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(l));
}
struct SrcDown {  // (float) V[:, st->j][row]  (Arnoldi step)
    const double* V;
    int ldv;
    const SolveState* sst;
    __device__ float operator()(int row) const { return __double2float_rn(__ldg(V + (size_t)sst->j * ldv + row)); }
    __device__ void prefetch(int o, int d, int lane) const { prefetch_rows_l2(V + (size_t)sst->j * ldv, o, d, lane); }
};
struct SrcVec {  // (float) v[row]
    const double* v;
    __device__ float operator()(int row) const { return __double2float_rn(__ldg(v + row)); }
    __device__ void prefetch(int o, int d, int lane) const { prefetch_rows_l2(v, o, d, lane); }
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
    __device__ void prefetch(int, int, int) const {}
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

// Four consecutive Acc of a 16-byte aligned shared-memory row as one load.
template <class Acc>
struct Vec4 {
    Acc x, y, z, w;
};
__device__ __forceinline__ Vec4<float> ld_vec4(const float* p) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ Vec4<double> ld_vec4(const double* p) {
    const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
    return {a.x, a.y, b.x, b.y};
}

template <class IdxT>
struct Idx4;
template <>
struct Idx4<uint16_t> {
    using type = ushort4;
};
template <>
struct Idx4<uint32_t> {
    using type = uint4;
};

// acc[row] -= sum val * x[col] over the row-sorted entries [e0, e0 + cnt)
// (e0 16-byte aligned), branch-free. Each lane takes four consecutive
// entries (one float4 + one 4-index load) and forms their inclusive
// segmented sums q_k (runs of equal rows); the run that crosses lane
// boundaries is completed by a segmented warp scan of the lanes' tail sums,
// whose carry is added to the lane's head run; the last entry of every row
// segment flushes into acc. Fixed association: deterministic.
template <class Acc, class IdxT>
__device__ __forceinline__ void fold_entries(const float* __restrict__ eval, const IdxT* __restrict__ eidx, int e0,
                                             int cnt, const Acc* xs, Acc* acc, int lane) {
    using I4 = typename Idx4<IdxT>::type;
    const float4* ev = reinterpret_cast<const float4*>(eval + e0);
    const I4* ei = reinterpret_cast<const I4*>(eidx + e0);
    for (int base = 0; base < cnt; base += 128) {
        const int i0 = base + 4 * lane;
        const int nv = cnt - i0;  // valid entries of this lane (<= 0: none, >= 4: all four)
        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
        I4 x4{};
        if (nv > 0) {  // padding entries inside the last quad are (0, col 0)
            v4 = __ldg(ev + (i0 >> 2));
            x4 = __ldg(ei + (i0 >> 2));
        }
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
        const unsigned xi[4] = {(unsigned)x4.x, (unsigned)x4.y, (unsigned)x4.z, (unsigned)x4.w};
        int r[4];
        Acc q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = k < nv ? (int)(xi[k] & 31u) : 32 + 4 * lane + k;  // invalid: unique, never flushed
        q[0] = (Acc)v[0] * xs[xi[0] >> 5];
#pragma unroll
        for (int k = 1; k < 4; ++k) {
            const Acc xk = xs[xi[k] >> 5];
            q[k] = (r[k] == r[k - 1]) ? fma((Acc)v[k], xk, q[k - 1]) : (Acc)v[k] * xk;
        }
        const int prev_tail = __shfl_up_sync(0xffffffffu, r[3], 1);
        const int next_head = __shfl_down_sync(0xffffffffu, r[0], 1);
        const bool cont = lane > 0 && r[0] == prev_tail;  // head run continues the lower lane's tail run
        const bool start = !(cont && r[3] == r[0]);
        const unsigned heads = __ballot_sync(0xffffffffu, start);
        const int dist = lane - (31 - __clz(heads & (0xffffffffu >> (31 - lane))));
        const int maxd = __reduce_max_sync(0xffffffffu, dist);
        Acc run = q[3];
        for (int off = 1; off <= maxd; off <<= 1) {
            const Acc t = __shfl_up_sync(0xffffffffu, run, off);
            if (off <= dist) run += t;
        }
        const Acc up = __shfl_up_sync(0xffffffffu, run, 1);
        const Acc carry = cont ? up : (Acc)0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool end = (k < 3) ? (r[k] != r[k + 1]) : (lane == 31 || next_head != r[3]);
            if (end && r[k] < 32) acc[r[k]] -= (r[k] == r[0]) ? q[k] + carry : q[k];
        }
        __syncwarp();
    }
}

// Row-quad layout (spk.cu pack_row_quads): lane r takes the rank-r row of
// the part (meta = row | quads << 5, ranks ordered by quads desc), and reads
// its quad i at quad slot S(i) + r, where S(i) counts the quads of the slots
// before i (the active lanes of slot i are a prefix: one coalesced float4 +
// index-quad load per slot). Each lane accumulates its row sequentially in
// column order; acc[row] -= sum. No cross-lane traffic but one ballot per slot.
template <class Acc, class IdxT>
__device__ __forceinline__ void fold_rows(const float* __restrict__ eval, const IdxT* __restrict__ eidx, int e0,
                                          int mq, unsigned meta, const Acc* xs, Acc* acc, int lane) {
    using I4 = typename Idx4<IdxT>::type;
    const float4* ev = reinterpret_cast<const float4*>(eval + e0);
    const I4* ei = reinterpret_cast<const I4*>(eidx + e0);
    const int q = (int)(meta >> 5);
    Acc a = (Acc)0;
    int S = lane;
    int i = 0;
    for (; i + 1 < mq; i += 2) {  // two slots' loads in flight
        const unsigned act0 = __ballot_sync(0xffffffffu, i < q);
        const int S1 = S + __popc(act0);
        float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
        I4 x0{}, x1{};
        if (i < q) {
            v0 = __ldg(ev + S);
            x0 = __ldg(ei + S);
        }
        if (i + 1 < q) {
            v1 = __ldg(ev + S1);
            x1 = __ldg(ei + S1);
        }
        S = S1 + __popc(__ballot_sync(0xffffffffu, i + 1 < q));
        a = fma((Acc)v0.x, xs[x0.x], a);
        a = fma((Acc)v0.y, xs[x0.y], a);
        a = fma((Acc)v0.z, xs[x0.z], a);
        a = fma((Acc)v0.w, xs[x0.w], a);
        a = fma((Acc)v1.x, xs[x1.x], a);
        a = fma((Acc)v1.y, xs[x1.y], a);
        a = fma((Acc)v1.z, xs[x1.z], a);
        a = fma((Acc)v1.w, xs[x1.w], a);
    }
    if (i < mq && i < q) {
        const float4 v0 = __ldg(ev + S);
        const I4 x0 = __ldg(ei + S);
        a = fma((Acc)v0.x, xs[x0.x], a);
        a = fma((Acc)v0.y, xs[x0.y], a);
        a = fma((Acc)v0.z, xs[x0.z], a);
        a = fma((Acc)v0.w, xs[x0.w], a);
    }
    __syncwarp();
    if (q > 0) acc[meta & 31u] -= a;
    __syncwarp();
}

// L2 prefetches of the next step's data, issued by the whole warp: one
// 128-byte line per lane and instruction (prefetch.global.L2 — no registers,
// no shared memory, no completion to wait for). A bulk prefetch
// (cp.async.bulk.prefetch.L2) takes its address in a uniform register, so
// issued by lane-dependent ranges it compiles to a serialised R2UR loop over
// the active lanes (ncu, config 3: 17% of the apply's instructions).
__device__ __forceinline__ void pf_line(const void* a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); }

// [p0, p0 + b0) and [p1, p1 + b1), lines spread over the lanes
__device__ __forceinline__ void warp_prefetch_l2(const void* p0, size_t b0, const void* p1, size_t b1, int lane) {
    const uintptr_t a0 = (uintptr_t)p0 & ~(uintptr_t)127, a1 = (uintptr_t)p1 & ~(uintptr_t)127;
    const int n0 = b0 ? (int)(((uintptr_t)p0 + b0 - a0 + 127) >> 7) : 0;
    const int n1 = b1 ? (int)(((uintptr_t)p1 + b1 - a1 + 127) >> 7) : 0;
    for (int k = lane; k < n0 + n1; k += 32) pf_line((const void*)(k < n0 ? a0 + ((uintptr_t)k << 7) : a1 + ((uintptr_t)(k - n0) << 7)));
}
__device__ __forceinline__ void warp_prefetch_l2(const void* p0, size_t b0, int lane) {
    warp_prefetch_l2(p0, b0, nullptr, 0, lane);
}

// 16-byte asynchronous global -> shared copy (LDGSTS), L2 only.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// The tile quads a pass reads ([quad][lane] float4, see kernels.cuh): the
// forward pass quad q for lanes l >= 4q, the backward pass quad q < 8 for
// lanes l < 4q and all of quad 8. Each quad is 4 lines of 8 lanes; lane
// k (+32) takes line k & 3 of quad k >> 2 when the pass reads any of it.
// full: the block's last panel ((L U)^-1, quads 0..ceil(rows/4)-1 of its
// first `rows` lanes — the rest is the identity padding, never read).
__device__ __forceinline__ void prefetch_tile(const SpkView& p, int P, bool fwd, int lane, bool full = false,
                                              int rows = 32) {
    if (!p.pf) return;
    const char* t = reinterpret_cast<const char*>(p.dtile + (size_t)P * kTileFloats);
    for (int k = lane; k < 36; k += 32) {
        const int q = k >> 2, li = k & 3;
        int l0 = 0, l1 = 32;
        if (q == 8) l1 = (fwd || full) ? 0 : 32;
        else if (full) l1 = 4 * q < rows ? rows : 0;
        else if (fwd) l0 = 4 * q;
        else l1 = 4 * q;
        if (8 * li < l1 && 8 * li + 8 > l0) pf_line(t + q * 512 + li * 128);
    }
}

// values and indices of `cnt` entries from e0 (warp-wide)
template <class IdxT>
__device__ __forceinline__ void prefetch_entries(const SpkView& p, int e0, int cnt, int lane) {
    if (!p.pf) return;
    warp_prefetch_l2(p.eval + e0, sizeof(float) * cnt, reinterpret_cast<const IdxT*>(p.eidx) + e0,
                     sizeof(IdxT) * cnt, lane);
}

// Next block's head: descriptors, row metadata, pivots and its first
// panel's forward data (warp-wide).
template <class IdxT>
__device__ __forceinline__ void prefetch_block_head(const SpkView& p, int b, int lane) {
    if (!p.pf) return;
    const int P0 = p.pstart[b], T = p.pstart[b + 1] - P0;
    const int o = p.bstart[b], d = p.bstart[b + 1] - o;
    const int e0 = p.ent_off[P0], e1 = p.ent_off[P0 + 1];
    warp_prefetch_l2(p.desc + P0, sizeof(SpkPanel) * T, p.piv + o, sizeof(int) * d, lane);
    if (p.rows) warp_prefetch_l2(p.rmeta + (size_t)P0 * 64, 128 * (size_t)T, lane);
    prefetch_entries<IdxT>(p, e0, e1 - e0, lane);
    prefetch_tile(p, P0, true, lane, T == 1, d);
}

// One block's substitution M_b^-1: gather rhs[piv] from src, forward with
// the unit-lower factor, backward with the upper one, write through dst.
// ybuf (Acc[32 T]) and dsh (SpkPanel[T]) are the calling warp's shared
// memory; next_b (or -1) is the block whose head is prefetched at the end.
// tbuf (optional, 8 x 32 float4 of the warp's shared memory): the step's
// tile quads are copied there asynchronously at the start of the step, so
// their latency overlaps the off-panel fold.
// ROWS: off-panel parts in the row-quad layout (fold_rows); msh (uint16
// [64 T] of the warp's shared memory) receives the block's row metadata.
// CACHED: a warp that applies the same block every step (fused cycle
// kernel) keeps the block's header, descriptors, row metadata and pivots in
// its shared memory (spk_cache_block): two dependent global loads less.
struct BlockCache {
    int4 hdr;  // o, d, T, P0
    int piv[1];  // d entries (the warp's buffer is sized for dmax)
};

template <bool ROWS>
__device__ __forceinline__ void spk_cache_block(const SpkView& p, int b, SpkPanel* dsh, uint16_t* msh, BlockCache* bc,
                                                int lane) {
    const int o = p.bstart[b], d = p.bstart[b + 1] - o, P0 = p.pstart[b];
    const int T = (d + 31) >> 5;
    if (lane < T) dsh[lane] = p.desc[P0 + lane];
    if (ROWS) {
        const uint32_t* m32 = reinterpret_cast<const uint32_t*>(p.rmeta + (size_t)P0 * 64);
        uint32_t* s32 = reinterpret_cast<uint32_t*>(msh);
        for (int t = 0; t < T; ++t) s32[t * 32 + lane] = __ldg(m32 + t * 32 + lane);
    }
    for (int k = lane; k < d; k += 32) bc->piv[k] = __ldg(p.piv + o + k);
    if (lane == 0) bc->hdr = make_int4(o, d, T, P0);
    __syncwarp();
}

template <class Acc, class IdxT, bool STAGE = false, bool ROWS = false, bool CACHED = false, class Src, class Dst>
__device__ __forceinline__ void spk_solve_block(const SpkView& p, int b, int next_b, Src src, Dst dst, Acc* ybuf,
                                                SpkPanel* dsh, int lane, float4* tbuf = nullptr,
                                                uint16_t* msh = nullptr, const BlockCache* bc = nullptr) {
    constexpr int kQMask = (1 << kRowQuadBits) - 1;
    const IdxT* eidx = reinterpret_cast<const IdxT*>(p.eidx);
    int o, d, P0;
    if (CACHED) {  // header, descriptors, metadata and pivots already on chip
        const int4 h = bc->hdr;
        o = h.x;
        d = h.y;
        P0 = h.w;
    } else {
        o = p.bstart[b];
        d = p.bstart[b + 1] - o;
        P0 = p.pstart[b];
    }
    const int T = (d + 31) >> 5;
    const int qd = lane >> 2;
    if (!CACHED) {
        if (lane < T) dsh[lane] = p.desc[P0 + lane];
        if (ROWS) {
            const uint32_t* m32 = reinterpret_cast<const uint32_t*>(p.rmeta + (size_t)P0 * 64);
            uint32_t* s32 = reinterpret_cast<uint32_t*>(msh);
            for (int t = 0; t < T; ++t) s32[t * 32 + lane] = __ldg(m32 + t * 32 + lane);
        }
        __syncwarp();
    }
    // rhs[pivot_rows[k]] for the whole block: all pivot loads first, then
    // all gathers (two latency rounds, not 2T)
    {
        int pv[kMaxPanels];
#pragma unroll
        for (int t = 0; t < kMaxPanels; ++t) {
            const int k = 32 * t + lane;
            pv[t] = (t < T && k < d) ? (CACHED ? bc->piv[k] : __ldg(p.piv + o + k)) : -1;
        }
#pragma unroll
        for (int t = 0; t < kMaxPanels; ++t)
            if (t < T) ybuf[32 * t + lane] = pv[t] >= 0 ? (Acc)src(o + pv[t]) : (Acc)0;
        for (int t = kMaxPanels; t < T; ++t) {
            const int k = 32 * t + lane;
            ybuf[k] = (k < d) ? (Acc)src(o + (CACHED ? bc->piv[k] : __ldg(p.piv + o + k))) : (Acc)0;
        }
    }
    __syncwarp();
    // ---- forward: y_k = rhs_k - sum_{c<k} L_kc y_c. The last panel's tile
    // is Uinv Linv (8 full quads, spk.cu): its forward and backward solves
    // are one mat-vec, peeled out of the loop (no extra live registers).
    auto fwd_step = [&](int t, auto last_c) {
        constexpr bool lastp = decltype(last_c)::value;
        const SpkPanel ds = dsh[t];
        // next step's data into L2 while this one computes
        if (!lastp) {
            const int nl1 = dsh[t + 1].nl;
            prefetch_entries<IdxT>(p, dsh[t + 1].off, ROWS ? 4 * (nl1 >> kRowQuadBits) : nl1, lane);
            prefetch_tile(p, P0 + t + 1, true, lane, t + 2 == T, d - 32 * (t + 1));
        } else if (T >= 2) {  // the backward pass starts at panel T-2
            const int nu1 = dsh[T - 2].nu;
            prefetch_entries<IdxT>(p, dsh[T - 2].uoff, ROWS ? 4 * (nu1 >> kRowQuadBits) : nu1, lane);
            prefetch_tile(p, P0 + T - 2, false, lane);
        } else if (next_b >= 0) {
            prefetch_block_head<IdxT>(p, next_b, lane);
            if (p.pf) src.prefetch(p.bstart[next_b], p.bstart[next_b + 1] - p.bstart[next_b], lane);
        }
        const float4* tile_f = reinterpret_cast<const float4*>(p.dtile + (size_t)(P0 + t) * kTileFloats);
        if (STAGE) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (lastp ? (32 * t + lane < d && 4 * q < d - 32 * t) : q <= qd)
                    cp_async16(tbuf + q * 32 + lane, tile_f + q * 32 + lane);
            cp_async_commit();
        }
        if (ROWS)
            fold_rows<Acc, IdxT>(p.eval, eidx, ds.off, ds.nl & kQMask, msh[64 * t + lane], ybuf, ybuf + 32 * t, lane);
        else
            fold_entries<Acc, IdxT>(p.eval, eidx, ds.off, ds.nl, ybuf, ybuf + 32 * t, lane);
        // y_t = Linv_tt r_t: quads 0..qd of row `lane` (zeros from the diagonal
        // on, unit diagonal implied); last panel: x_t = (Uinv Linv)_tt r_t
        float4 f4[8];
        if (STAGE) cp_async_wait_all();  // each lane reads back only the quads it copied
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            f4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            const bool need = lastp ? (32 * t + lane < d && 4 * q < d - 32 * t) : q <= qd;
            if (need) f4[q] = STAGE ? tbuf[q * 32 + lane] : __ldg(tile_f + q * 32 + lane);
        }
        const Acc* r = ybuf + 32 * t;
        Acc a0 = lastp ? (Acc)0 : r[lane], a1 = (Acc)0, a2 = (Acc)0, a3 = (Acc)0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const Vec4<Acc> rq = ld_vec4(r + 4 * q);  // broadcast: one LDS.128 for four columns
            a0 = fma((Acc)f4[q].x, rq.x, a0);
            a1 = fma((Acc)f4[q].y, rq.y, a1);
            a2 = fma((Acc)f4[q].z, rq.z, a2);
            a3 = fma((Acc)f4[q].w, rq.w, a3);
        }
        const Acc yv = (a0 + a1) + (a2 + a3);
        __syncwarp();
        ybuf[32 * t + lane] = yv;
        __syncwarp();
        if (lastp && 32 * t + lane < d) dst(o + 32 * t + lane, yv);
    };
    for (int t = 0; t + 1 < T; ++t) fwd_step(t, std::false_type{});
    fwd_step(T - 1, std::true_type{});
    // ---- backward: x_k = (y_k - sum_{c>k} U_kc x_c) / U_kk
    for (int t = T - 2; t >= 0; --t) {
        const SpkPanel ds = dsh[t];
        if (t > 0) {
            const int nu1 = dsh[t - 1].nu;
            prefetch_entries<IdxT>(p, dsh[t - 1].uoff, ROWS ? 4 * (nu1 >> kRowQuadBits) : nu1, lane);
            prefetch_tile(p, P0 + t - 1, false, lane);
        } else if (next_b >= 0) {
            prefetch_block_head<IdxT>(p, next_b, lane);
            if (p.pf) src.prefetch(p.bstart[next_b], p.bstart[next_b + 1] - p.bstart[next_b], lane);
        }
        const float4* tile_b = reinterpret_cast<const float4*>(p.dtile + (size_t)(P0 + t) * kTileFloats);
        if (STAGE) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q >= qd) cp_async16(tbuf + q * 32 + lane, tile_b + (q == qd ? 8 : q) * 32 + lane);
            cp_async_commit();
        }
        if (ROWS)
            fold_rows<Acc, IdxT>(p.eval, eidx, ds.uoff, ds.nu & kQMask, msh[64 * t + 32 + lane], ybuf, ybuf + 32 * t,
                                 lane);
        else
            fold_entries<Acc, IdxT>(p.eval, eidx, ds.uoff, ds.nu, ybuf, ybuf + 32 * t, lane);
        // x_t = Uinv_tt y'_t: quad 8 (the diagonal quad) and quads qd+1..7 of row `lane`
        const int k = 32 * t + lane;
        {
            float4 f4[8];
            if (STAGE) cp_async_wait_all();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                f4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (q >= qd) f4[q] = STAGE ? tbuf[q * 32 + lane] : __ldg(tile_b + (q == qd ? 8 : q) * 32 + lane);
            }
            const Acc* r = ybuf + 32 * t;
            Acc a0 = (Acc)0, a1 = (Acc)0, a2 = (Acc)0, a3 = (Acc)0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const Vec4<Acc> rq = ld_vec4(r + 4 * q);
                a0 = fma((Acc)f4[q].x, rq.x, a0);
                a1 = fma((Acc)f4[q].y, rq.y, a1);
                a2 = fma((Acc)f4[q].z, rq.z, a2);
                a3 = fma((Acc)f4[q].w, rq.w, a3);
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

}  // namespace spk
}  // namespace hpbj
