// Launch wrappers of the sm_100a kernels (one .cu per kernel family).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"

namespace hpbj {

constexpr int kShortRow = 32;             // rows sorted in registers by one thread
constexpr size_t kSmemSortMax = 128 * 1024;

// CSR on the device: int32 indices (nnz < 2^31), FP64 values.
struct DevCsr {
    int n = 0;
    int nnz = 0;
    int* rp = nullptr;
    int* ci = nullptr;
    double* val = nullptr;
};

// ---- permute.cu -----------------------------------------------------------
void scan_exclusive(const int* in, int* out, int n, int* tmp, cudaStream_t st, int64_t* launches);
void launch_permute_pattern(const DevCsr& a, const int* perm, DevCsr& b, int* src, int* tmp,
                            const int* long_rows_new, int n_long, int max_long, cudaStream_t st,
                            int64_t* launches);
void launch_gather_values(const int* src, const double* val, double* nval, int nnz, cudaStream_t st,
                          int64_t* launches);
void launch_permute_vec(int n, const int* perm, const double* x, double* y, bool inverse, cudaStream_t st,
                        int64_t* launches);
// perm (entries already range-checked) is a bijection: *bad = 0 (bits: (n + 31) / 32 words of scratch)
void launch_perm_check(int n, const int* perm, unsigned* bits, int* bad, cudaStream_t st, int64_t* launches);

// ---- block_lu.cu ----------------------------------------------------------
struct PertRecord {
    int block;
    int column;
    double original;
    double replaced;
};

struct LuParams {
    int s;
    const int* bstart;      // s + 1, permuted indices
    const int64_t* fac_off;  // s, float offsets into fac (packed panels)
    DevCsr a;               // permuted matrix
    float* fac;
    int* piv;               // n: local pivot row for pivot position k of block b at bstart[b] + k
    int* pert_count;        // s
    PertRecord* pert;       // capacity pert_cap
    int* pert_n;
    int pert_cap;
    unsigned long long* singular;  // min over (block << 32 | column); ~0 if none
    unsigned long long* prof = nullptr;  // optional phase timers of k_block_lu_ll (HPBJ_LU_PROF=1)
    double eps;
    float* scratch;         // global tiles for blocks too large for shared memory
    int smem_dim;           // blocks with dim <= smem_dim factor in shared memory
    int scratch_ld;
    int warp_dim = 0;       // blocks with dim <= warp_dim: one warp per block (set by the launcher)
    int* next_block = nullptr;  // left-looking LU: block counter (zeroed by the launcher)
    const int* block_order = nullptr;  // its schedule (largest blocks first), or null: index order
};

// Packed factor layout: block b with dim d, T = ceil(d/32)
// row panels of 32 pivot-ordered rows x dp4 = roundup(d, 4) columns; element
// (k, c) at fac_off[b] + (k/32)*32*dp4 + (c/4)*128 + (k%32)*4 + (c%4).
__host__ __device__ inline int64_t panel_floats(int d) {
    const int T = (d + 31) / 32;
    const int dp4 = (d + 3) & ~3;
    return (int64_t)T * 32 * dp4;
}

void launch_block_lu(const LuParams& p, int dmax, int num_sms, cudaStream_t st, int64_t* launches);
size_t block_lu_scratch_floats(int dmax, int num_sms, int* smem_dim, int* scratch_ld);

// ---- spk.cu ---------------------------------------------------------------
// Sparse-panel factor storage (see spk.cu): per 32-row panel, the off-panel
// L then U entries row-sorted (FP32 value + packed column << 5 | row), and
// the inverse of the 32x32 diagonal tile as 9 float4 quads per row.
constexpr int kTileFloats = 9 * 128;
constexpr int kIdx16MaxDim = 2047;  // 16-bit packed indices up to this block size

struct SpkPanel {
    int off;   // first L entry (16-byte aligned)
    int nl;    // row-sorted: L entries; row quads: max quads per row | total quads << 11
    int nu;    // same for U
    int uoff;  // first U entry (16-byte aligned)
};
constexpr int kRowQuadBits = 11;

struct SpkBuild {
    int s;
    int num_panels;
    const int* bstart;
    const int* pstart;      // s + 1: first panel of each block
    int* panel_block;       // num_panels
    const int64_t* fac_off;
    const float* dense;     // dense panels from block_lu
    int* ent_count;         // pass 1 output (entries, parts padded to 4)
    const int* ent_off;     // exclusive scan of the counts
    SpkPanel* desc;         // pass 2 outputs
    float* dtile;           // kTileFloats per panel
    float* eval;
    void* eidx;             // uint16_t (dmax <= kIdx16MaxDim) or uint32_t
    int idx32;
    int rows;               // pass 2 layout: 0 row-sorted runs, 1 rank-major row quads (see spk.cu)
    int* ent_count_rows;    // pass 1 output: entries of the row-quad layout
    unsigned long long* totals;  // pass 1 output: [0] entries row-sorted, [1] row-quad
    uint16_t* rmeta;        // row-quad layout: per panel part, 32 x (row | quads << 5) in rank order
    int dmax;
    uint16_t* rowcnt;       // pass 1 output: [panel][2][32] off-panel nonzeros of each row (L part, U part)
};

// Tile quads of row l (q = 0..7 cover columns 4q..4q+3, qd = l / 4): q < qd
// strictly-lower Linv, q > qd upper Uinv, q == qd the Linv part of the
// diagonal quad (zeros from the diagonal on); quad 8 the Uinv part of the
// diagonal quad. Stored [quad][lane] so a warp's loads are coalesced.
struct SpkView {
    int s;
    int dmax;
    const int* bstart;
    const int* pstart;
    const int* piv;
    const SpkPanel* desc;
    const float* dtile;
    const float* eval;
    const void* eidx;
    int idx32;
    const int* ent_off;   // num_panels + 1 (prefetch ranges)
    int rows;             // off-panel layout (SpkBuild::rows)
    const uint16_t* rmeta;
    int64_t n_entries;    // stored off-panel entries (arena sizes for L2 prefetch)
    int num_panels;
    int n;
    int pf;               // L2 prefetch (per-line, warp-wide) of the next step's entries / tiles
};

void launch_spk_count(const SpkBuild& p, cudaStream_t st, int64_t* launches);
void launch_spk_tile(const SpkBuild& p, cudaStream_t st, int64_t* launches);
void launch_spk_pack(const SpkBuild& p, cudaStream_t st, int64_t* launches);
// Arnoldi step: z32 = M^-1 V[:, st->j] (FP32 arithmetic, column resolved on the device).
void launch_apply_step(const SpkView& v, const double* V, int ldv, const SolveState* sst, float* z32,
                       cudaStream_t st, int64_t* launches);
// z = M^-1 v (Preconditioner::apply<float>), permuted frame.
void launch_apply_vec(const SpkView& v, const double* vin, double* z64, cudaStream_t st, int64_t* launches);
// x += M^-1 (V y): fused basis combination, FP64 arithmetic on the FP32 factors.
void launch_apply_update(const SpkView& v, const double* V, int ldv, const double* y, const SolveState* sst,
                         double* x, cudaStream_t st, int64_t* launches);

// Neumann-series applies (apply_neumann, preconditioner.cpp:200-220). init = 1:
// term = acc = M^-1 src; init = 0: term -= M^-1 src, acc += term. src is V[:, st->j]
// (V != null; f32) / sum_i y_i V[i] (V != null; f64) or vin. out/xadd optional.
void launch_apply_neumann_f32(const SpkView& v, const double* vin, const double* V, int ldv, float* term,
                              float* acc, double* out, int init, const SolveState* sst, cudaStream_t st,
                              int64_t* launches);
void launch_apply_neumann_f64(const SpkView& v, const double* vin, const double* V, int ldv, const double* y,
                              double* term, double* acc, double* xadd, int init, const SolveState* sst,
                              cudaStream_t st, int64_t* launches);

// ---- ilu.cu ---------------------------------------------------------------
struct KrylovBufs;
// ILU(0) factors in place in A's pattern (original ordering), sync-free
// ticketed passes; flags: factored rows, ytag/ztag: epoch-tagged apply
// results, ticket64 monotone across applies, apply_grid fixed per
// factorisation.
struct IluParams {
    int n = 0;
    const int* rp = nullptr;
    const int* ci = nullptr;
    const int* dpos = nullptr;
    double* lu = nullptr;
    int nch = 0;               // 32-row chunks of the applies
    int* flags = nullptr;      // n: factored-row flags (factorisation)
    double2* ytag = nullptr;   // n: forward results (value, epoch)
    double2* ztag = nullptr;   // n: backward results (value, epoch)
    int* ticket32 = nullptr;
    unsigned long long* ticket64 = nullptr;
    int apply_grid = 1;
    int seq = 0;               // apply with the one-warp sweep (deep dependency graphs)
};
// first row without a structural diagonal, or -1
int launch_ilu0_diag(int n, const int* rp, const int* ci, int* dpos, int* scratch, cudaStream_t st,
                     int64_t* launches);
// err: min (i << 32 | k) over zero pivots met (~0 when none)
void launch_ilu0_factor(const IluParams& p, unsigned long long* err, int num_sms, cudaStream_t st,
                        int64_t* launches);
// first row with a zero factored diagonal, or -1
int launch_ilu0_zero_diag(const IluParams& p, int* scratch, cudaStream_t st, int64_t* launches);
int ilu0_apply_grid(int n, int num_sms);
// times the ticketed and the one-warp apply once each and sets p.seq (clobbers vin/z scratch)
void ilu0_choose_apply(IluParams& p, double* vin, double* z, cudaStream_t st, int64_t* launches);
int ilu0_chunks(int n);
// z = U^-1 L^-1 src; src = V[:, st->j] (V != null, skipped when st->done) or vin;
// z (optional) plain copy of the result, xadd (optional): x += z
void launch_ilu0_apply(const IluParams& p, const double* vin, const double* V, int ldv, const SolveState* sst,
                       double* z, double* xadd, cudaStream_t st, int64_t* launches);
// u = sum_{i < st->j} y_i V_i, or x += that sum when xadd != null
void launch_basis_combine(const KrylovBufs& kb, const SolveState* sst, int n, double* u, double* xadd,
                          cudaStream_t st, int64_t* launches);
// z = V[:, st->j] (skipped when st->done)
void launch_copy_column(const KrylovBufs& kb, const SolveState* sst, int n, double* z, cudaStream_t st,
                        int64_t* launches);

// ---- spmv.cu --------------------------------------------------------------
struct SpmvPlan {
    int group = 8;            // lanes per row
    int long_thresh = 256;    // rows longer than this get a CTA of their own
    int n_long = 0;
    int* long_rows = nullptr; // indices of long rows (device), one CTA each
};

// y = A x, x FP32 (preconditioned vector) or FP64; early exit if st->done.
void launch_spmv_f32x(const DevCsr& a, const SpmvPlan& plan, const float* x, double* y,
                      const SolveState* sst, cudaStream_t st, int64_t* launches);
void launch_spmv_f64x(const DevCsr& a, const SpmvPlan& plan, const double* x, double* y,
                      cudaStream_t st, int64_t* launches, const SolveState* sst = nullptr);
// r = b - A x and st->rnorm = ||r||_2 (deterministic grid reduction).
void launch_residual(const DevCsr& a, const SpmvPlan& plan, const double* x, const double* b, double* r,
                     SolveState* sst, double* partials, cudaStream_t st, int64_t* launches);
// st->scratch = ||x||_2
void launch_norm(const double* x, int n, SolveState* sst, double* partials, cudaStream_t st,
                 int64_t* launches);

// ---- arnoldi.cu -----------------------------------------------------------
struct KrylovBufs {
    double* V = nullptr;   // (m+1) x ldv
    int ldv = 0;
    double* w = nullptr;   // SpMV output / global MGS scratch
    double* H = nullptr;   // (m+1) x m, column-major (gmres.hpp:24)
    double* R = nullptr;   // Givens-rotated copy
    double* cs = nullptr;
    double* sn = nullptr;
    double* g = nullptr;   // m + 1
    double* y = nullptr;   // m
    double* est = nullptr; // m: Givens estimate after each step of the cycle
    double* partials = nullptr;
    double* hist = nullptr;     // device residual history (est/||b|| per step)
    int* hist_cycle = nullptr;  // cycle index of each history row
    double* cycres = nullptr;   // true relative residual per cycle
    int m = 0;
};

struct MgsLaunch {
    int grid = 0;
    int threads = 1024;
    int slice = 0;
    size_t smem = 0;    // dynamic: Givens scratch (scr doubles) + the w slice when w_in_smem
    int scr = 0;
    bool w_in_smem = true;
    bool pipelined = true;  // textbook MGS: k_mgs_pipe (no pass waits for the grid) instead of k_mgs (a grid barrier per pass)
    bool icwy = false;  // compact-WY (2 barriers/step) instead of textbook MGS (j+2)
};

constexpr int kMaxRestart = 128;  // compact-WY tables; textbook MGS has no limit

MgsLaunch plan_mgs(int n, int num_sms, int m);
size_t orth_partials_doubles(int num_sms);
// cond: WHILE-node handle of the Arnoldi loop (0 outside graphs); the kernel
// sets it to !done when it finishes the step.
void launch_mgs(const MgsLaunch& L, const KrylovBufs& kb, double* gram, GridBarrier* gb, SolveState* sst,
                int n, cudaGraphConditionalHandle cond, cudaStream_t st, int64_t* launches);
void launch_cycle_init(const KrylovBufs& kb, SolveState* sst, const double* r, int n,
                       cudaGraphConditionalHandle cond, cudaStream_t st, int64_t* launches);
// restart-driver bookkeeping after the true residual; sets the outer WHILE
// handle to (!converged && cycles < max_restarts && steps > 0).
void launch_cycle_end(const KrylovBufs& kb, SolveState* sst, cudaGraphConditionalHandle cond, cudaStream_t st,
                      int64_t* launches);
void launch_solve_y(const KrylovBufs& kb, SolveState* sst, cudaStream_t st, int64_t* launches);

// ---- diag.cu --------------------------------------------------------------
struct DiagParams {
    int s;
    int dmax;
    const int* bstart;
    const int64_t* fac_off;
    const float* fac;       // dense LU panels
    const int* piv;
    DevCsr a;               // permuted matrix
    double* cond;           // s: cond_1 estimate
    double* ebound;         // s: (cond*2^-53 + 2^-24)*cond
};
void launch_block_cond(const DiagParams& p, int num_sms, cudaStream_t st, int64_t* launches);

// ---- fused.cu -------------------------------------------------------------
// A whole Arnoldi cycle (apply, SpMV, compact-WY MGS, Givens per step) as one
// persistent cooperative kernel; ok = false when the shared-memory tables do
// not fit (then the per-kernel path runs).
struct FusedPlan {
    bool ok = false;
    int grid = 0;
    int slice = 0;
    int ystride = 0;
    int nnz_cap = 0;
    size_t smem = 0;
    bool rows = false;  // SPK row-quad layout
};
// rowlen: row lengths of the permuted matrix (the CTA slices' matrix rows are
// cached in shared memory)
// brp: row starts of the permuted matrix (host), or null when unavailable
FusedPlan plan_fused(int n, int s, int dmax, int num_sms, int m, bool has_long, const int* brp, bool rows);
bool fused_possible(int n, int s, int num_sms);
void launch_arnoldi_cycle(const FusedPlan& F, const SpkView& pc, const DevCsr& a, const SpmvPlan& plan,
                          const KrylovBufs& kb, double* gram, SolveState* sst, GridBarrier* gb, float* z32,
                          unsigned long long* prof, cudaStream_t st, int64_t* launches);

}  // namespace hpbj
