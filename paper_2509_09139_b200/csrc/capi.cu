// libhpbj.so C ABI (include/hpbj.h): context, device buffers, and the restart
// driver of hybrid_restart_gmres (gmres.cpp:200-274) with every numerical
// step on the device. The host only sequences launches and reads a handful
// of scalars once per restart cycle (never per Arnoldi iteration).

#include <algorithm>
#include <chrono>

#include <omp.h>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <unordered_map>
#include <string>
#include <vector>

#include "device.cuh"
#include "kernels.cuh"

using namespace hpbj;

namespace {

// Device memory pool of one context: freed buffers are kept and reused by
// later requests of similar size, so re-setup / e2e steps (set_matrix,
// bj_setup, workspace) never pay cudaMalloc/cudaFree (which synchronise).
struct Pool {
    std::multimap<size_t, void*> free_;
    std::unordered_map<void*, size_t> size_;
    bool poison = false;  // HPBJ_POISON=1: every block handed out is filled with 0xff (debug)
    void* get(size_t bytes) {
        bytes = std::max<size_t>(256, (bytes + 255) & ~size_t(255));
        auto it = free_.lower_bound(bytes);
        if (it != free_.end() && it->first <= 2 * bytes + (1 << 20)) {
            void* p = it->second;
            free_.erase(it);
            if (poison) {  // legacy-stream memset: finish it before a non-blocking stream initialises the block
                HPBJ_CUDA(cudaMemset(p, 0xff, bytes));
                HPBJ_CUDA(cudaDeviceSynchronize());
            }
            return p;
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            // give cached blocks back to the driver and retry once
            for (auto& kv : free_) {
                cudaFree(kv.second);
                size_.erase(kv.second);
            }
            free_.clear();
            (void)cudaGetLastError();
            HPBJ_CUDA(cudaMalloc(&p, bytes));
        }
        size_[p] = bytes;
        if (poison) {
            HPBJ_CUDA(cudaMemset(p, 0xff, bytes));
            HPBJ_CUDA(cudaDeviceSynchronize());
        }
        return p;
    }
    void put(void* p) {
        if (!p) return;
        auto it = size_.find(p);
        if (it == size_.end()) {
            cudaFree(p);
            return;
        }
        free_.emplace(it->second, p);
    }
    ~Pool() {
        for (auto& kv : size_) cudaFree(kv.first);
    }
};

thread_local Pool* t_pool = nullptr;

// Slot-stable allocation: a context member keeps its device block across
// release/re-setup while the size fits, so buffer addresses (and with them
// the instantiated solve graph) stay valid from one setup to the next.
struct Slots {
    std::unordered_map<void*, std::pair<void*, size_t>> map;
};
thread_local Slots* t_slots = nullptr;

template <class T>
void dslot(T*& member, size_t count) {
    if (count == 0) count = 1;
    const size_t bytes = sizeof(T) * count;
    auto it = t_slots->map.find((void*)&member);
    if (it != t_slots->map.end() && it->second.second >= bytes) {
        member = static_cast<T*>(it->second.first);
        return;
    }
    if (it != t_slots->map.end()) t_pool->put(it->second.first);
    void* p = t_pool->get(bytes);
    t_slots->map[(void*)&member] = {p, bytes};
    member = static_cast<T*>(p);
}

template <class T>
T* dalloc(size_t count) {
    if (count == 0) count = 1;
    return static_cast<T*>(t_pool->get(sizeof(T) * count));
}

template <class T>
void dfree(T*& p) {  // slot-backed members: forget the pointer, keep the block
    p = nullptr;
}
template <class T>
void dput(T*& p) {  // transient blocks: back to the pool
    if (p) t_pool->put(p);
    p = nullptr;
}

struct KernelTimer {
    std::vector<cudaEvent_t> ev;  // pairs
    size_t used = 0;
    void reserve(size_t pairs) {
        while (ev.size() < 2 * pairs) {
            cudaEvent_t e;
            HPBJ_CUDA(cudaEventCreate(&e));
            ev.push_back(e);
        }
    }
    ~KernelTimer() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

// Grow-only page-locked staging buffer for host<->device copies at full
// PCIe/C2C speed; an event fences reuse while a previous async copy is in flight.
struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    void* get(size_t bytes) {
        if (ev) HPBJ_CUDA(cudaEventSynchronize(ev));
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            HPBJ_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
            cap = bytes;
        }
        return p;
    }
    void fence(cudaStream_t st) {
        if (!ev) HPBJ_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        HPBJ_CUDA(cudaEventRecord(ev, st));
    }
    ~PinnedBuf() {
        if (ev) cudaEventDestroy(ev);
        if (p) cudaFreeHost(p);
    }
};

constexpr double kU53 = 1.1102230246251565e-16;  // 2^-53
constexpr double kU24 = 5.9604644775390625e-08;  // 2^-24

}  // namespace

constexpr int kPcNone = 0, kPcBJ = 1, kPcIlu = 2, kPcIdentity = 3;

struct hpbj_ctx {
    Pool pool;  // destroyed last
    Slots slots;
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;      // SPK tile pass, concurrent with the count/pack passes
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;
    int64_t launches = 0;

    // matrix (original ordering)
    bool has_matrix = false;
    DevCsr A;
    std::vector<int> h_rp;          // row starts of A (int32)
    PinnedBuf stage_mat;  // set_matrix: int32 rp, int32 ci, FP64 val
    PinnedBuf stage_vec;  // hpbj_gmres host path: b, x
    std::vector<int> h_perm32;      // bj_setup scratch (persistent: no page faults per setup)
    std::vector<int> h_brp;         // row starts of Q A Q^T, fetched for the fused-cycle plan
    bool h_brp_valid = false;
    SpmvPlan planA;
    double* d_tmpx = nullptr;  // n
    double* d_tmpy = nullptr;  // n

    // block-Jacobi preconditioner (permuted frame)
    bool has_pc = false;     // block-Jacobi factors present
    int active = 0;          // preconditioner the solve uses: kPcNone / kPcBJ / kPcIlu / kPcIdentity
    bool has_ilu = false;
    IluParams ilu;           // ILU(0) factors in A's pattern (ilu.cu)
    double* d_ilu_lu = nullptr;
    int* d_ilu_dpos = nullptr;
    int* d_ilu_flags = nullptr;
    double2* d_ilu_ytag = nullptr;
    double2* d_ilu_ztag = nullptr;
    int* d_ilu_tick32 = nullptr;
    unsigned long long* d_ilu_tick64 = nullptr;
    unsigned long long* d_ilu_err = nullptr;
    double* d_ilu_z = nullptr;  // preconditioned vector (FP64 preconditioners)
    double* d_ilu_u = nullptr;  // basis combination of the x-update
    int s = 0;
    double eps = 1e-10;
    int dmin = 0, dmax = 0;
    int* d_perm = nullptr;
    DevCsr B;
    int* d_src = nullptr;
    int* d_bstart = nullptr;
    int64_t* d_fac_off = nullptr;
    float* d_fac = nullptr;
    int64_t fac_floats = 0;
    int* d_piv = nullptr;
    int* d_pert_count = nullptr;
    double* d_cond = nullptr;  // diagnostics (on demand, invalidated by a refactor)
    double* d_ebound = nullptr;
    bool diag_valid = false;
    PertRecord* d_pert = nullptr;
    int* d_pert_n = nullptr;
    int* d_lu_next = nullptr;       // left-looking LU: next block to take (dynamic schedule)
    int* d_lu_order = nullptr;      // blocks by decreasing size (largest first)
    std::vector<int> h_lu_order;
    unsigned long long* d_singular = nullptr;
    float* d_lu_scratch = nullptr;
    int lu_smem_dim = 0, lu_scratch_ld = 0;
    std::vector<int> h_bstart;
    std::vector<int64_t> h_fac_off;
    // sparse-panel (SPK) factors for the apply
    int num_panels = 0;
    int64_t spk_entries = 0, spk_diag = 0;
    int* d_pstart = nullptr;
    int* d_panel_block = nullptr;
    int* d_ent_count = nullptr;
    int* d_ent_off = nullptr;
    int* d_scan_tmp = nullptr;
    SpkPanel* d_desc = nullptr;
    float* d_dtile = nullptr;
    float* d_eval = nullptr;
    uint32_t* d_eidx = nullptr;  // packed (col << 5 | row), 16- or 32-bit
    int* d_ent_count_rows = nullptr;
    unsigned long long* d_spk_totals = nullptr;
    uint16_t* d_rmeta = nullptr;
    uint16_t* d_rowcnt = nullptr;  // count pass -> pack pass: off-panel nonzeros per panel row (L, U)
    int spk_rows = 0;            // off-panel layout: 0 row-sorted runs, 1 row quads (spk.cu)
    int spk_rows_env = -1;       // HPBJ_SPK_ROWS=0|1 (read once at context creation)
    int apply_pf = 1;            // HPBJ_APPLY_PF=0: no L2 bulk prefetch in the standalone apply
    double spk_tile_bytes = 0;   // inverse-tile bytes one apply reads (all panels)
    SpmvPlan planB;
    int* d_long_sort = nullptr;
    int n_long_sort = 0, max_long_sort = 0;

    // solve workspace
    int ws_m = -1;
    KrylovBufs kb;
    SolveState* d_st = nullptr;
    float* d_z32 = nullptr;
    int neumann = 0;                 // BlockJacobiOptions::neumann_order (preconditioner.hpp:34)
    float* d_nterm32 = nullptr;      // Neumann series term (Arnoldi step, FP32)
    double* d_nterm64 = nullptr;     // Neumann series term / sum (x-update, FP64)
    double* d_nacc64 = nullptr;
    double* d_xp = nullptr;  // x (permuted)
    double* d_bp = nullptr;  // b (permuted)
    double* d_r = nullptr;
    double* d_red = nullptr;  // reduction partials
    size_t red_cap = 0;
    double* d_bo = nullptr;   // host-API staging (original ordering)
    double* d_xo = nullptr;
    double* d_gram = nullptr;
    GridBarrier* d_gb = nullptr;
    MgsLaunch mgs;
    int64_t hist_cap = 0;
    bool use_graph = true;
    bool use_fused = true;
    FusedPlan fused;  // per-solve: whole Arnoldi cycle in one kernel when ok
    unsigned long long* d_fprof = nullptr;  // HPBJ_FUSED_PROF=1: phase timers of the fused kernel
    unsigned long long* d_lu_prof = nullptr;  // HPBJ_LU_PROF=1: phase timers of the left-looking LU
    cudaGraphExec_t graph_exec = nullptr;
    int graph_builds = 0;
    std::vector<uintptr_t> graph_sig;

    // profiling
    bool profiling = false;
    KernelTimer timer;
    hpbj_kernel_stat stats[HPBJ_K_COUNT] = {};

    ~hpbj_ctx() {
        t_pool = &pool;
        t_slots = &slots;
        if (graph_exec) cudaGraphExecDestroy(graph_exec);
        if (d_fprof) cudaFree(d_fprof);
        if (d_lu_prof) cudaFree(d_lu_prof);
        release_matrix();
        release_ws();
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
        if (stream) cudaStreamDestroy(stream);
    }

    void release_pc() {
        dfree(d_perm);
        dfree(B.rp);
        dfree(B.ci);
        dfree(B.val);
        dfree(d_src);
        dfree(d_bstart);
        dfree(d_fac_off);
        dfree(d_fac);
        dfree(d_piv);
        dfree(d_pert_count);
        dfree(d_cond);
        dfree(d_ebound);
        dfree(d_pert);
        dfree(d_pert_n);
        dfree(d_singular);
        dfree(d_lu_scratch);
        dfree(planB.long_rows);
        dfree(d_long_sort);
        dfree(d_pstart);
        dfree(d_panel_block);
        dfree(d_ent_count);
        dfree(d_ent_off);
        dfree(d_scan_tmp);
        dfree(d_desc);
        dfree(d_dtile);
        dfree(d_eval);
        dfree(d_eidx);
        dfree(d_ent_count_rows);
        dfree(d_spk_totals);
        dfree(d_rmeta);
        dfree(d_rowcnt);
        has_pc = false;
        dfree(d_ilu_lu);
        dfree(d_ilu_dpos);
        dfree(d_ilu_flags);
        dfree(d_ilu_ytag);
        dfree(d_ilu_ztag);
        dfree(d_ilu_tick32);
        dfree(d_ilu_tick64);
        dfree(d_ilu_err);
        dfree(d_ilu_z);
        dfree(d_ilu_u);
        has_ilu = false;
        active = kPcNone;
    }
    void release_matrix() {
        release_pc();
        dfree(A.rp);
        dfree(A.ci);
        dfree(A.val);
        dfree(planA.long_rows);
        dfree(d_tmpx);
        dfree(d_tmpy);
        has_matrix = false;
    }
    void release_ws() {
        dfree(kb.V);
        dfree(kb.w);
        dfree(kb.H);
        dfree(kb.R);
        dfree(kb.cs);
        dfree(kb.sn);
        dfree(kb.g);
        dfree(kb.y);
        dfree(kb.est);
        dfree(kb.partials);
        dfree(d_st);
        dfree(d_z32);
        dfree(d_nterm32);
        dfree(d_nterm64);
        dfree(d_nacc64);
        dfree(d_xp);
        dfree(d_bp);
        dfree(d_r);
        dfree(d_red);
        dfree(d_bo);
        dfree(d_xo);
        dfree(d_gram);
        dfree(d_gb);
        dfree(kb.hist);
        dfree(kb.hist_cycle);
        dfree(kb.cycres);
        hist_cap = 0;
        ws_m = -1;
    }
};

namespace {

// Lanes per row from the mean row length; hub rows get CTAs of their own.
int spmv_group(int64_t nnz, int n) {
    const double avg = n > 0 ? double(nnz) / n : 0.0;
    // measured on B200 (configs 1-3): one thread per row (two rows
    // interleaved) wins up to ~12 nnz/row, then 2/4/8 lanes
    int g = avg <= 12.0 ? 1 : avg <= 20.0 ? 2 : avg <= 32.0 ? 4 : avg <= 64.0 ? 8 : 32;
    if (const char* e = getenv("HPBJ_SPMV_G")) g = atoi(e);
    return g;
}
int spmv_long_thresh(int g) { return std::max(256, 16 * g); }

// rows: indices (in the matrix's own numbering) of rows longer than the
// plan's threshold, in any order
void set_plan(SpmvPlan& p, int group, std::vector<int>& rows) {
    p.group = group;
    p.long_thresh = spmv_long_thresh(group);
    std::sort(rows.begin(), rows.end());
    p.n_long = (int)rows.size();
    if (p.n_long) {
        dslot(p.long_rows, rows.size());
        HPBJ_CUDA(cudaMemcpy(p.long_rows, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    }
}

void make_plan(SpmvPlan& p, const int* rp, int n) {
    const int g = spmv_group(rp[n], n);
    const int thr = spmv_long_thresh(g);
    std::vector<int> rows;
#pragma omp parallel if (n > 65536)
    {
        std::vector<int> mine;
#pragma omp for schedule(static) nowait
        for (int i = 0; i < n; ++i)
            if (rp[i + 1] - rp[i] > thr) mine.push_back(i);
#pragma omp critical
        rows.insert(rows.end(), mine.begin(), mine.end());
    }
    set_plan(p, g, rows);
}

// Row starts of Q A Q^T on the host, only when the fused cycle kernel could
// take the system (its plan sizes the per-CTA matrix slices from them).
const int* host_brp(hpbj_ctx* c) {
    if (!fused_possible(c->A.n, c->s, c->num_sms) || !c->B.rp) return nullptr;
    if (!c->h_brp_valid) {
        c->h_brp.resize((size_t)c->B.n + 1);
        HPBJ_CUDA(cudaMemcpyAsync(c->h_brp.data(), c->B.rp, sizeof(int) * ((size_t)c->B.n + 1),
                                  cudaMemcpyDeviceToHost, c->stream));
        HPBJ_CUDA(cudaStreamSynchronize(c->stream));
        c->h_brp_valid = true;
    }
    return c->h_brp.data();
}

void ensure_ws(hpbj_ctx* c, int m) {
    if (c->ws_m == m) return;
    c->release_ws();
    const int n = c->A.n;
    const int ldv = ((n + 31) / 32) * 32;
    KrylovBufs& kb = c->kb;
    kb.m = m;
    kb.ldv = ldv;
    dslot(kb.V, (size_t)(m + 1) * ldv);
    HPBJ_CUDA(cudaMemset(kb.V, 0, sizeof(double) * (size_t)(m + 1) * ldv));
    dslot(kb.w, ldv);
    HPBJ_CUDA(cudaMemset(kb.w, 0, sizeof(double) * ldv));
    dslot(kb.H, (size_t)(m + 1) * m);
    dslot(kb.R, (size_t)(m + 1) * m);
    dslot(kb.cs, m);
    dslot(kb.sn, m);
    dslot(kb.g, m + 1);
    dslot(kb.y, m);
    dslot(kb.est, m);
    dslot(kb.partials, orth_partials_doubles(c->num_sms));
    dslot(c->d_gram, (size_t)(m + 1) * (m + 1));
    dslot(c->d_gb, 1);
    HPBJ_CUDA(cudaMemset(c->d_gb, 0, sizeof(GridBarrier)));
    dslot(c->d_st, 1);
    HPBJ_CUDA(cudaMemset(c->d_st, 0, sizeof(SolveState)));
    dslot(c->d_z32, ldv);
    HPBJ_CUDA(cudaMemset(c->d_z32, 0, sizeof(float) * ldv));
    dslot(c->d_nterm32, ldv);
    dslot(c->d_nterm64, ldv);
    dslot(c->d_nacc64, ldv);
    dslot(c->d_xp, ldv);
    dslot(c->d_bp, ldv);
    dslot(c->d_r, ldv);
    dslot(c->d_red, 2048);
    c->red_cap = 2048;
    dslot(c->d_bo, ldv);
    dslot(c->d_xo, ldv);
    c->mgs = plan_mgs(n, c->num_sms, m);
    c->ws_m = m;
}

SpkView spk_view(const hpbj_ctx* c) {
    return SpkView{c->s,      c->dmax,   c->d_bstart, c->d_pstart, c->d_piv, c->d_desc,
                   c->d_dtile, c->d_eval, c->d_eidx,  c->dmax > kIdx16MaxDim ? 1 : 0, c->d_ent_off,
                   c->spk_rows, c->d_rmeta, c->spk_entries, c->num_panels, (int)c->A.n, c->apply_pf};
}

// Repack the dense LU panels into the sparse-panel apply format.
void build_spk(hpbj_ctx* c) {
    cudaStream_t st = c->stream;
    SpkBuild p{};
    p.s = c->s;
    p.num_panels = c->num_panels;
    p.bstart = c->d_bstart;
    p.pstart = c->d_pstart;
    p.panel_block = c->d_panel_block;
    p.fac_off = c->d_fac_off;
    p.dense = c->d_fac;
    p.ent_count = c->d_ent_count;
    p.ent_count_rows = c->d_ent_count_rows;
    p.totals = c->d_spk_totals;
    p.ent_off = c->d_ent_off;
    p.rowcnt = c->d_rowcnt;
    p.dtile = c->d_dtile;
    p.dmax = c->dmax;
    launch_spk_count(p, st, &c->launches);
    // the tile inverses (latency bound) run on the side stream while the
    // count result comes back and the pack pass (bandwidth bound) runs here
    HPBJ_CUDA(cudaEventRecord(c->ev_fork, st));
    HPBJ_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    launch_spk_tile(p, c->side, &c->launches);
    HPBJ_CUDA(cudaEventRecord(c->ev_join, c->side));
    // Off-panel layout: row quads (fold_rows: one coalesced quad per row and
    // slot, ~3x fewer fold instructions than the segmented fold) for blocks
    // deeper than the fused cycle kernel takes (it folds row-sorted runs),
    // or when padding rows to whole quads costs < 25% more entries;
    // HPBJ_SPK_ROWS=0/1 forces one. Measured (B200): apply 343 -> 286 us on
    // config 3, 70 -> 66 us on config 2.
    unsigned long long totals[2] = {0, 0};
    HPBJ_CUDA(cudaMemcpyAsync(totals, c->d_spk_totals, sizeof(totals), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaStreamSynchronize(st));
    // Blocks of <= 96 rows run in the fused cycle kernel, which folds
    // row-sorted runs (row quads pad its short rows by ~46%: apply phase
    // +11% on config 1); deeper blocks take row quads.
    c->spk_rows = c->spk_rows_env >= 0 ? c->spk_rows_env : (c->dmax > 96 ? 1 : 0);
    if (totals[c->spk_rows] >= (unsigned long long)INT32_MAX)
        fail(HPBJ_EINVAL, "block_jacobi: factor nonzeros exceed 2^31");
    scan_exclusive(c->spk_rows ? c->d_ent_count_rows : c->d_ent_count, c->d_ent_off, c->num_panels, c->d_scan_tmp, st,
                   &c->launches);
    const int tot = (int)totals[c->spk_rows];
    c->spk_entries = tot;
    const bool idx32 = c->dmax > kIdx16MaxDim;
    dslot(c->d_eval, (size_t)tot + 32);  // parts are 4-entry aligned
    dslot(c->d_eidx, idx32 ? (size_t)tot + 32 : (size_t)tot / 2 + 16);
    p.desc = c->d_desc;
    p.dtile = c->d_dtile;
    p.eval = c->d_eval;
    p.eidx = c->d_eidx;
    p.idx32 = idx32 ? 1 : 0;
    p.rows = c->spk_rows;
    p.rmeta = c->d_rmeta;
    // tile bytes an apply reads: a full panel 2 x 144 quads (lane l: quads
    // 0..l/4 forward, l/4..7 backward), a block's last panel of r rows its
    // (L U)^-1 rows: r x ceil(r / 4) quads
    c->spk_tile_bytes = 0;
    for (int64_t b = 0; b < c->s; ++b) {
        const int d = c->h_bstart[b + 1] - c->h_bstart[b];
        const int T = (d + 31) / 32, r = d - 32 * (T - 1);
        c->spk_tile_bytes += 16.0 * (288.0 * (T - 1) + (double)r * ((r + 3) / 4));
    }
    launch_spk_pack(p, st, &c->launches);
    HPBJ_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));  // everything after the build sees the tiles
}

void factor(hpbj_ctx* c, hpbj_setup_info* info) {
    cudaStream_t st = c->stream;
    c->diag_valid = false;
    const unsigned long long none = ~0ull;
    HPBJ_CUDA(cudaMemcpyAsync(c->d_singular, &none, sizeof(none), cudaMemcpyHostToDevice, st));
    HPBJ_CUDA(cudaMemsetAsync(c->d_pert_n, 0, sizeof(int), st));
    LuParams p;
    p.s = c->s;
    p.bstart = c->d_bstart;
    p.fac_off = c->d_fac_off;
    p.a = c->B;
    p.fac = c->d_fac;
    p.piv = c->d_piv;
    p.pert_count = c->d_pert_count;
    p.pert = c->d_pert;
    p.pert_n = c->d_pert_n;
    p.next_block = c->d_lu_next;
    p.block_order = c->d_lu_order;
    p.pert_cap = 4096;
    p.singular = c->d_singular;
    p.eps = c->eps;
    p.scratch = c->d_lu_scratch;
    p.smem_dim = c->lu_smem_dim;
    p.scratch_ld = c->lu_scratch_ld;
    static const bool lu_prof = getenv("HPBJ_LU_PROF") != nullptr;
    if (lu_prof) {
        if (!c->d_lu_prof) HPBJ_CUDA(cudaMalloc(&c->d_lu_prof, 4 * sizeof(unsigned long long)));
        HPBJ_CUDA(cudaMemsetAsync(c->d_lu_prof, 0, 4 * sizeof(unsigned long long), st));
        p.prof = c->d_lu_prof;
    }
    cudaEvent_t e0, e1, eg, el;
    HPBJ_CUDA(cudaEventCreate(&e0));
    HPBJ_CUDA(cudaEventCreate(&e1));
    HPBJ_CUDA(cudaEventCreate(&eg));
    HPBJ_CUDA(cudaEventCreate(&el));
    HPBJ_CUDA(cudaEventRecord(e0, st));
    launch_gather_values(c->d_src, c->A.val, c->B.val, c->B.nnz, st, &c->launches);
    HPBJ_CUDA(cudaEventRecord(eg, st));
    launch_block_lu(p, c->dmax, c->num_sms, st, &c->launches);
    HPBJ_CUDA(cudaEventRecord(el, st));
    build_spk(c);
    HPBJ_CUDA(cudaEventRecord(e1, st));
    unsigned long long sing = 0;
    int pert_n = 0;
    HPBJ_CUDA(cudaMemcpyAsync(&sing, c->d_singular, sizeof(sing), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaMemcpyAsync(&pert_n, c->d_pert_n, sizeof(int), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaStreamSynchronize(st));
    if (lu_prof) {
        unsigned long long t[3];
        HPBJ_CUDA(cudaMemcpy(t, c->d_lu_prof, sizeof(t), cudaMemcpyDeviceToHost));
        const double tot = double(t[0] + t[1] + t[2]);
        fprintf(stderr, "[hpbj lu] CTA cycles: left-looking updates %.3g (%.0f%%), panel factorisation %.3g (%.0f%%), "
                        "L store + output %.3g (%.0f%%)\n", double(t[0]), 100 * t[0] / tot, double(t[1]),
                100 * t[1] / tot, double(t[2]), 100 * t[2] / tot);
    }
    float ms = 0.f, ms_lu = 0.f, ms_spk = 0.f;
    HPBJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    HPBJ_CUDA(cudaEventElapsedTime(&ms_lu, eg, el));
    HPBJ_CUDA(cudaEventElapsedTime(&ms_spk, el, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(eg);
    cudaEventDestroy(el);
    if (info) {
        info->ms_lu = ms_lu;
        info->ms_spk = ms_spk;
        info->num_blocks = c->s;
        info->dim_min = c->dmin;
        info->dim_max = c->dmax;
        info->perturbations = pert_n;
        info->singular_block = -1;
        info->singular_column = -1;
        info->factor_bytes = c->fac_floats * (int64_t)sizeof(float);
        info->ms_factor = ms;
    }
    if (sing != none) {
        const int64_t blk = (int64_t)(sing >> 32), col = (int64_t)(sing & 0xffffffffu);
        if (info) {
            info->singular_block = blk;
            info->singular_column = col;
        }
        c->has_pc = false;
        if (c->active == kPcBJ) c->active = kPcNone;
        fail(HPBJ_ESINGULAR, "gp_lu: singular block, zero pivot in column " + std::to_string(col) +
                                 " (block " + std::to_string(blk) + ")");
    }
}

// The solve's frame: Q A Q^T for block Jacobi (contiguous blocks), A itself
// for the order-dependent ILU(0) and for the identity.
const DevCsr& sys(const hpbj_ctx* c) { return c->active == kPcBJ ? c->B : c->A; }
const SpmvPlan& sys_plan(const hpbj_ctx* c) { return c->active == kPcBJ ? c->planB : c->planA; }
void to_frame(hpbj_ctx* c, const double* x, double* xf) {
    if (c->active == kPcBJ) launch_permute_vec(c->A.n, c->d_perm, x, xf, false, c->stream, &c->launches);
    else HPBJ_CUDA(cudaMemcpyAsync(xf, x, sizeof(double) * c->A.n, cudaMemcpyDeviceToDevice, c->stream));
}
void from_frame(hpbj_ctx* c, const double* xf, double* x) {
    if (c->active == kPcBJ) launch_permute_vec(c->A.n, c->d_perm, xf, x, true, c->stream, &c->launches);
    else HPBJ_CUDA(cudaMemcpyAsync(x, xf, sizeof(double) * c->A.n, cudaMemcpyDeviceToDevice, c->stream));
}
// kernels per Arnoldi step / per cycle of the unfused graph (launch accounting)
int64_t step_launches(const hpbj_ctx* c) {
    return 2 + (c->active == kPcBJ ? 1 + 2 * std::max(0, c->neumann) : c->active == kPcIlu ? 1 : 1);
}
int64_t cycle_launches(const hpbj_ctx* c) {
    return 4 + (c->active == kPcBJ ? 1 + 2 * std::max(0, c->neumann) : c->active == kPcIlu ? 2 : 1);
}

void record_kernel(hpbj_ctx* c, size_t slot, bool begin) {
    if (!c->profiling) return;
    HPBJ_CUDA(cudaEventRecord(c->timer.ev[2 * slot + (begin ? 0 : 1)], c->stream));
}

// One restart cycle of hybrid_restart_gmres as device launches (gmres.cpp:
// 236-256 around run_cycle :97-166). With conditional handles (graph mode)
// the Arnoldi loop is a WHILE node driven by the orthogonalisation kernel.
void enqueue_cycle_head(hpbj_ctx* c, cudaGraphConditionalHandle hin) {
    launch_cycle_init(c->kb, c->d_st, c->d_r, c->A.n, hin, c->stream, &c->launches);
}
void enqueue_step(hpbj_ctx* c, cudaGraphConditionalHandle hin, int it) {
    KrylovBufs& kb = c->kb;
    if (c->active != kPcBJ) {  // FP64 preconditioners: z64 = M^-1 V[:, j], w = A z64
        record_kernel(c, 3 * it + 0, true);
        if (c->active == kPcIlu)
            launch_ilu0_apply(c->ilu, nullptr, kb.V, kb.ldv, c->d_st, c->d_ilu_z, nullptr, c->stream, &c->launches);
        else
            launch_copy_column(kb, c->d_st, c->A.n, c->d_ilu_z, c->stream, &c->launches);
        record_kernel(c, 3 * it + 0, false);
        record_kernel(c, 3 * it + 1, true);
        launch_spmv_f64x(c->A, c->planA, c->d_ilu_z, kb.w, c->stream, &c->launches, c->d_st);
        record_kernel(c, 3 * it + 1, false);
        record_kernel(c, 3 * it + 2, true);
        launch_mgs(c->mgs, kb, c->d_gram, c->d_gb, c->d_st, c->A.n, hin, c->stream, &c->launches);
        record_kernel(c, 3 * it + 2, false);
        return;
    }
    record_kernel(c, 3 * it + 0, true);
    if (c->neumann > 0) {
        // z = sum_{i<=k} (I - M^-1 A)^i M^-1 v_j in FP32 (preconditioned<float>, gmres.cpp:91-95);
        // A term on the FP64 SpMV of the FP32 term, the step's w as scratch
        launch_apply_neumann_f32(spk_view(c), nullptr, kb.V, kb.ldv, c->d_nterm32, c->d_z32, nullptr, 1, c->d_st,
                                 c->stream, &c->launches);
        for (int i = 1; i <= c->neumann; ++i) {
            launch_spmv_f32x(c->B, c->planB, c->d_nterm32, kb.w, c->d_st, c->stream, &c->launches);
            launch_apply_neumann_f32(spk_view(c), kb.w, nullptr, 0, c->d_nterm32, c->d_z32, nullptr, 0, c->d_st,
                                     c->stream, &c->launches);
        }
    } else {
        launch_apply_step(spk_view(c), kb.V, kb.ldv, c->d_st, c->d_z32, c->stream, &c->launches);
    }
    record_kernel(c, 3 * it + 0, false);
    record_kernel(c, 3 * it + 1, true);
    launch_spmv_f32x(c->B, c->planB, c->d_z32, kb.w, c->d_st, c->stream, &c->launches);
    record_kernel(c, 3 * it + 1, false);
    record_kernel(c, 3 * it + 2, true);
    launch_mgs(c->mgs, kb, c->d_gram, c->d_gb, c->d_st, c->A.n, hin, c->stream, &c->launches);
    record_kernel(c, 3 * it + 2, false);
}
// The fused path: the whole Arnoldi loop of a cycle is one cooperative kernel.
void enqueue_cycle_fused(hpbj_ctx* c) {
    launch_arnoldi_cycle(c->fused, spk_view(c), c->B, c->planB, c->kb, c->d_gram, c->d_st, c->d_gb, c->d_z32,
                         c->d_fprof, c->stream, &c->launches);
}
void enqueue_cycle_tail(hpbj_ctx* c, cudaGraphConditionalHandle hout) {
    KrylovBufs& kb = c->kb;
    launch_solve_y(kb, c->d_st, c->stream, &c->launches);
    if (c->active == kPcIlu) {  // x += M^-1 (V y), FP64 (gmres.cpp:150-159)
        launch_basis_combine(kb, c->d_st, c->A.n, c->d_ilu_u, nullptr, c->stream, &c->launches);
        launch_ilu0_apply(c->ilu, c->d_ilu_u, nullptr, 0, c->d_st, nullptr, c->d_xp, c->stream, &c->launches);
    } else if (c->active == kPcIdentity) {
        launch_basis_combine(kb, c->d_st, c->A.n, nullptr, c->d_xp, c->stream, &c->launches);
    } else if (c->neumann > 0) {  // preconditioned<double> (gmres.cpp:158): FP64 series, x += sum
        launch_apply_neumann_f64(spk_view(c), nullptr, kb.V, kb.ldv, kb.y, c->d_nterm64, c->d_nacc64, nullptr, 1,
                                 c->d_st, c->stream, &c->launches);
        for (int i = 1; i <= c->neumann; ++i) {
            launch_spmv_f64x(c->B, c->planB, c->d_nterm64, kb.w, c->stream, &c->launches);
            launch_apply_neumann_f64(spk_view(c), kb.w, nullptr, 0, nullptr, c->d_nterm64, c->d_nacc64,
                                     i == c->neumann ? c->d_xp : nullptr, 0, c->d_st, c->stream, &c->launches);
        }
    } else {
        launch_apply_update(spk_view(c), kb.V, kb.ldv, kb.y, c->d_st, c->d_xp, c->stream, &c->launches);
    }
    launch_residual(sys(c), sys_plan(c), c->d_xp, c->d_bp, c->d_r, c->d_st, c->d_red, c->stream, &c->launches);
    launch_cycle_end(kb, c->d_st, hout, c->stream, &c->launches);
}

std::vector<uintptr_t> graph_signature(const hpbj_ctx* c) {
    const KrylovBufs& k = c->kb;
    const SpmvPlan& p = sys_plan(c);
    const DevCsr& M = sys(c);
    const MgsLaunch& L = c->mgs;
    return {(uintptr_t)k.V, (uintptr_t)k.w, (uintptr_t)k.H, (uintptr_t)k.R, (uintptr_t)k.cs, (uintptr_t)k.sn,
            (uintptr_t)k.g, (uintptr_t)k.y, (uintptr_t)k.est, (uintptr_t)k.partials, (uintptr_t)k.hist,
            (uintptr_t)k.hist_cycle, (uintptr_t)k.cycres, (uintptr_t)k.m, (uintptr_t)k.ldv,
            (uintptr_t)c->d_st, (uintptr_t)c->d_z32, (uintptr_t)c->d_xp, (uintptr_t)c->d_bp, (uintptr_t)c->d_r,
            (uintptr_t)c->d_red, (uintptr_t)c->d_gram, (uintptr_t)c->d_gb, (uintptr_t)M.rp, (uintptr_t)M.ci,
            (uintptr_t)M.val, (uintptr_t)M.n, (uintptr_t)M.nnz, (uintptr_t)p.group,
            (uintptr_t)p.long_thresh, (uintptr_t)p.n_long, (uintptr_t)p.long_rows,
            (uintptr_t)c->s, (uintptr_t)c->d_bstart, (uintptr_t)c->d_fac_off, (uintptr_t)c->d_fac,
            (uintptr_t)c->d_piv, (uintptr_t)c->dmax, (uintptr_t)c->d_pstart, (uintptr_t)c->d_desc,
            (uintptr_t)c->d_dtile, (uintptr_t)c->d_eval, (uintptr_t)c->d_eidx, (uintptr_t)L.grid, (uintptr_t)L.threads, (uintptr_t)L.slice,
            (uintptr_t)L.smem, (uintptr_t)L.icwy, (uintptr_t)L.w_in_smem, (uintptr_t)c->fused.ok,
            (uintptr_t)c->fused.grid, (uintptr_t)c->fused.slice, (uintptr_t)c->fused.ystride,
            (uintptr_t)c->fused.smem, (uintptr_t)c->fused.nnz_cap, (uintptr_t)c->d_ent_off,
            (uintptr_t)c->spk_rows, (uintptr_t)c->d_rmeta,
            (uintptr_t)c->neumann, (uintptr_t)c->d_nterm32, (uintptr_t)c->d_nterm64, (uintptr_t)c->d_nacc64,
            (uintptr_t)c->active, (uintptr_t)c->d_ilu_lu, (uintptr_t)c->d_ilu_dpos, (uintptr_t)c->d_ilu_flags,
            (uintptr_t)c->d_ilu_ytag, (uintptr_t)c->d_ilu_ztag,
            (uintptr_t)c->d_ilu_tick64, (uintptr_t)c->d_ilu_z, (uintptr_t)c->d_ilu_u,
            (uintptr_t)c->ilu.apply_grid, (uintptr_t)c->ilu.seq, (uintptr_t)c->A.rp, (uintptr_t)c->A.ci, (uintptr_t)c->A.val,
            (uintptr_t)c->planA.group, (uintptr_t)c->planA.n_long, (uintptr_t)c->planA.long_rows};
}

// The whole restart loop as one CUDA graph: WHILE(cycles) { cycle_init;
// WHILE(steps) { apply; spmv; orth }; solve_y; x += M^-1 V y; residual;
// bookkeeping }, the inner loop being one fused kernel when it fits
// (fused.cu). Rebuilt only when a buffer or launch shape changes.
void ensure_graph(hpbj_ctx* c) {
    std::vector<uintptr_t> sig = graph_signature(c);
    if (c->graph_exec && sig == c->graph_sig) return;
    if (c->graph_exec) {
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
    }
    cudaStream_t st = c->stream;
    cudaGraph_t g;
    HPBJ_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hout;
    HPBJ_CUDA(cudaGraphConditionalHandleCreate(&hout, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams op = {};
    op.type = cudaGraphNodeTypeConditional;
    op.conditional.handle = hout;
    op.conditional.type = cudaGraphCondTypeWhile;
    op.conditional.size = 1;
    cudaGraphNode_t onode;
    HPBJ_CUDA(cudaGraphAddNode(&onode, g, nullptr, 0, &op));
    cudaGraph_t body = op.conditional.phGraph_out[0];
    if (c->fused.ok) {
        // WHILE(cycles) { cycle_init; arnoldi_cycle; solve_y; update; residual; bookkeeping }
        HPBJ_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        enqueue_cycle_head(c, 0);
        enqueue_cycle_fused(c);
        enqueue_cycle_tail(c, hout);
        HPBJ_CUDA(cudaStreamEndCapture(st, &body));
    } else {
        cudaGraphConditionalHandle hin;
        HPBJ_CUDA(cudaGraphConditionalHandleCreate(&hin, body, 0, 0));
        HPBJ_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        enqueue_cycle_head(c, hin);
        cudaStreamCaptureStatus cstat;
        cudaGraph_t capg;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        HPBJ_CUDA(cudaStreamGetCaptureInfo(st, &cstat, nullptr, &capg, &deps, &ndeps));
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hin;
        ip.conditional.type = cudaGraphCondTypeWhile;
        ip.conditional.size = 1;
        cudaGraphNode_t inode;
        HPBJ_CUDA(cudaGraphAddNode(&inode, capg, deps, ndeps, &ip));
        cudaGraph_t ibody = ip.conditional.phGraph_out[0];
        HPBJ_CUDA(cudaStreamUpdateCaptureDependencies(st, &inode, 1, cudaStreamSetCaptureDependencies));
        enqueue_cycle_tail(c, hout);
        HPBJ_CUDA(cudaStreamEndCapture(st, &body));

        HPBJ_CUDA(cudaStreamBeginCaptureToGraph(st, ibody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        enqueue_step(c, hin, 0);
        HPBJ_CUDA(cudaStreamEndCapture(st, &ibody));
    }
    HPBJ_CUDA(cudaGraphInstantiate(&c->graph_exec, g, 0));
    HPBJ_CUDA(cudaGraphDestroy(g));
    c->graph_sig = sig;
    ++c->graph_builds;
    if (getenv("HPBJ_DEBUG")) fprintf(stderr, "[hpbj] solve graph built (#%d)\n", c->graph_builds);
}

// Algorithmic HBM bytes: what one pass must move at
// minimum in the stored formats — each factor/matrix byte and each vector
// element read or written once.
double apply_bytes(const hpbj_ctx* c) {
    const double n = c->A.n;
    const double idx_b = c->dmax > kIdx16MaxDim ? 4.0 : 2.0;
    return (4.0 + idx_b) * (double)c->spk_entries          // off-panel value + packed index
           + c->spk_tile_bytes + 16.0 * c->num_panels     // inverse-tile quads read + descriptors
           + (c->spk_rows ? 128.0 * c->num_panels : 0.0)  // row-quad metadata
           + 4.0 * n                                      // pivot rows (int32)
           + 8.0 * n                                      // v (FP64) in
           + 4.0 * n                                      // z (FP32) out
           + 8.0 * (c->s + 1);                            // block / panel starts
}
double spmv_bytes(const hpbj_ctx* c) {
    const double n = c->A.n, nnz = c->A.nnz;
    return 12.0 * nnz + 4.0 * (n + 1) + 4.0 * n + 8.0 * n;  // val+col, row ptr, z in (FP32), w out
}
double orth_bytes(const hpbj_ctx* c, int j) {
    // step j: V_0..V_j read once (compulsory; the second MGS pass re-reads
    // them from L2), w in, v_{j+1} out
    const double n = c->A.n;
    return 8.0 * n * (j + 1) + 8.0 * n + 8.0 * n;
}
double fused_step_bytes(const hpbj_ctx* c, int j) {  // w stays on chip: no SpMV write / orth read of w
    const double n = c->A.n;
    return apply_bytes(c) + spmv_bytes(c) - 8.0 * n + orth_bytes(c, j) - 8.0 * n + 8.0 * n /* w to HBM */;
}

void ensure_hist(hpbj_ctx* c, int64_t max_restarts) {
    const int64_t need = max_restarts * c->kb.m + 1;
    if (c->hist_cap >= need) return;
    dfree(c->kb.hist);
    dfree(c->kb.hist_cycle);
    dfree(c->kb.cycres);
    dslot(c->kb.hist, need);
    dslot(c->kb.hist_cycle, need);
    dslot(c->kb.cycres, max_restarts + 1);
    c->hist_cap = need;
}

// Config validation (gmres.cpp:203-207), before any workspace is sized.
hpbj_gmres_opts checked_opts(const hpbj_gmres_opts* o) {
    hpbj_gmres_opts opt;
    hpbj_gmres_default_opts(&opt);
    if (o) opt = *o;
    if (opt.restart_m < 1 || !(opt.tol > 0.0) || opt.max_restarts < 1)
        fail(HPBJ_EINVAL, "gmres: invalid config");
    if (opt.restart_m > 1024) fail(HPBJ_EINVAL, "gmres: restart_m > 1024 unsupported");
    if (opt.max_restarts > (int64_t)1 << 24) fail(HPBJ_EINVAL, "gmres: max_restarts too large");
    return opt;
}

void solve(hpbj_ctx* c, const double* d_b, double* d_x, const hpbj_gmres_opts* o, hpbj_report* rep,
           hpbj_history_point* hist, int64_t hist_cap, double* cycle_res, int64_t cyc_cap) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!c->has_matrix) fail(HPBJ_ELOGIC, "gmres: no matrix");
    if (c->active == kPcNone || (c->active == kPcBJ && !c->has_pc) || (c->active == kPcIlu && !c->has_ilu))
        fail(HPBJ_ELOGIC, "gmres: no preconditioner set up");
    const hpbj_gmres_opts opt = checked_opts(o);
    const int n = c->A.n;
    const int m = (int)opt.restart_m;
    const double floor_u = opt.floor_roundoff > 0.0 ? opt.floor_roundoff : kU24;
    ensure_ws(c, m);
    {  // residual partials: one per SpMV CTA incl. one per hub row
        const size_t need = 1184 + 64 + (size_t)sys_plan(c).n_long;
        if (need > c->red_cap) {
            dfree(c->d_red);
            dslot(c->d_red, need);
            c->red_cap = need;
        }
    }
    ensure_hist(c, opt.max_restarts);
    cudaStream_t st = c->stream;
    KrylovBufs& kb = c->kb;
    hpbj_report R{};
    int64_t hlen = 0, clen = 0;
    auto push_hist = [&](int64_t cyc, int64_t it, double rel) {
        if (hist && hlen < hist_cap) hist[hlen] = hpbj_history_point{cyc, it, rel};
        ++hlen;
    };

    // permuted b; ||b||
    to_frame(c, d_b, c->d_bp);
    launch_norm(c->d_bp, n, c->d_st, c->d_red, st, &c->launches);
    SolveState hs{};
    HPBJ_CUDA(cudaMemcpyAsync(&hs, c->d_st, sizeof(hs), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaStreamSynchronize(st));
    const double bnorm = hs.scratch;
    HPBJ_CUDA(cudaMemsetAsync(c->d_xp, 0, sizeof(double) * kb.ldv, st));
    if (bnorm == 0.0) {  // gmres.cpp:215-220
        R.converged = 1;
        push_hist(0, 0, 0.0);
        HPBJ_CUDA(cudaMemsetAsync(d_x, 0, sizeof(double) * n, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
        R.history_len = hlen;
        R.ms_solve = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (rep) *rep = R;
        return;
    }
    const double thr = opt.absolute_tol ? opt.tol : opt.tol * bnorm;
    hs = SolveState{};
    hs.n = n;
    hs.m = m;
    hs.ldv = kb.ldv;
    hs.thr = thr;
    hs.bnorm = bnorm;
    hs.breakdown_factor = opt.breakdown_tol_factor * kU53;
    hs.floor_roundoff = floor_u;
    hs.max_restarts = (int32_t)opt.max_restarts;
    HPBJ_CUDA(cudaMemcpyAsync(c->d_st, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));

    // r = b - A*0, ||r|| (gmres.cpp:223-230)
    launch_residual(sys(c), sys_plan(c), c->d_xp, c->d_bp, c->d_r, c->d_st, c->d_red, st, &c->launches);
    HPBJ_CUDA(cudaMemcpyAsync(&hs, c->d_st, sizeof(hs), cudaMemcpyDeviceToHost, st));
    HPBJ_CUDA(cudaStreamSynchronize(st));
    double rnorm = hs.rnorm;
    push_hist(0, 0, rnorm / bnorm);
    R.final_residual = rnorm / bnorm;
    if (rnorm <= thr) {
        R.converged = 1;
    } else {
        const bool use_graph = !c->profiling && c->use_graph;
        c->fused = c->use_fused && c->active == kPcBJ && c->neumann <= 0 ? plan_fused(n, c->s, c->dmax, c->num_sms, m, c->planB.n_long > 0,
                                             host_brp(c), c->spk_rows != 0)
                                : FusedPlan{};
        if (c->fused.ok && getenv("HPBJ_FUSED_PROF") && !c->d_fprof) {
            HPBJ_CUDA(cudaMalloc(&c->d_fprof, 8 * sizeof(unsigned long long)));
            HPBJ_CUDA(cudaMemset(c->d_fprof, 0, 8 * sizeof(unsigned long long)));
        }
        if (use_graph) {
            ensure_graph(c);
            const auto tg0 = std::chrono::steady_clock::now();
            HPBJ_CUDA(cudaGraphLaunch(c->graph_exec, st));
            if (getenv("HPBJ_DEBUG")) {
                HPBJ_CUDA(cudaStreamSynchronize(st));
                const auto tg1 = std::chrono::steady_clock::now();
                fprintf(stderr, "[hpbj] solve: pre-graph %.3f ms, graph %.3f ms\n",
                        std::chrono::duration<double, std::milli>(tg0 - t0).count(),
                        std::chrono::duration<double, std::milli>(tg1 - tg0).count());
            }
            c->launches += 0;  // kernel launches inside the graph are counted below
        } else {
            if (c->profiling) c->timer.reserve((size_t)3 * m);
            for (;;) {
                enqueue_cycle_head(c, 0);
                if (c->fused.ok) {
                    record_kernel(c, 0, true);
                    enqueue_cycle_fused(c);
                    record_kernel(c, 0, false);
                } else {
                    for (int it = 0; it < m; ++it) enqueue_step(c, 0, it);
                }
                enqueue_cycle_tail(c, 0);
                HPBJ_CUDA(cudaMemcpyAsync(&hs, c->d_st, sizeof(hs), cudaMemcpyDeviceToHost, st));
                HPBJ_CUDA(cudaStreamSynchronize(st));
                if (c->profiling && c->fused.ok) {
                    // one launch per cycle; algorithmic bytes summed over its steps
                    float ms = 0.f;
                    HPBJ_CUDA(cudaEventElapsedTime(&ms, c->timer.ev[0], c->timer.ev[1]));
                    hpbj_kernel_stat& ks = c->stats[HPBJ_K_CYCLE];
                    ks.launches += 1;
                    ks.total_ms += ms;
                    ks.steps += hs.last_steps;
                    for (int j = 0; j < hs.last_steps; ++j) ks.total_bytes += fused_step_bytes(c, j);
                } else if (c->profiling) {
                    for (int it = 0; it < hs.last_steps; ++it)
                        for (int k = 0; k < 3; ++k) {
                            float ms = 0.f;
                            HPBJ_CUDA(cudaEventElapsedTime(&ms, c->timer.ev[2 * (3 * it + k)],
                                                           c->timer.ev[2 * (3 * it + k) + 1]));
                            c->stats[k].launches += 1;
                            c->stats[k].total_ms += ms;
                            c->stats[k].steps += 1;
                            c->stats[k].total_bytes += k == 0   ? apply_bytes(c)
                                                       : k == 1 ? spmv_bytes(c)
                                                                : orth_bytes(c, it);
                        }
                }
                if (hs.converged || hs.cycles >= hs.max_restarts || hs.last_steps == 0) break;
            }
        }
        HPBJ_CUDA(cudaMemcpyAsync(&hs, c->d_st, sizeof(hs), cudaMemcpyDeviceToHost, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
        if (use_graph && c->fused.ok)  // per cycle: init, arnoldi_cycle, solve_y, update, residual, end
            c->launches += (int64_t)hs.cycles * 6;
        else if (use_graph)  // per step: apply(s), spmv(s), orth; per cycle: init, solve_y, update, residual, end
            c->launches += (int64_t)hs.total_iterations * step_launches(c) + (int64_t)hs.cycles * cycle_launches(c);
        std::vector<double> hv(hs.hist_len), cr(hs.cycles);
        std::vector<int> hc(hs.hist_len);
        if (hs.hist_len) {
            HPBJ_CUDA(cudaMemcpyAsync(hv.data(), kb.hist, sizeof(double) * hs.hist_len, cudaMemcpyDeviceToHost, st));
            HPBJ_CUDA(cudaMemcpyAsync(hc.data(), kb.hist_cycle, sizeof(int) * hs.hist_len, cudaMemcpyDeviceToHost, st));
        }
        if (hs.cycles)
            HPBJ_CUDA(cudaMemcpyAsync(cr.data(), kb.cycres, sizeof(double) * hs.cycles, cudaMemcpyDeviceToHost, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < hs.hist_len; ++k) push_hist(hc[k], k + 1, hv[k]);
        for (int k = 0; k < hs.cycles; ++k) {
            if (cycle_res && clen < cyc_cap) cycle_res[clen] = cr[k];
            ++clen;
        }
        if (c->d_fprof && c->fused.ok) {
            unsigned long long t[4];
            HPBJ_CUDA(cudaMemcpy(t, c->d_fprof, sizeof(t), cudaMemcpyDeviceToHost));
            HPBJ_CUDA(cudaMemset(c->d_fprof, 0, sizeof(t)));
            const double k = 1e-3 / std::max(1, hs.total_iterations);
            fprintf(stderr, "[hpbj fused] grid %d slice %d: us/step apply+b1 %.2f spmv %.2f passA+b2 %.2f passB+b3 %.2f\n",
                    c->fused.grid, c->fused.slice, t[0] * k, t[1] * k, t[2] * k, t[3] * k);
        }
        R.converged = hs.converged;
        R.total_iterations = hs.total_iterations;
        R.breakdown = hs.breakdown_any;
        R.ls_rank_deficient = hs.rank_any;
        R.restarts = hs.cycles > 0 ? hs.cycles - 1 : 0;
        R.final_residual = hs.rnorm / bnorm;
    }
    from_frame(c, c->d_xp, d_x);
    HPBJ_CUDA(cudaStreamSynchronize(st));
    R.history_len = hlen;
    R.cycles = clen;
    R.ms_solve = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (rep) *rep = R;
}

}  // namespace

// ============================================================================
// guard() for context entry points (errors land in the context's slot).
template <class F>
int cguard(hpbj_ctx* ctx, F&& f) {
    return guard(&ctx->err, std::forward<F>(f));
}

extern "C" {

int hpbj_create(hpbj_ctx** out, int device) {
    if (!out) return HPBJ_EINVAL;
    *out = nullptr;
    return guard(nullptr, [&] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            fail(HPBJ_ENODEV, "hpbj: no CUDA device (there is no CPU fallback)");
        if (device < 0 || device >= count) fail(HPBJ_EINVAL, "hpbj: bad device index");
        HPBJ_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        HPBJ_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) fail(HPBJ_ENODEV, "hpbj: needs an sm_100a (Blackwell) device");
        auto* c = new hpbj_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        HPBJ_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        HPBJ_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
        HPBJ_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        HPBJ_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        const char* ng = getenv("HPBJ_NOGRAPH");
        c->use_graph = !(ng && ng[0] == '1');
        const char* nf = getenv("HPBJ_FUSED");
        c->use_fused = !(nf && nf[0] == '0');
        const char* pz = getenv("HPBJ_POISON");
        c->pool.poison = pz && pz[0] == '1';
        if (const char* e = getenv("HPBJ_SPK_ROWS")) c->spk_rows_env = e[0] == '1' ? 1 : 0;
        if (const char* e = getenv("HPBJ_APPLY_PF")) c->apply_pf = e[0] == '1' ? 1 : 0;
        *out = c;
    });
}

void hpbj_destroy(hpbj_ctx* ctx) { delete ctx; }

const char* hpbj_last_error(const hpbj_ctx* ctx) { return ctx ? ctx->err.c_str() : thread_error(); }

int64_t hpbj_kernel_launches(const hpbj_ctx* ctx) { return ctx ? ctx->launches : 0; }

int hpbj_set_profiling(hpbj_ctx* ctx, int enable) {
    if (!ctx) return HPBJ_EINVAL;
    ctx->profiling = enable != 0;
    for (auto& s : ctx->stats) s = hpbj_kernel_stat{};
    return HPBJ_OK;
}

int hpbj_get_kernel_stats(hpbj_ctx* ctx, hpbj_kernel_stat* out) {
    if (!ctx || !out) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        for (int k = 0; k < HPBJ_K_COUNT; ++k) {
            out[k] = ctx->stats[k];
            out[k].bytes_per_launch = out[k].launches ? out[k].total_bytes / (double)out[k].launches : 0.0;
        }
    });
}

int hpbj_set_graph(hpbj_ctx* ctx, int enable) {
    if (!ctx) return HPBJ_EINVAL;
    ctx->use_graph = enable != 0;
    return HPBJ_OK;
}

int hpbj_set_fused(hpbj_ctx* ctx, int enable) {
    if (!ctx) return HPBJ_EINVAL;
    ctx->use_fused = enable != 0;
    return HPBJ_OK;
}

// The matrix after validation: int64 -> int32 indices and the FP64 values
// straight into pinned staging (nthr threads), asynchronous copies on the
// context stream (they overlap the caller's partition_graph), the SpMV plan.
// (Staging on a worker thread during partition_graph was measured: no gain —
// the partitioner's latency-bound BFS slows down by about the time saved.)
static void set_matrix_stage(hpbj_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val,
                             int nthr) {
    const auto t1 = std::chrono::steady_clock::now();
    HPBJ_CUDA(cudaSetDevice(ctx->device));
    ctx->release_matrix();
    ctx->release_ws();
    const int ni = (int)n, nnz = (int)row_ptr[n];
    const size_t b_rp = sizeof(int) * ((size_t)ni + 1), b_ci = sizeof(int) * (size_t)nnz;
    const size_t o_ci = (b_rp + 15) & ~(size_t)15, o_val = (o_ci + b_ci + 15) & ~(size_t)15;
    char* stg = static_cast<char*>(ctx->stage_mat.get(o_val + sizeof(double) * (size_t)nnz));
    int* rp = reinterpret_cast<int*>(stg);
    int* ci = reinterpret_cast<int*>(stg + o_ci);
    double* vs = reinterpret_cast<double*>(stg + o_val);
    if ((int64_t)ctx->h_rp.size() < n + 1) ctx->h_rp.resize(n + 1);
    int* hrp = ctx->h_rp.data();
#pragma omp parallel num_threads(nthr)
    {
#pragma omp for schedule(static) nowait
        for (int64_t i = 0; i <= n; ++i) rp[i] = hrp[i] = (int)row_ptr[i];
#pragma omp for schedule(static) nowait
        for (int64_t k = 0; k < nnz; ++k) ci[k] = (int)col[k];
#pragma omp for schedule(static)
        for (int64_t k = 0; k < nnz; ++k) vs[k] = val[k];
    }
    const auto t2 = std::chrono::steady_clock::now();
    ctx->A.n = ni;
    ctx->A.nnz = nnz;
    dslot(ctx->A.rp, ni + 1);
    dslot(ctx->A.ci, nnz);
    dslot(ctx->A.val, nnz);
    cudaStream_t st = ctx->stream;
    HPBJ_CUDA(cudaMemcpyAsync(ctx->A.rp, rp, b_rp, cudaMemcpyHostToDevice, st));
    HPBJ_CUDA(cudaMemcpyAsync(ctx->A.ci, ci, b_ci, cudaMemcpyHostToDevice, st));
    HPBJ_CUDA(cudaMemcpyAsync(ctx->A.val, vs, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice, st));
    ctx->stage_mat.fence(st);  // later work on the stream is ordered after the copies
    const auto t3 = std::chrono::steady_clock::now();
    make_plan(ctx->planA, ctx->h_rp.data(), ni);
    dslot(ctx->d_tmpx, ni);
    dslot(ctx->d_tmpy, ni);
    ctx->has_matrix = true;
    if (getenv("HPBJ_DEBUG")) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        fprintf(stderr, "[hpbj] set_matrix: stage %.1f alloc+enqueue %.1f plan %.1f ms\n", ms(t1, t2), ms(t2, t3),
                ms(t3, std::chrono::steady_clock::now()));
    }
}

static void check_matrix_args(int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val) {
    check_csr(n, row_ptr, col, val);
    if (n >= (int64_t)INT32_MAX || row_ptr[n] >= (int64_t)INT32_MAX) fail(HPBJ_EINVAL, "hpbj: n and nnz must be < 2^31");
}

int hpbj_set_matrix(hpbj_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        check_matrix_args(n, row_ptr, col, val);
        set_matrix_stage(ctx, n, row_ptr, col, val, omp_get_max_threads());
    });
}

int hpbj_update_values(hpbj_ctx* ctx, const double* val) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_matrix) fail(HPBJ_ELOGIC, "update_values: no matrix");
        HPBJ_CUDA(cudaMemcpyAsync(ctx->A.val, val, sizeof(double) * ctx->A.nnz, cudaMemcpyHostToDevice,
                                  ctx->stream));
        // The block-Jacobi solve runs in the permuted frame: its SpMV and true
        // residual read B = Q A Q^T, so B's values follow A now. The factors
        // stay those of the matrix they were built from (a lagged
        // preconditioner, as a reference Preconditioner is immutable) until
        // hpbj_bj_refactor.
        if (ctx->d_src && ctx->B.val)
            launch_gather_values(ctx->d_src, ctx->A.val, ctx->B.val, ctx->B.nnz, ctx->stream, &ctx->launches);
        HPBJ_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int hpbj_spmv(hpbj_ctx* ctx, const double* x, double* y) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_matrix) fail(HPBJ_ELOGIC, "spmv: no matrix");
        const int n = ctx->A.n;
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_tmpx, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        launch_spmv_f64x(ctx->A, ctx->planA, ctx->d_tmpx, ctx->d_tmpy, ctx->stream, &ctx->launches);
        HPBJ_CUDA(cudaMemcpyAsync(y, ctx->d_tmpy, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        HPBJ_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int hpbj_bj_setup(hpbj_ctx* ctx, int64_t s, const int64_t* perm, const int64_t* block_starts, double eps_pivot,
                  hpbj_setup_info* info) {
    if (!ctx) return HPBJ_EINVAL;
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->singular_block = info->singular_column = -1;
    }
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_matrix) fail(HPBJ_ELOGIC, "block_jacobi: no matrix");
        if (eps_pivot < 0.0) fail(HPBJ_EINVAL, "gp_lu: negative eps_pivot");
        const bool dbg = getenv("HPBJ_DEBUG") != nullptr;
        auto tnow = [] { return std::chrono::steady_clock::now(); };
        auto tms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto T0 = tnow();
        const int n = ctx->A.n;
        if (s < 1 || s > n) fail(HPBJ_EINVAL, "partition: block count must satisfy 1 <= s <= n");
        // validate the partition (targets in range here, bijection on the
        // device before the permutation kernels run; contiguous nonempty
        // blocks) and, in the same pass over the rows, collect the rows that
        // need a CTA sort after the scatter and the SpMV hub rows (permuted
        // indices)
        std::vector<int>& hperm = ctx->h_perm32;
        if ((int)hperm.size() < n) hperm.resize(n);
        const int spg = spmv_group(ctx->A.nnz, n), spthr = spmv_long_thresh(spg);
        const int* hrp = ctx->h_rp.data();
        std::vector<int> lrows, hubs;
        int maxlen = 0, bad = 0;
#pragma omp parallel if (n > 65536)
        {
            std::vector<int> lr, hb;
            int ml = 0;
#pragma omp for schedule(static) reduction(| : bad) nowait
            for (int i = 0; i < n; ++i) {
                const int64_t p = perm[i];
                if (p < 0 || p >= n) {
                    bad = 1;
                    continue;
                }
                hperm[i] = (int)p;
                const int len = hrp[i + 1] - hrp[i];
                if (len > kShortRow) {
                    lr.push_back((int)p);
                    ml = std::max(ml, len);
                    if (len > spthr) hb.push_back((int)p);
                }
            }
#pragma omp critical
            {
                lrows.insert(lrows.end(), lr.begin(), lr.end());
                hubs.insert(hubs.end(), hb.begin(), hb.end());
                maxlen = std::max(maxlen, ml);
            }
        }
        if (bad) fail(HPBJ_EINVAL, "permute_symmetric: not a bijection");
        if (block_starts[0] != 0 || block_starts[s] != n)
            fail(HPBJ_EINVAL, "block_jacobi: partition does not cover the matrix");
        std::vector<int> bst(s + 1);
        int dmin = n, dmax = 0;
        for (int64_t b = 0; b < s; ++b) {
            const int64_t d = block_starts[b + 1] - block_starts[b];
            if (d <= 0) fail(HPBJ_EINVAL, "partition: block " + std::to_string(b) + " is empty");
            dmin = std::min<int>(dmin, (int)d);
            dmax = std::max<int>(dmax, (int)d);
            bst[b] = (int)block_starts[b];
        }
        bst[s] = n;
        const auto T1 = tnow();
        ctx->release_pc();
        cudaStream_t st = ctx->stream;
        ctx->s = (int)s;
        ctx->eps = eps_pivot;
        ctx->dmin = dmin;
        ctx->dmax = dmax;
        ctx->h_bstart = bst;
        ctx->h_fac_off.resize(s);
        int64_t off = 0;
        for (int64_t b = 0; b < s; ++b) {
            ctx->h_fac_off[b] = off;
            off += panel_floats(bst[b + 1] - bst[b]);
        }
        ctx->fac_floats = off;
        std::vector<int> hps(s + 1, 0);
        for (int64_t b = 0; b < s; ++b) hps[b + 1] = hps[b] + (bst[b + 1] - bst[b] + 31) / 32;
        ctx->num_panels = hps[s];
        const int nnz = ctx->A.nnz;
        dslot(ctx->d_perm, n);
        ctx->B.n = n;
        ctx->B.nnz = nnz;
        dslot(ctx->B.rp, n + 1);
        dslot(ctx->B.ci, nnz);
        dslot(ctx->B.val, nnz);
        dslot(ctx->d_src, nnz);
        dslot(ctx->d_bstart, s + 1);
        dslot(ctx->d_fac_off, s);
        dslot(ctx->d_fac, off);
        dslot(ctx->d_piv, n);
        dslot(ctx->d_pert_count, s);
        dslot(ctx->d_pert, 4096);
        dslot(ctx->d_pert_n, 1);
        dslot(ctx->d_lu_next, 1);
        dslot(ctx->d_singular, 1);
        const int np = ctx->num_panels;
        dslot(ctx->d_pstart, s + 1);
        dslot(ctx->d_panel_block, np);
        dslot(ctx->d_ent_count, np);
        dslot(ctx->d_ent_count_rows, np);
        dslot(ctx->d_spk_totals, 2);
        dslot(ctx->d_rmeta, (size_t)np * 64);
        dslot(ctx->d_rowcnt, (size_t)np * 64);
        dslot(ctx->d_ent_off, np + 1);
        dslot(ctx->d_scan_tmp, 16384);
        dslot(ctx->d_desc, np);
        dslot(ctx->d_dtile, (size_t)np * kTileFloats);
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_pstart, hps.data(), sizeof(int) * (s + 1), cudaMemcpyHostToDevice, st));
        {  // LU schedule: largest blocks first (counting sort on the size, stable)
            std::vector<int>& ord = ctx->h_lu_order;
            ord.resize(s);
            std::vector<int> cnt(dmax + 2, 0);
            for (int64_t b = 0; b < s; ++b) ++cnt[dmax - (bst[b + 1] - bst[b])];
            for (int k = 0, acc = 0; k <= dmax; ++k) {
                const int c0 = cnt[k];
                cnt[k] = acc;
                acc += c0;
            }
            for (int64_t b = 0; b < s; ++b) ord[cnt[dmax - (bst[b + 1] - bst[b])]++] = (int)b;
            dslot(ctx->d_lu_order, s);
            HPBJ_CUDA(cudaMemcpyAsync(ctx->d_lu_order, ord.data(), sizeof(int) * s, cudaMemcpyHostToDevice, st));
        }
        const size_t scr = block_lu_scratch_floats(dmax, ctx->num_sms, &ctx->lu_smem_dim, &ctx->lu_scratch_ld);
        if (scr) dslot(ctx->d_lu_scratch, scr);
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_perm, hperm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_bstart, bst.data(), sizeof(int) * (s + 1), cudaMemcpyHostToDevice, st));
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_fac_off, ctx->h_fac_off.data(), sizeof(int64_t) * s,
                                  cudaMemcpyHostToDevice, st));
        const auto T2 = tnow();
        ctx->n_long_sort = (int)lrows.size();
        ctx->max_long_sort = maxlen;
        if (!lrows.empty()) {
            dslot(ctx->d_long_sort, lrows.size());
            HPBJ_CUDA(cudaMemcpyAsync(ctx->d_long_sort, lrows.data(), sizeof(int) * lrows.size(),
                                      cudaMemcpyHostToDevice, st));
        }
        set_plan(ctx->planB, spg, hubs);
        const auto T3 = tnow();
        int* tmp = dalloc<int>((size_t)n + 8192);
        {
            launch_perm_check(n, ctx->d_perm, reinterpret_cast<unsigned*>(tmp), tmp + n, st, &ctx->launches);
            int hbad = 0;
            HPBJ_CUDA(cudaMemcpyAsync(&hbad, tmp + n, sizeof(int), cudaMemcpyDeviceToHost, st));
            HPBJ_CUDA(cudaStreamSynchronize(st));
            if (hbad) {
                dput(tmp);
                fail(HPBJ_EINVAL, "permute_symmetric: not a bijection");
            }
        }
        ctx->h_brp_valid = false;
        cudaEvent_t e0, e1;
        HPBJ_CUDA(cudaEventCreate(&e0));
        HPBJ_CUDA(cudaEventCreate(&e1));
        HPBJ_CUDA(cudaEventRecord(e0, st));
        launch_permute_pattern(ctx->A, ctx->d_perm, ctx->B, ctx->d_src, tmp, ctx->d_long_sort, ctx->n_long_sort,
                               ctx->max_long_sort, st, &ctx->launches);
        HPBJ_CUDA(cudaEventRecord(e1, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        HPBJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        dput(tmp);
        ctx->has_pc = true;
        ctx->active = kPcBJ;
        const auto T4 = tnow();
        factor(ctx, info);
        if (info) info->ms_permute = ms;
        if (dbg)
            fprintf(stderr, "[hpbj] bj_setup host: validate %.3f alloc+h2d %.3f longrows+plan %.3f permute(sync) %.3f "
                            "factor %.3f ms\n", tms(T0, T1), tms(T1, T2), tms(T2, T3), tms(T3, T4), tms(T4, tnow()));
    });
}

int hpbj_bj_refactor(hpbj_ctx* ctx, hpbj_setup_info* info) {
    if (!ctx) return HPBJ_EINVAL;
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->singular_block = info->singular_column = -1;
    }
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->d_fac) fail(HPBJ_ELOGIC, "refactor: no block-Jacobi partition set up");
        ctx->has_pc = true;
        ctx->active = kPcBJ;
        factor(ctx, info);
    });
}

int hpbj_bj_apply(hpbj_ctx* ctx, const double* v, double* z) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_pc) fail(HPBJ_ELOGIC, "apply: block-Jacobi preconditioner not set up");
        const int n = ctx->A.n;
        cudaStream_t st = ctx->stream;
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_tmpx, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        launch_permute_vec(n, ctx->d_perm, ctx->d_tmpx, ctx->d_tmpy, false, st, &ctx->launches);
        launch_apply_vec(spk_view(ctx), ctx->d_tmpy, ctx->d_tmpx, st, &ctx->launches);
        launch_permute_vec(n, ctx->d_perm, ctx->d_tmpx, ctx->d_tmpy, true, st, &ctx->launches);
        HPBJ_CUDA(cudaMemcpyAsync(z, ctx->d_tmpy, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
    });
}

int hpbj_ilu0_setup(hpbj_ctx* ctx, hpbj_setup_info* info) {
    if (!ctx) return HPBJ_EINVAL;
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->singular_block = info->singular_column = -1;
    }
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_matrix) fail(HPBJ_ELOGIC, "ilu0: no matrix");
        const int n = ctx->A.n;
        const int64_t nnz = ctx->A.nnz;
        cudaStream_t st = ctx->stream;
        if (ctx->active == kPcIlu) ctx->active = kPcNone;
        ctx->has_ilu = false;
        dslot(ctx->d_ilu_lu, nnz);
        dslot(ctx->d_ilu_dpos, n);
        dslot(ctx->d_ilu_flags, n);
        dslot(ctx->d_ilu_ytag, n);
        dslot(ctx->d_ilu_ztag, n);
        dslot(ctx->d_ilu_tick32, 4);
        dslot(ctx->d_ilu_tick64, 1);
        dslot(ctx->d_ilu_err, 1);
        const size_t ldv = ((size_t)n + 31) / 32 * 32;
        dslot(ctx->d_ilu_z, ldv);
        dslot(ctx->d_ilu_u, ldv);
        const auto t0 = std::chrono::steady_clock::now();
        const int bad = launch_ilu0_diag(n, ctx->A.rp, ctx->A.ci, ctx->d_ilu_dpos, ctx->d_ilu_tick32, st,
                                         &ctx->launches);
        if (bad >= 0) {
            if (info) info->singular_column = bad;
            fail(HPBJ_EINVAL, "ilu0: structurally zero diagonal in row " + std::to_string(bad));
        }
        IluParams& p = ctx->ilu;
        p.n = n;
        p.rp = ctx->A.rp;
        p.ci = ctx->A.ci;
        p.dpos = ctx->d_ilu_dpos;
        p.lu = ctx->d_ilu_lu;
        p.nch = ilu0_chunks(n);
        p.flags = ctx->d_ilu_flags;
        p.ytag = ctx->d_ilu_ytag;
        p.ztag = ctx->d_ilu_ztag;
        p.ticket32 = ctx->d_ilu_tick32;
        p.ticket64 = ctx->d_ilu_tick64;
        p.apply_grid = ilu0_apply_grid(n, ctx->num_sms);
        const unsigned long long none = ~0ull;
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_ilu_err, &none, sizeof(none), cudaMemcpyHostToDevice, st));
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_ilu_lu, ctx->A.val, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st));
        launch_ilu0_factor(p, ctx->d_ilu_err, ctx->num_sms, st, &ctx->launches);
        unsigned long long err = none;
        HPBJ_CUDA(cudaMemcpyAsync(&err, ctx->d_ilu_err, sizeof(err), cudaMemcpyDeviceToHost, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
        int zero_row = err != none ? (int)(err & 0xffffffffu) : launch_ilu0_zero_diag(p, ctx->d_ilu_tick32, st,
                                                                                      &ctx->launches);
        if (info) info->ms_factor = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (zero_row >= 0) {
            if (info) info->singular_column = zero_row;
            fail(HPBJ_ERUNTIME, "ilu0: zero diagonal pivot in row " + std::to_string(zero_row));
        }
        ilu0_choose_apply(p, ctx->d_tmpx, ctx->d_tmpy, st, &ctx->launches);
        ctx->has_ilu = true;
        ctx->active = kPcIlu;
    });
}

int hpbj_identity_setup(hpbj_ctx* ctx) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_matrix) fail(HPBJ_ELOGIC, "identity: no matrix");
        dslot(ctx->d_ilu_z, ((size_t)ctx->A.n + 31) / 32 * 32);
        ctx->active = kPcIdentity;
    });
}

int hpbj_precond_apply(hpbj_ctx* ctx, const double* v, double* z) {
    if (!ctx) return HPBJ_EINVAL;
    if (ctx->active == kPcBJ) return hpbj_bj_apply(ctx, v, z);
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (ctx->active == kPcNone) fail(HPBJ_ELOGIC, "apply: no preconditioner set up");
        const int n = ctx->A.n;
        cudaStream_t st = ctx->stream;
        if (ctx->active == kPcIdentity) {
            std::memcpy(z, v, sizeof(double) * n);
            return;
        }
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_tmpx, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        launch_ilu0_apply(ctx->ilu, ctx->d_tmpx, nullptr, 0, nullptr, ctx->d_tmpy, nullptr, st, &ctx->launches);
        HPBJ_CUDA(cudaMemcpyAsync(z, ctx->d_tmpy, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
    });
}

int hpbj_get_ilu0_values(hpbj_ctx* ctx, double* lu) {
    if (!ctx) return HPBJ_EINVAL;
    return cguard(ctx, [&] {
        if (!ctx->has_ilu) fail(HPBJ_ELOGIC, "ilu0: factors not set up");
        HPBJ_CUDA(cudaMemcpy(lu, ctx->d_ilu_lu, sizeof(double) * ctx->A.nnz, cudaMemcpyDeviceToHost));
    });
}

int hpbj_bj_set_neumann_order(hpbj_ctx* ctx, int order) {
    if (!ctx) return HPBJ_EINVAL;
    return cguard(ctx, [&] {
        ctx->neumann = order;  // <= 0: direct block solves (gmres.cpp:93 tests > 0)
    });
}

int hpbj_bj_apply_neumann(hpbj_ctx* ctx, const double* v, double* z, int k) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_pc) fail(HPBJ_ELOGIC, "apply_neumann: block factors not available");
        if (k < 0 || k > ctx->neumann)
            fail(HPBJ_EINVAL, "apply_neumann: order exceeds the one the preconditioner was built with");
        const int n = ctx->A.n;
        cudaStream_t st = ctx->stream;
        dslot(ctx->d_nterm32, n);
        dslot(ctx->d_z32, n);
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_tmpx, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        launch_permute_vec(n, ctx->d_perm, ctx->d_tmpx, ctx->d_tmpy, false, st, &ctx->launches);
        // apply_neumann<float>: term = acc = M^-1 v; k times: term -= M^-1 A term, acc += term
        launch_apply_neumann_f32(spk_view(ctx), ctx->d_tmpy, nullptr, 0, ctx->d_nterm32, ctx->d_z32,
                                 k == 0 ? ctx->d_tmpx : nullptr, 1, nullptr, st, &ctx->launches);
        for (int i = 1; i <= k; ++i) {
            launch_spmv_f32x(ctx->B, ctx->planB, ctx->d_nterm32, ctx->d_tmpy, nullptr, st, &ctx->launches);
            launch_apply_neumann_f32(spk_view(ctx), ctx->d_tmpy, nullptr, 0, ctx->d_nterm32, ctx->d_z32,
                                     i == k ? ctx->d_tmpx : nullptr, 0, nullptr, st, &ctx->launches);
        }
        launch_permute_vec(n, ctx->d_perm, ctx->d_tmpx, ctx->d_tmpy, true, st, &ctx->launches);
        HPBJ_CUDA(cudaMemcpyAsync(z, ctx->d_tmpy, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        HPBJ_CUDA(cudaStreamSynchronize(st));
    });
}

int hpbj_get_block_factors(hpbj_ctx* ctx, int64_t block, int64_t* dim, float* f, int64_t* pivot_rows) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_pc) fail(HPBJ_ELOGIC, "factors: block-Jacobi preconditioner not set up");
        if (block < 0 || block >= ctx->s) fail(HPBJ_ERANGE, "factors: block index out of range");
        const int o = ctx->h_bstart[block];
        const int d = ctx->h_bstart[block + 1] - o;
        if (dim) *dim = d;
        const int64_t pf = panel_floats(d);
        std::vector<float> packed(pf);
        std::vector<int> piv(d);
        HPBJ_CUDA(cudaMemcpy(packed.data(), ctx->d_fac + ctx->h_fac_off[block], sizeof(float) * pf,
                             cudaMemcpyDeviceToHost));
        HPBJ_CUDA(cudaMemcpy(piv.data(), ctx->d_piv + o, sizeof(int) * d, cudaMemcpyDeviceToHost));
        const int dp4 = (d + 3) & ~3;
        if (f)
            for (int k = 0; k < d; ++k)
                for (int c2 = 0; c2 < d; ++c2)
                    f[(size_t)k * d + c2] =
                        packed[(size_t)(k / 32) * 32 * dp4 + (c2 / 4) * 128 + (k % 32) * 4 + (c2 % 4)];
        if (pivot_rows)
            for (int k = 0; k < d; ++k) pivot_rows[k] = piv[k];
    });
}

int hpbj_get_block_diagnostics(hpbj_ctx* ctx, double* cond_estimate, double* error_bound) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_pc) fail(HPBJ_ELOGIC, "diagnostics: block-Jacobi preconditioner not set up");
        if (!ctx->diag_valid) {
            dslot(ctx->d_cond, ctx->s);
            dslot(ctx->d_ebound, ctx->s);
            DiagParams p{ctx->s, ctx->dmax, ctx->d_bstart, ctx->d_fac_off, ctx->d_fac, ctx->d_piv, ctx->B,
                         ctx->d_cond, ctx->d_ebound};
            launch_block_cond(p, ctx->num_sms, ctx->stream, &ctx->launches);
            ctx->diag_valid = true;
        }
        if (cond_estimate)
            HPBJ_CUDA(cudaMemcpyAsync(cond_estimate, ctx->d_cond, sizeof(double) * ctx->s, cudaMemcpyDeviceToHost,
                                      ctx->stream));
        if (error_bound)
            HPBJ_CUDA(cudaMemcpyAsync(error_bound, ctx->d_ebound, sizeof(double) * ctx->s, cudaMemcpyDeviceToHost,
                                      ctx->stream));
        HPBJ_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int hpbj_get_block_stats(hpbj_ctx* ctx, int64_t* dims, int64_t* perturbations) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_pc) fail(HPBJ_ELOGIC, "stats: block-Jacobi preconditioner not set up");
        std::vector<int> pc(ctx->s);
        HPBJ_CUDA(cudaMemcpy(pc.data(), ctx->d_pert_count, sizeof(int) * ctx->s, cudaMemcpyDeviceToHost));
        for (int b = 0; b < ctx->s; ++b) {
            if (dims) dims[b] = ctx->h_bstart[b + 1] - ctx->h_bstart[b];
            if (perturbations) perturbations[b] = pc[b];
        }
    });
}

void hpbj_gmres_default_opts(hpbj_gmres_opts* o) {
    if (!o) return;
    o->restart_m = 50;
    o->tol = 1e-8;
    o->max_restarts = 40;
    o->absolute_tol = 0;
    o->reserved = 0;
    o->breakdown_tol_factor = 1e2;
    o->floor_roundoff = kU24;
}

int hpbj_gmres(hpbj_ctx* ctx, const double* b, double* x, const hpbj_gmres_opts* opts, hpbj_report* rep,
               hpbj_history_point* hist, int64_t hist_cap, double* cycle_res, int64_t cyc_cap) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] {
        if (!ctx->has_matrix) fail(HPBJ_ELOGIC, "gmres: no matrix");
        const int n = ctx->A.n;
        ensure_ws(ctx, (int)checked_opts(opts).restart_m);
        double* sb = static_cast<double*>(ctx->stage_vec.get(sizeof(double) * 2 * (size_t)n));
        double* sx = sb + n;
#pragma omp parallel for schedule(static) if (n > 65536)
        for (int i = 0; i < n; ++i) sb[i] = b[i];
        HPBJ_CUDA(cudaMemcpyAsync(ctx->d_bo, sb, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        solve(ctx, ctx->d_bo, ctx->d_xo, opts, rep, hist, hist_cap, cycle_res, cyc_cap);
        HPBJ_CUDA(cudaMemcpyAsync(sx, ctx->d_xo, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
        HPBJ_CUDA(cudaStreamSynchronize(ctx->stream));
#pragma omp parallel for schedule(static) if (n > 65536)
        for (int i = 0; i < n; ++i) x[i] = sx[i];
    });
}

int hpbj_gmres_device(hpbj_ctx* ctx, const double* d_b, double* d_x, const hpbj_gmres_opts* opts,
                      hpbj_report* rep, hpbj_history_point* hist, int64_t hist_cap, double* cycle_res,
                      int64_t cyc_cap) {
    if (!ctx) return HPBJ_EINVAL;
    t_pool = &ctx->pool;
    t_slots = &ctx->slots;
    return cguard(ctx, [&] { solve(ctx, d_b, d_x, opts, rep, hist, hist_cap, cycle_res, cyc_cap); });
}

}  // extern "C"
