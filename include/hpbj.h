/*
 * hpbj.h — C ABI of the B200-native hybrid-precision block-Jacobi GMRES(m)
 * solver (libhpbj.so). Drop-in for the reference's C++ solver interface in
 * /root/reference/proj/include/bjgmres (arXiv 2509.09139 artifact).
 *
 * Every entry point below names the reference interface it replaces
 * (file:line under proj/). Plain pointers and sizes only; no exceptions
 * cross the ABI. Host arrays are caller-owned and copied; device memory is
 * owned by the context. A context is single-threaded (one solve at a time);
 * several contexts may coexist, each on its own CUDA stream.
 *
 * There is NO CPU fallback: every numerical step of setup and solve runs in
 * sm_100a kernels; without a CUDA device hpbj_create returns HPBJ_ENODEV.
 * Only the graph partitioning (hpbj_graph_from_matrix / hpbj_partition_graph)
 * runs on the host, by design (BASELINE.json north star), bit-identical to
 * the reference.
 *
 * Status codes map 1:1 onto the reference's exception types:
 *   HPBJ_EINVAL    -> std::invalid_argument
 *   HPBJ_ELOGIC    -> std::logic_error
 *   HPBJ_ESINGULAR -> bjgmres::SingularBlockError (lu.hpp:52-60), column via
 *                     hpbj_setup_info.singular_column
 *   HPBJ_ERANGE    -> std::out_of_range
 *   HPBJ_ECUDA / HPBJ_ENOMEM / HPBJ_ENODEV -> std::runtime_error
 */
#ifndef HPBJ_H
#define HPBJ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPBJ_OK 0
#define HPBJ_EINVAL 1
#define HPBJ_ELOGIC 2
#define HPBJ_ESINGULAR 3
#define HPBJ_ECUDA 4
#define HPBJ_ENOMEM 5
#define HPBJ_ERANGE 6
#define HPBJ_ENODEV 7
#define HPBJ_EIO 8       /* file / parse errors (std::runtime_error)        */
#define HPBJ_ERUNTIME 9  /* numerical failure (std::runtime_error), e.g. an ILU(0) zero pivot */

typedef struct hpbj_ctx hpbj_ctx;

/* Preconditioner setup outcome (PreconditionerStats, preconditioner.hpp:14-20,
 * aggregated; per-block counts via hpbj_get_block_stats). */
typedef struct hpbj_setup_info {
    int64_t num_blocks;
    int64_t dim_min;
    int64_t dim_max;
    int64_t perturbations;    /* pivots replaced by +-eps*||block||_inf (Eq. 7) */
    int64_t singular_block;   /* -1 unless HPBJ_ESINGULAR */
    int64_t singular_column;  /* SingularBlockError::column() */
    int64_t factor_bytes;     /* stored FP32 factor bytes on device */
    double ms_permute;        /* device: Q A Q^T build (CUDA events) */
    double ms_factor;         /* device: value gather + batched FP32 LU + apply-format build (CUDA events) */
    double ms_lu;             /* device: the batched LU kernel alone */
    double ms_spk;            /* device: the apply-format (SPK) build alone */
} hpbj_setup_info;

/* GmresConfig (gmres.hpp:89-97). floor_roundoff is the unit roundoff of the
 * precision the preconditioner runs in: the attainable-floor cycle break is
 * est <= 10 * floor_roundoff * beta (gmres.cpp:130-145). The FP32
 * preconditioner of this build makes it 2^-24 (0 selects that default). */
typedef struct hpbj_gmres_opts {
    int64_t restart_m;             /* default 50 */
    double tol;                    /* default 1e-8, on ||r||/||b|| unless absolute_tol */
    int64_t max_restarts;          /* default 40 */
    int32_t absolute_tol;          /* default 0 */
    int32_t reserved;
    double breakdown_tol_factor;   /* default 1e2 (u = 2^-53, FP64 basis) */
    double floor_roundoff;         /* default 2^-24 */
} hpbj_gmres_opts;

/* SolveReport (gmres.hpp:105-117). */
typedef struct hpbj_report {
    int32_t converged;
    int32_t breakdown;
    int32_t ls_rank_deficient;
    int32_t reserved;
    int64_t total_iterations;
    int64_t restarts;        /* cycles executed minus one */
    int64_t history_len;     /* rows written to hist (iteration 0 + one per step) */
    int64_t cycles;          /* rows written to cycle_res */
    double final_residual;   /* true FP64 ||b-Ax||/||b|| at exit */
    double ms_solve;         /* wall time of the solve, host clock */
} hpbj_report;

/* HistoryPoint (gmres.hpp:99-103). */
typedef struct hpbj_history_point {
    int64_t cycle;
    int64_t iteration;
    double relative_residual;
} hpbj_history_point;

/* Device timings collected while profiling is enabled (hpbj_set_profiling):
 * per kernel class, launches, summed CUDA-event time and the algorithmic
 * HBM bytes of one launch. */
typedef struct hpbj_kernel_stat {
    int64_t launches;
    double total_ms;
    double bytes_per_launch;  /* total_bytes / launches */
    int64_t steps;            /* Arnoldi steps covered by these launches */
    double total_bytes;       /* algorithmic HBM bytes of all launches */
} hpbj_kernel_stat;

#define HPBJ_K_APPLY 0   /* block forward/back substitution (Arnoldi step)       */
#define HPBJ_K_SPMV 1    /* FP64 CSR SpMV (Arnoldi step)                         */
#define HPBJ_K_MGS 2     /* compact-WY / textbook MGS + norm + Givens            */
#define HPBJ_K_CYCLE 3   /* fused Arnoldi cycle (apply+SpMV+MGS+Givens per step) */
#define HPBJ_K_COUNT 4

/* ---- context ------------------------------------------------------------ */
int hpbj_create(hpbj_ctx** out, int device);
void hpbj_destroy(hpbj_ctx* ctx);
/* Message of the last failure on ctx (or of the calling thread if ctx == NULL). */
const char* hpbj_last_error(const hpbj_ctx* ctx);
/* Kernels this context launched since creation (the driver's evidence). */
int64_t hpbj_kernel_launches(const hpbj_ctx* ctx);
int hpbj_set_profiling(hpbj_ctx* ctx, int enable);
int hpbj_get_kernel_stats(hpbj_ctx* ctx, hpbj_kernel_stat* out /* HPBJ_K_COUNT */);
/* Whole Arnoldi cycle as one persistent kernel when it fits (default on);
 * off: one apply, SpMV and orthogonalisation launch per step. */
int hpbj_set_fused(hpbj_ctx* ctx, int enable);
/* Solve as one CUDA graph with device-driven WHILE nodes (default on); off:
 * the host enqueues every kernel of every cycle (same kernels, same results;
 * each launch is visible to a profiler — HPBJ_NOGRAPH=1 sets the default). */
int hpbj_set_graph(hpbj_ctx* ctx, int enable);

/* ---- host-side partitioning (bit-identical to the reference) ------------ */
/* graph_from_matrix (graph.hpp:30, graph.cpp:17-51). Adjacency as CSR:
 * adj_start[n+1], adj_nbr/adj_w[adj_start[n]]; cap = capacity of adj_nbr/adj_w
 * (2*nnz always suffices). */
int hpbj_graph_from_matrix(int64_t n, const int64_t* row_ptr, const int64_t* col,
                           const double* val, int64_t* adj_start, int64_t* adj_nbr,
                           double* adj_w, int64_t cap);
/* partition_graph(graph_from_matrix(A), s, imbalance_tol)
 * (partition.hpp:38-39, partition.cpp:60-144) in O(nnz + n). Outputs
 * Partition::assignment[n], perm[n] (old -> new), block_starts[s+1]. */
int hpbj_partition_graph(int64_t n, const int64_t* row_ptr, const int64_t* col,
                         const double* val, int64_t s, double imbalance_tol,
                         int64_t* assignment, int64_t* perm, int64_t* block_starts);
/* Same, on an explicit graph (WeightedGraph, graph.hpp:17-25). */
int hpbj_partition_adjacency(int64_t n, const int64_t* adj_start, const int64_t* adj_nbr,
                             const double* adj_w, int64_t s, double imbalance_tol,
                             int64_t* assignment, int64_t* perm, int64_t* block_starts);
/* partition_from_assignment (partition.hpp:33, partition.cpp:14-41). */
int hpbj_partition_from_assignment(int64_t n, const int64_t* assignment, int64_t s,
                                   int64_t* perm, int64_t* block_starts);

/* ---- matrix ------------------------------------------------------------- */
/* SparseMatrix(n, n, row_starts, col_indices, values) (sparse_matrix.hpp:26-27;
 * invariants checked as sparse_matrix.cpp:14-50). Copies to the device. */
int hpbj_set_matrix(hpbj_ctx* ctx, int64_t n, const int64_t* row_ptr, const int64_t* col,
                    const double* val);
/* New values, same pattern (transient Newton sequence, config 4). */
int hpbj_update_values(hpbj_ctx* ctx, const double* val);
/* spmv<double> (spmv.hpp:31-47), original ordering, host buffers. */
int hpbj_spmv(hpbj_ctx* ctx, const double* x, double* y);

/* ---- block-Jacobi preconditioner ---------------------------------------- */
/* Preconditioner::block_jacobi(A, Partition, BlockJacobiOptions)
 * (preconditioner.hpp:60-61, preconditioner.cpp:100-153) with the Hybrid
 * policy: Q A Q^T, diagonal blocks, batched FP32 LU with partial pivoting
 * (ties -> smallest row) and Eq. 7 regularisation (lu.cpp:10-20, 134-225). */
int hpbj_bj_setup(hpbj_ctx* ctx, int64_t s, const int64_t* perm,
                  const int64_t* block_starts, double eps_pivot, hpbj_setup_info* info);
/* Numeric refactorisation for new values with the same partition. */
int hpbj_bj_refactor(hpbj_ctx* ctx, hpbj_setup_info* info);
/* Preconditioner::apply<float> (preconditioner.hpp:69-70, preconditioner.cpp:159-188),
 * original ordering; v is rounded to FP32 on load, z returned widened. */
int hpbj_bj_apply(hpbj_ctx* ctx, const double* v, double* z);
/* BlockJacobiOptions::neumann_order (preconditioner.hpp:34, preconditioner.cpp:110):
 * order k > 0 makes hpbj_gmres apply the truncated Neumann series in place of
 * the block solves (preconditioned<T>, gmres.cpp:91-95), FP32 in the Arnoldi
 * step and FP64 in the x-update. k <= 0 (default 0) = direct block solves. */
int hpbj_bj_set_neumann_order(hpbj_ctx* ctx, int order);

/* ---- other preconditioners behind the same solve ----
 * Each setup makes its preconditioner the one hpbj_gmres uses; block Jacobi
 * (hpbj_bj_setup / hpbj_bj_refactor) switches back. */
/* Preconditioner::from_ilu0 (preconditioner.cpp:94-98) with ilu0
 * (lu.cpp:227-312): FP64 factors in A's pattern, original ordering; the solve
 * applies them in FP64 (lu_solve<double>) — use floor_roundoff = 2^-53
 * (DoubleOnly), the only policy under which the reference can apply ILU(0).
 * HPBJ_EINVAL "ilu0: structurally zero diagonal in row i", HPBJ_ERUNTIME
 * "ilu0: zero diagonal pivot in row k" (info->singular_column = the row). */
int hpbj_ilu0_setup(hpbj_ctx* ctx, hpbj_setup_info* info);
/* Preconditioner::identity (preconditioner.cpp:90-92). */
int hpbj_identity_setup(hpbj_ctx* ctx);
/* Preconditioner::apply of the active preconditioner, original ordering:
 * apply<double> for ILU(0) / identity, apply<float> for block Jacobi. */
int hpbj_precond_apply(hpbj_ctx* ctx, const double* v, double* z);
/* The factored values in A's pattern: per row L (unit diagonal implied),
 * U's diagonal, U — the reference's LUFactors lower/upper concatenated. */
int hpbj_get_ilu0_values(hpbj_ctx* ctx, double* lu);
/* Preconditioner::apply_neumann<float> (preconditioner.hpp:79-83,
 * preconditioner.cpp:200-220): z = sum_{i=0..k} (I - Phi^-1 A)^i Phi^-1 v,
 * original ordering. HPBJ_ELOGIC without factors, HPBJ_EINVAL for k < 0 or
 * k > the order set with hpbj_bj_set_neumann_order. */
int hpbj_bj_apply_neumann(hpbj_ctx* ctx, const double* v, double* z, int k);
/* Per-block factors F = L_strict + U in pivot order, row-major dim x dim,
 * and LUFactors::pivot_rows (lu.hpp:37-50). */
int hpbj_get_block_factors(hpbj_ctx* ctx, int64_t block, int64_t* dim, float* f,
                           int64_t* pivot_rows);
/* PreconditionerStats::{cond_estimate, error_bound} per block
 * (cond_estimate_block / block_error_bound, preconditioner.cpp:13-88): 1-norm
 * condition estimate of each block (exact for dim <= 64, Hager otherwise) and
 * (cond*2^-53 + 2^-24)*cond. Computed on the device on first request after a
 * (re)factorisation. */
int hpbj_get_block_diagnostics(hpbj_ctx* ctx, double* cond_estimate, double* error_bound);
/* PreconditionerStats::{block_dim, perturbation_count} per block. */
int hpbj_get_block_stats(hpbj_ctx* ctx, int64_t* dims, int64_t* perturbations);

/* ---- solve -------------------------------------------------------------- */
void hpbj_gmres_default_opts(hpbj_gmres_opts* opts);
/* hybrid_restart_gmres(A, P, b, GmresConfig) (gmres.hpp:145-147,
 * gmres.cpp:200-274): host b in, host x out. hist (cap hist_cap) receives
 * SolveReport::residual_history, cycle_res (cap cyc_cap) cycle_residuals;
 * either may be NULL. */
int hpbj_gmres(hpbj_ctx* ctx, const double* b, double* x, const hpbj_gmres_opts* opts,
               hpbj_report* rep, hpbj_history_point* hist, int64_t hist_cap,
               double* cycle_res, int64_t cyc_cap);
/* Same with b and x already resident in device memory (original ordering). */
int hpbj_gmres_device(hpbj_ctx* ctx, const double* d_b, double* d_x,
                      const hpbj_gmres_opts* opts, hpbj_report* rep,
                      hpbj_history_point* hist, int64_t hist_cap, double* cycle_res,
                      int64_t cyc_cap);

/* ---- Matrix Market and binary CSR cache (host) ----------- */
/* read_matrix_market_file (matrix_market.cpp:36-106): coordinate real/integer,
 * general/symmetric, 1-based, duplicates summed as SparseMatrix::from_triplets.
 * The arrays are malloc'ed by the library; release them with hpbj_free.
 * Parse errors return HPBJ_EIO with "matrix market: line N: ..." in
 * hpbj_last_error(NULL). */
int hpbj_mm_read(const char* path, int64_t* nrows, int64_t* ncols, int64_t** row_ptr, int64_t** col,
                 double** val);
/* write_matrix_market_file (matrix_market.cpp:108-121): real general, %.17g. */
int hpbj_mm_write(const char* path, int64_t nrows, int64_t ncols, const int64_t* row_ptr, const int64_t* col,
                  const double* val);
/* Binary CSR cache ("HPBJCSR1", n, nnz, int64 row_ptr, int64 col, FP64 val). */
int hpbj_csr_cache_write(const char* path, int64_t n, const int64_t* row_ptr, const int64_t* col,
                         const double* val);
int hpbj_csr_cache_read(const char* path, int64_t* n, int64_t** row_ptr, int64_t** col, double** val);
void hpbj_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* HPBJ_H */
