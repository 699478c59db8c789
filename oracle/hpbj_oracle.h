/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle's plain-C restatement of the
 * reference algorithm (arXiv 2509.09139 artifact, /root/reference/proj).
 * Never linked into libhpbj.so; loaded by tests/, smoke() and bench.py's
 * CPU-baseline leg only. Pinned against the real reference library
 * (oracle/_ref) and the committed golden fixtures by tests/test_oracle.py.
 *
 * Modes of orc_solve:
 *   ORC_DOUBLE  reference PrecisionMode::DoubleOnly
 *   ORC_HYBRID  reference PrecisionMode::Hybrid (FP32 Krylov loop)
 *   ORC_MIX     the B200 build's precision mix (north star): FP64 SpMV and
 *               Arnoldi, FP32 factors + FP32 block apply, floor 2^-24
 */
#ifndef HPBJ_ORACLE_H
#define HPBJ_ORACLE_H
#include <stdint.h>

#define ORC_DOUBLE 0
#define ORC_HYBRID 1
#define ORC_MIX 2

typedef struct orc_report {
    int64_t converged, total_iterations, restarts, breakdown, rank_deficient;
    int64_t hist_len, cyc_len;
    double final_residual;
    int64_t singular_block, singular_column;
} orc_report;

int orc_spmv(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x, double* y,
             int fp32);
int orc_graph(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t* st, int64_t* nb,
              double* w, int64_t cap);
int orc_partition(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s, double tol,
                  int64_t* assignment);
int orc_factors(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
                const int64_t* assignment, double eps, double* f64, int64_t* pivot_rows, int64_t* pert,
                int64_t* sing_block, int64_t* sing_col);
int orc_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
              const int64_t* assignment, double eps, int fp32, const double* vin, double* zout);
int orc_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t s,
              const int64_t* assignment, const double* b, int64_t m, double tol, int64_t max_restarts,
              int mode, double eps, double* x, orc_report* rep, double* hist, int64_t hist_cap, double* cycres,
              int64_t cyc_cap);
#endif
