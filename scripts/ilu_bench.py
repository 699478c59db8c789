"""ILU(0)-GMRES (DoubleOnly) on the device vs the reference library on the
BASELINE.json workloads: factor time, solve time, iterations."""
import json
import sys
import time

import numpy as np

import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

configs = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 2]
with_ref = "--ref" in sys.argv
rows = []
for c in configs:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    m = {0: 30, 1: 50, 2: 50, 3: 50, 4: 30}[c]
    cfg = hp.GmresConfig(restart_m=m, tol=1e-10, max_restarts=40, precision="double")
    ctx = hp.Context(0)
    hp.Preconditioner.from_ilu0(a, ctx=ctx)  # warm-up (allocations, module load)
    t0 = time.perf_counter()
    p = hp.Preconditioner.from_ilu0(a, ctx=ctx)
    t_fac = (time.perf_counter() - t0) * 1e3
    out = hp.hybrid_restart_gmres(a, p, s.b, cfg)  # builds the graph
    t0 = time.perf_counter()
    out = hp.hybrid_restart_gmres(a, p, s.b, cfg)
    t_sol = (time.perf_counter() - t0) * 1e3
    v = np.random.default_rng(0).uniform(-1, 1, s.n)
    p.apply(v)
    t0 = time.perf_counter()
    for _ in range(10):
        p.apply(v)
    t_app = (time.perf_counter() - t0) * 1e2
    row = dict(config=c, n=s.n, nnz=int(s.row_ptr[-1]), factor_ms=round(t_fac, 3), solve_ms=round(t_sol, 3),
               iterations=out.report.total_iterations, converged=out.report.converged,
               apply_host_ms=round(t_app, 3), ms_per_iteration=round(t_sol / max(1, out.report.total_iterations), 4))
    if with_ref:
        from oracle import Ref
        ref = Ref()
        t0 = time.perf_counter()
        r = ref.solve_ilu0(s.row_ptr, s.col, s.val, s.b, m, 1e-10, 40, hybrid=False)
        row.update(ref_total_ms=round((time.perf_counter() - t0) * 1e3, 1), ref_iterations=r.total_iterations)
    rows.append(row)
    print(json.dumps(row), flush=True)
