"""Dev helper: setup + solve one config on the GPU, print timings/iterations."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

for c in [int(a) for a in sys.argv[1:]] or [0, 1]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    for rep in range(3):
        t0 = time.perf_counter()
        part = hp.partition_graph(a, s.num_blocks, 0.1)
        t1 = time.perf_counter()
        ctx = hp.Context(0)
        t2 = time.perf_counter()
        p = hp.Preconditioner.block_jacobi(a, part, ctx=ctx)
        t3 = time.perf_counter()
        ctx.set_profiling(True)
        r = hp.hybrid_restart_gmres(a, p, s.b, hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts))
        t4 = time.perf_counter()
        st = ctx.kernel_stats()
        err = np.linalg.norm(r.x - s.x_true) / np.linalg.norm(s.x_true)
        print(json.dumps(dict(config=c, rep=rep, part_ms=(t1-t0)*1e3, ctx_ms=(t2-t1)*1e3, setup_ms=(t3-t2)*1e3,
              permute_ms=p.info.ms_permute, factor_ms=p.info.ms_factor, solve_ms=(t4-t3)*1e3,
              its=r.report.total_iterations, conv=r.report.converged, res=r.report.final_residual, err=err,
              apply_us=1e3*st[0]['total_ms']/max(1,st[0]['launches']), spmv_us=1e3*st[1]['total_ms']/max(1,st[1]['launches']),
              mgs_us=1e3*st[2]['total_ms']/max(1,st[2]['launches']), launches=ctx.launches(), dmax=p.info.dim_max)), flush=True)
