"""Dev helper: setup + solve one config on the GPU, print timings/iterations."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

for c in [int(a) for a in sys.argv[1:]] or [0, 1]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    ctx = hp.Context(0)
    ctx.set_matrix(a)
    cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
    for rep in range(int(os.environ.get("REPS", "3"))):
        t0 = time.perf_counter()
        part = hp.partition_graph(a, s.num_blocks, 0.1)
        t1 = time.perf_counter()
        info = ctx.bj_setup(part, 1e-10)
        t2 = time.perf_counter()
        ctx.set_profiling(os.environ.get("PROF", "0") == "1")
        x, rep_ = ctx.gmres(s.b, cfg)
        t3 = time.perf_counter()
        st = ctx.kernel_stats()
        err = np.linalg.norm(x - s.x_true) / np.linalg.norm(s.x_true)
        print(json.dumps(dict(config=c, rep=rep, part_ms=(t1 - t0) * 1e3, setup_ms=(t2 - t1) * 1e3,
                              permute_ms=info.ms_permute, factor_ms=info.ms_factor, solve_ms=(t3 - t2) * 1e3,
                              its=rep_.total_iterations, conv=rep_.converged, res=rep_.final_residual, err=err,
                              apply_us=1e3 * st[0]['total_ms'] / max(1, st[0]['launches']),
                              spmv_us=1e3 * st[1]['total_ms'] / max(1, st[1]['launches']),
                              mgs_us=1e3 * st[2]['total_ms'] / max(1, st[2]['launches']),
                              launches=ctx.launches(), dmax=info.dim_max)), flush=True)
