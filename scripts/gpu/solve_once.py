"""Setup + solve one config on the GPU through the C ABI (ncu target of
scripts/profile_round.sh): python solve_once.py CONFIG [...]; REPS systems each."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

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
        x, r = ctx.gmres(s.b, cfg)
        t3 = time.perf_counter()
        err = np.linalg.norm(x - s.x_true) / np.linalg.norm(s.x_true)
        print(json.dumps(dict(config=c, rep=rep, part_ms=(t1 - t0) * 1e3, setup_ms=(t2 - t1) * 1e3,
                              lu_ms=info.ms_lu, spk_ms=info.ms_spk, solve_ms=(t3 - t2) * 1e3,
                              its=r.total_iterations, conv=r.converged, res=r.final_residual, err=err)), flush=True)
