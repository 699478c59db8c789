"""Reproducibility probe: fresh contexts, fused / per-kernel cycle, config 4
step 0 and step 1 (update_values + refactor); prints which runs are
bit-identical to the first and the largest difference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

s = generate(4)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
part = hp.partition_graph(a, s.num_blocks, 0.1)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
st1 = generate(4, step=1)
for fused in (True, False):
    out = []
    for rep in range(5):
        p = hp.Preconditioner.block_jacobi(a, part)
        p.ctx.set_fused(fused)
        x0, r0 = p.ctx.gmres(s.b, cfg)
        x0b, _ = p.ctx.gmres(s.b, cfg)
        p.ctx.update_values(st1.val)
        p.ctx.bj_refactor()
        x1, r1 = p.ctx.gmres(st1.b, cfg)
        out.append((x0, x1))
        print("fused", fused, "rep", rep, "its", r0.total_iterations, r1.total_iterations,
              "same-ctx repeat eq", np.array_equal(x0, x0b),
              "step0 eq first", np.array_equal(out[0][0], x0), float(np.max(np.abs(out[0][0] - x0))),
              "step1 eq first", np.array_equal(out[0][1], x1), float(np.max(np.abs(out[0][1] - x1))), flush=True)
