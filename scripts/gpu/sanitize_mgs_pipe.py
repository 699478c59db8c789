"""compute-sanitizer case for the pipelined textbook MGS (k_mgs_pipe: flag /
data words exchanged between CTAs without a grid barrier): config 0 and a
one-CTA system, host-enqueued per-kernel cycle. Run with HPBJ_ORTH=mgs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402
from tests import fixtures as fx  # noqa: E402

assert os.environ.get("HPBJ_ORTH") == "mgs"
s = generate(0)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
p = hp.Preconditioner.block_jacobi(a, hp.partition_graph(a, s.num_blocks, 0.1))
p.ctx.set_graph(False)
p.ctx.set_fused(False)
r = hp.hybrid_restart_gmres(a, p, s.b, hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts))
assert r.report.converged
print(f"config 0 pipelined MGS: {r.report.total_iterations} iterations", flush=True)
m = fx.laplacian_2d(20, 20)
pm = hp.Preconditioner.block_jacobi(m, hp.partition_graph(m, 4, 0.1))
pm.ctx.set_graph(False)
pm.ctx.set_fused(False)
r = hp.hybrid_restart_gmres(m, pm, np.ones(m.n), hp.GmresConfig(restart_m=30, tol=1e-9, max_restarts=20))
assert r.report.converged
print(f"one-CTA pipelined MGS: {r.report.total_iterations} iterations", flush=True)
