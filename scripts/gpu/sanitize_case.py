"""Small cases for compute-sanitizer (one tool per gpurun call): the fused
Arnoldi-cycle kernel with its grid barrier (config 0, host-enqueued), the
per-kernel cycle (apply, SpMV, compact-WY orthogonalisation), the batched LU
kernels (small blocks and the left-looking kernel), and the ILU(0)
ticket/flag protocol (factorisation + sync-free triangular solves)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402
from tests import fixtures as fx  # noqa: E402

s = generate(0)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
part = hp.partition_graph(a, s.num_blocks, 0.1)
p = hp.Preconditioner.block_jacobi(a, part)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
p.ctx.set_graph(False)
for fused in (True, False):
    p.ctx.set_fused(fused)
    r = hp.hybrid_restart_gmres(a, p, s.b, cfg)
    assert r.report.converged, r.report
    print(f"config 0 fused={fused}: {r.report.total_iterations} iterations", flush=True)
# left-looking LU (blocks of 97..200 rows) on a mesh
m = fx.laplacian_2d(60, 60)
pl = hp.Preconditioner.block_jacobi(m, hp.partition_graph(m, 24, 0.1))
z = pl.apply(np.ones(m.n))
print("mesh LU + apply ok", float(np.abs(z).max()), flush=True)
# ILU(0): factorisation and the ticketed / sweep applies
pi = hp.Preconditioner.from_ilu0(a)
pi.ctx.set_graph(False)
r = hp.hybrid_restart_gmres(a, pi, s.b, hp.GmresConfig(restart_m=30, tol=1e-10, max_restarts=40, precision="double"))
assert r.report.converged
print(f"ILU(0): {r.report.total_iterations} iterations", flush=True)
