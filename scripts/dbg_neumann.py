"""Debug: Neumann-order solves on the device vs the reference library."""
import sys

import numpy as np
import paper_2509_09139_b200 as hp
from oracle import Ref
from tests import fixtures as fx

ref = Ref()
for name, a, s in [("cd30", fx.convection_diffusion_2d(30, 30, 20.0, -10.0), 12),
                   ("rdd300", fx.random_dd(300, 5, 21), 6), ("lap20", fx.laplacian_2d(20, 20), 8)]:
    if len(sys.argv) > 1 and name not in sys.argv[1].split(","):
        continue
    part = hp.partition_graph(a, s, 0.1)
    b = fx.ones(a.n)
    for order in [int(o) for o in (sys.argv[2].split(',') if len(sys.argv) > 2 else '012')]:
        print('start', name, order, flush=True)
        p = hp.Preconditioner.block_jacobi(a, part, hp.BlockJacobiOptions(neumann_order=order))
        print(' setup ok', flush=True)
        out = hp.hybrid_restart_gmres(a, p, b, hp.GmresConfig(restart_m=30, tol=1e-10, max_restarts=40))
        r = out.report
        ro = ref.solve(a.row_starts, a.col_indices, a.values, s, b, 30, 1e-10, 40, hybrid=True,
                       assignment=part.assignment, neumann_order=order)
        print(name, order, "dev", r.converged, r.total_iterations, r.final_residual, [h.relative_residual for h in r.residual_history[:4]],
              "ref", ro.converged, ro.total_iterations, ro.final_residual)
