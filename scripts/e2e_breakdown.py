"""Dev helper: host-side breakdown of the e2e (host-buffer) path of bench.py."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate
c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
ctx = hp.Context(0)
for r in range(5):
    t0 = time.perf_counter(); ctx.set_matrix(a)
    t1 = time.perf_counter(); p = hp.partition_graph(a, s.num_blocks, 0.1)
    t2 = time.perf_counter(); ctx.bj_setup(p, 1e-10)
    t3 = time.perf_counter(); x, rep = ctx.gmres(s.b, cfg)
    t4 = time.perf_counter()
    print(f"rep {r}: set_matrix {1e3*(t1-t0):.2f} partition {1e3*(t2-t1):.2f} bj_setup {1e3*(t3-t2):.2f} "
          f"gmres {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms", flush=True)
