"""Dev helper: per-launch time of the fused Arnoldi-cycle kernel in the
profiling path (what bench.py's roofline uses) vs the graph solve time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
ctx = hp.Context(0)
ctx.set_matrix(a)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
part = hp.partition_graph(a, s.num_blocks, 0.1)
ctx.bj_setup(part, 1e-10)
for prof in (False, True, False, True):
    ctx.set_profiling(prof)
    t0 = time.perf_counter()
    x, rep = ctx.gmres(s.b, cfg)
    t1 = time.perf_counter()
    st = ctx.kernel_stats()[3]
    ctx.set_profiling(False)
    print(f"prof={prof} solve {1e3 * (t1 - t0):.3f} ms its {rep.total_iterations} cycle launches {st['launches']} "
          f"ms/launch {st['total_ms'] / max(1, st['launches']):.3f} steps {st['steps']} "
          f"GB/s {st['total_bytes'] / max(1e-9, st['total_ms']) / 1e6:.0f}")
