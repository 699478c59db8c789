"""Dev probe: host partition time around CUDA activity (OpenMP contention check)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

s = generate(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
def part(tag):
    t0 = time.perf_counter(); p = hp.partition_graph(a, s.num_blocks, 0.1); print(f"{tag}: {(time.perf_counter()-t0)*1e3:.2f} ms", flush=True); return p
part("cold"); part("warm")
ctx = hp.Context(0); part("after ctx")
ctx.set_matrix(a); part("after set_matrix")
p = part("again")
ctx.bj_setup(p, 1e-10); part("after bj_setup")
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
ctx.gmres(s.b, cfg); part("after gmres"); part("after gmres 2")
time.sleep(0.5); part("after sleep")
ctx.gmres(s.b, cfg); time.sleep(0.05); part("after gmres+50ms")
