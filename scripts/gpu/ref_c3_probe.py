"""Time the reference library's stock run_spec path (graph + partition_graph +
block_jacobi + hybrid_restart_gmres) on one config-3 system on this host."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
from paper_2509_09139_b200.workloads import generate
from oracle import Ref
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t = time.time(); s = generate(c); tg = time.time() - t
R = Ref()
t = time.time()
out = R.solve(s.row_ptr, s.col, s.val, s.num_blocks, s.b, s.restart_m, s.tol, s.max_restarts, hybrid=True)
print(json.dumps({"config": c, "gen_s": tg, "wall_s": time.time() - t, "its": out.total_iterations,
                  "timings": out.timings, "cores": os.cpu_count()}), flush=True)
