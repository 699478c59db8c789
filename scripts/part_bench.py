"""Dev helper: host partition timing per config (HPBJ_DEBUG=1 prints the phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate
for c in [int(x) for x in sys.argv[1:]]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    for r in range(int(os.environ.get("REPS", "3"))):
        t0 = time.perf_counter(); p = hp.partition_graph(a, s.num_blocks, 0.1); t1 = time.perf_counter()
        print(c, r, f"{(t1-t0)*1e3:.1f} ms", flush=True)
