"""Dev helper (host only): time graph + partition per config, R repeats.
HPBJ_DEBUG=1 prints the phases; HPBJ_PART_PIPE=0 disables the pipelined refinement."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

for c in [int(a) for a in sys.argv[1:]] or [1]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    ts = []
    for r in range(int(os.environ.get("R", "5"))):
        t0 = time.perf_counter()
        hp.partition_graph(a, s.num_blocks, 0.1)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"config {c}: partition ms {' '.join(f'{t:.2f}' for t in ts)}", flush=True)
