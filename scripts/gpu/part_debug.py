"""Host partitioner phase timings (HPBJ_DEBUG=1 prints them) on this host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
for _ in range(4):
    t = time.perf_counter()
    hp.partition_graph(a, s.num_blocks, 0.1)
    print(f"partition_graph {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr, flush=True)
