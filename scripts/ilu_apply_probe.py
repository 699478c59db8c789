"""Times one ILU(0) apply on a workload (profiling aid): python scripts/ilu_apply_probe.py CONFIG [REPS]."""
import sys
import time

import numpy as np

import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

c = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
p = hp.Preconditioner.from_ilu0(a)
v = np.random.default_rng(0).uniform(-1, 1, s.n)
for _ in range(reps):
    t0 = time.perf_counter()
    p.apply(v)
    print(f"apply {1e3 * (time.perf_counter() - t0):.3f} ms")
