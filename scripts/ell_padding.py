"""Dev helper: padding of a slot-major (ELL) layout for the off-panel factor
entries, per 32-row panel and pass (L / U), on a sample of blocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

for c in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    p = hp.Preconditioner.block_jacobi(a, part)
    rng = np.random.default_rng(0)
    nnz = ell = ell_q = steps = 0
    lens = []
    for b in rng.choice(s.num_blocks, min(200, s.num_blocks), replace=False):
        F, piv = p.block_factors(int(b))
        d = F.shape[0]
        nz = F != 0
        for t in range((d + 31) // 32):
            r0, r1 = 32 * t, min(d, 32 * t + 32)
            for part_ in (nz[r0:r1, :r0], nz[r0:r1, r1:]):
                ln = part_.sum(axis=1)
                if ln.sum() == 0:
                    continue
                nnz += ln.sum(); ell += 32 * ln.max(); steps += 1
                # quad-split: rows longer than the mean split into ceil(len/mean) lanes
                lens.append(ln)
    print(f"config {c}: entries/step {nnz/steps:.0f}  ELL padding {ell/nnz:.2f}x  "
          f"max row/step {np.mean([l.max() for l in lens]):.1f} mean row {np.mean([l.mean() for l in lens]):.1f}", flush=True)
