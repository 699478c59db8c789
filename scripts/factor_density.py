"""Dev helper: structure of the FP32 block factors (bytes of candidate layouts, per dense float = 4 B)."""
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
    tot = dict(dense=0, padded=0, nnz=0, ch4=0, ell=0, csr=0, diagcompact=0, diagdense=0)
    for b in rng.choice(s.num_blocks, min(300, s.num_blocks), replace=False):
        F, piv = p.block_factors(int(b))
        d = F.shape[0]
        T = (d + 31) // 32
        nz = F != 0
        tot["dense"] += d * d
        tot["padded"] += T * 32 * ((d + 3) // 4 * 4)
        tot["nnz"] += nz.sum()
        for t in range(T):
            r0, r1 = 32 * t, min(d, 32 * t + 32)
            rows = nz[r0:r1]
            nl = rows[:, :r0].sum(axis=1)
            nu = rows[:, r1:].sum(axis=1)
            diag = rows[:, r0:r1].sum()
            tot["ell"] += 32 * (nl.max() + nu.max()) * 1.5  # float + u16 index
            tot["csr"] += (nl.sum() + nu.sum()) * 1.5
            tot["diagcompact"] += diag + 32  # values + masks
            tot["diagdense"] += 32 * 32
            nch = 0
            for c0 in range(0, d, 4):
                if r0 <= c0 < r0 + 32:
                    continue
                if rows[:, c0:c0 + 4].any():
                    nch += 1
            tot["ch4"] += (nch * 4) * 32
    D = tot["dense"]
    print(c, {k: round(float(v) / D, 3) for k, v in tot.items()},
          "ell+diagc", round(float(tot["ell"] + tot["diagcompact"]) / D, 3),
          "csr+diagc", round(float(tot["csr"] + tot["diagcompact"]) / D, 3),
          "ch4+diagc", round(float(tot["ch4"] + tot["diagcompact"]) / D, 3), flush=True)
