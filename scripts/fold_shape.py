"""Dev helper: off-panel row-length structure of the FP32 block factors per
32-row panel (what the SPK apply's fold iterates over), sampled blocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate

for c in [int(a) for a in sys.argv[1:]] or [2, 3]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    p = hp.Preconditioner.block_jacobi(a, part)
    rng = np.random.default_rng(0)
    st = dict(parts=0, ent=0, seg128=0, lane4max=0, lane8max=0, pad4=0, lane4sum=0, tiles_nz=0, tiles=0)
    hist = np.zeros(10)
    for b in rng.choice(s.num_blocks, min(200, s.num_blocks), replace=False):
        F, piv = p.block_factors(int(b))
        d = F.shape[0]
        nz = F != 0
        T = (d + 31) // 32
        for t in range(T):
            r0, r1 = 32 * t, min(d, 32 * t + 32)
            rows = nz[r0:r1]
            st["tiles_nz"] += rows[:, r0:r1].sum()
            st["tiles"] += (r1 - r0) * (r1 - r0)
            for lens in (rows[:, :r0].sum(axis=1), rows[:, r1:].sum(axis=1)):
                e = int(lens.sum())
                st["parts"] += 1
                st["ent"] += e
                st["seg128"] += -(-e // 128)
                st["lane4max"] += int(np.max(-(-lens // 4))) if len(lens) else 0
                st["lane8max"] += int(np.max(-(-lens // 8))) if len(lens) else 0
                st["pad4"] += int(np.sum(-(-lens // 4) * 4))
                st["lane4sum"] += int(np.sum(-(-lens // 4)))
                if e:
                    cv = lens.std() / max(lens.mean(), 1e-9)
                    hist[min(9, int(cv * 5))] += 1
    P = st["parts"]
    print(c, "per part: entries %.1f, seg128 iters %.2f, lane4 iters(max) %.2f, lane8 %.2f, pad4 overhead %.3f, lane4 util %.2f, tile density %.2f"
          % (st["ent"] / P, st["seg128"] / P, st["lane4max"] / P, st["lane8max"] / P, st["pad4"] / max(1, st["ent"]),
             st["lane4sum"] / max(1, 32 * st["lane4max"]), st["tiles_nz"] / st["tiles"]), "cv hist", hist.astype(int).tolist(), flush=True)
