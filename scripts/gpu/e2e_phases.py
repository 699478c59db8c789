"""Host-side phases of one end-to-end system (bench.py's e2e step) on the GPU
box: set_matrix (validate + stage + async H2D), partition_graph, bj_setup,
gmres with host b / x, each bracketed by a device sync."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
ctx = hp.Context(0)
for it in range(4):
    t = [time.perf_counter()]
    ctx.set_matrix(a)
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    t.append(time.perf_counter())
    ctx.bj_setup(part, 1e-10)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    x, rep = ctx.gmres(s.b, cfg)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = [1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)]
    print(f"iter {it}: set_matrix host {d[0]:.1f} + copy wait {d[1]:.1f}, partition {d[2]:.1f}, bj_setup {d[3]:.1f}, "
          f"gmres {d[4]:.1f}, total {1e3 * (t[-1] - t[0]):.1f} ms", flush=True)
