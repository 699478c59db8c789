"""e2e step variants (bench.py's e2e_step: set_matrix, partition_graph,
bj_setup, gmres with host b / x), CUDA-event timed, median of 5: the
synchronous upload vs the asynchronous one with k staging threads."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200 import _abi  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

s = generate(3)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
ctx = hp.Context(0)


def sync_set(c):
    c.check(c.lib.hpbj_set_matrix(c.h, a.n, hp._p(a.row_starts, _abi.i64p), hp._p(a.col_indices, _abi.i64p),
                                  hp._p(a.values, _abi.f64p)))


res = {"sync": [], "async T=2": [], "async T=5": []}
for it in range(8):
    for label, stage_t in (("sync", None), ("async T=2", "2"), ("async T=5", "5")):
        if stage_t:
            os.environ["HPBJ_STAGE_T"] = stage_t
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if stage_t:
            ctx.set_matrix(a)
        else:
            sync_set(ctx)
        part = hp.partition_graph(a, s.num_blocks, 0.1)
        ctx.bj_setup(part, 1e-10)
        ctx.gmres(s.b, cfg)
        e1.record()
        torch.cuda.synchronize()
        if it:
            res[label].append(e0.elapsed_time(e1))
for label, t in res.items():
    print(f"{label}: median {statistics.median(t):.1f} ms  {[round(x, 1) for x in t]}", flush=True)
