"""Per-kernel A/B on the GPU: for each config and each env variant (a child
process per variant, env switches are read at setup/solve), setup + solve
REPS systems with per-launch CUDA events and print the mean us per launch of
the apply / SpMV / orthogonalisation kernels, solve ms, LU ms, iterations.
usage: kern_ab.py CONFIGS 'VAR=a VAR2=b' 'VAR=c' ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CHILD = r'''
import json, os, sys, time
sys.path.insert(0, sys.argv[2])
import numpy as np
import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate
c = int(sys.argv[1])
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
ctx = hp.Context(0)
ctx.set_matrix(a)
cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
part = hp.partition_graph(a, s.num_blocks, 0.1)
reps = int(os.environ.get("REPS", "3"))
out = {}
lu, solve = [], []
for rep in range(reps + 1):
    info = ctx.bj_setup(part, 1e-10)
    t0 = time.perf_counter()
    x, r = ctx.gmres(s.b, cfg)
    t1 = time.perf_counter()
    if rep:
        lu.append(info.ms_lu); solve.append((t1 - t0) * 1e3)
ctx.set_fused(False)
ctx.set_profiling(True)
for rep in range(reps):
    ctx.bj_setup(part, 1e-10)
    x2, r2 = ctx.gmres(s.b, cfg)
ks = ctx.kernel_stats()
ctx.set_profiling(False)
err = float(np.linalg.norm(x - s.x_true) / np.linalg.norm(s.x_true))
res = dict(its=r.total_iterations, its_prof=r2.total_iterations, err=err, lu_ms=min(lu), solve_ms=min(solve),
           spk_ms=info.ms_spk)
for k, v in zip(["apply", "spmv", "orth", "cycle"], ks):
    if v["launches"]:
        res[k + "_us"] = round(v["total_ms"] * 1e3 / v["launches"], 2)
        res[k + "_gbs"] = round(v["total_bytes"] / (v["total_ms"] * 1e-3) / 1e9, 1) if v["total_ms"] else None
print("RESULT " + json.dumps(res))
'''

configs = [int(x) for x in sys.argv[1].split(",")]
variants = sys.argv[2:] or [""]
for c in configs:
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, "-c", CHILD, str(c), ROOT], env=env, capture_output=True, text=True,
                           timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        print(f"config {c} [{v}]: " + (line[-1][7:] if line else "FAILED " + r.stderr[-800:]), flush=True)
