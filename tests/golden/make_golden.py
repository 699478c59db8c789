"""Generate the committed golden fixtures from the REAL reference library.

Runs in the build container only (needs oracle/_ref/libbjref.so, compiled
from /root/reference by ``make -C oracle ref``). Outputs:

* ``tests/golden/config<k>.json`` — per config: input digest, reference
  partition digests (assignment / perm / block_starts, bit-exact pins for our
  host partitioner), reference Hybrid and DoubleOnly solve reports
  (iterations, cycle residuals, history, x digest + strided sample).
* ``tests/golden/config0.npz`` — full assignment and x for config 0.
* ``tests/golden/cache/`` (git-ignored) — full reference assignments for
  local development only.

Usage: python tests/golden/make_golden.py [config ...]   (default 0 1 4 2 3)
Configs 2 and 3 take minutes: the reference partitioner is O(n*s)
(partition.cpp:45-56 called per block at :87-89).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Ref  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def solve_record(out, x_true):
    n = len(out.x)
    idx = np.linspace(0, n - 1, num=min(n, 1000)).astype(np.int64)
    return {
        "converged": out.converged,
        "total_iterations": int(out.total_iterations),
        "restarts": int(out.restarts),
        "final_residual": out.final_residual,
        "breakdown": out.breakdown,
        "cycle_residuals": out.cycle_residuals.tolist(),
        "history_rel": out.history[:, 2].tolist(),
        "history_cycle": out.history[:, 0].astype(int).tolist(),
        "x_sha256": sha(out.x),
        "x_norm2": float(np.linalg.norm(out.x)),
        "x_sample_idx": idx.tolist(),
        "x_sample": out.x[idx].tolist(),
        "rel_err_vs_xtrue": float(np.linalg.norm(out.x - x_true) / np.linalg.norm(x_true)),
        "timings_ms": out.timings,
        "perturbations": int(out.perturbations),
    }


def do_config(R: Ref, c: int):
    t0 = time.time()
    s = generate(c, 0)
    rec = {
        "config": c,
        "n": s.n,
        "nnz": s.nnz,
        "input_sha256": s.digest(),
        "num_blocks": s.num_blocks,
        "restart_m": s.restart_m,
        "tol": s.tol,
        "max_restarts": s.max_restarts,
    }
    asg, perm, bst, tm = R.partition(s.row_ptr, s.col, s.val, s.num_blocks, 0.1)
    dims = np.diff(bst)
    rec["partition"] = {
        "assignment_sha256": sha(asg),
        "perm_sha256": sha(perm),
        "block_starts_sha256": sha(bst),
        "dim_min": int(dims.min()),
        "dim_max": int(dims.max()),
        "sum_dim_sq": int((dims.astype(np.int64) ** 2).sum()),
        "timings_ms": tm,
    }
    os.makedirs(os.path.join(OUT, "cache"), exist_ok=True)
    np.save(os.path.join(OUT, "cache", f"config{c}_assignment.npy"), asg)
    print(f"config {c}: partition done {time.time() - t0:.1f}s", flush=True)

    if c == 4:
        steps = []
        for k in range(64):
            sk = generate(4, k)
            o = R.solve(sk.row_ptr, sk.col, sk.val, sk.num_blocks, sk.b, sk.restart_m, sk.tol,
                        sk.max_restarts, hybrid=True, assignment=asg)
            steps.append({
                "step": k,
                "input_sha256": sk.digest(),
                "converged": o.converged,
                "total_iterations": int(o.total_iterations),
                "final_residual": o.final_residual,
                "x_sha256": sha(o.x),
                "x_norm2": float(np.linalg.norm(o.x)),
                "rel_err_vs_xtrue": float(np.linalg.norm(o.x - sk.x_true) / np.linalg.norm(sk.x_true)),
                "timings_ms": o.timings,
            })
        rec["steps"] = steps
    hyb = R.solve(s.row_ptr, s.col, s.val, s.num_blocks, s.b, s.restart_m, s.tol, s.max_restarts,
                  hybrid=True, assignment=asg)
    rec["hybrid"] = solve_record(hyb, s.x_true)
    print(f"config {c}: hybrid {hyb.total_iterations} its {time.time() - t0:.1f}s", flush=True)
    dbl = R.solve(s.row_ptr, s.col, s.val, s.num_blocks, s.b, s.restart_m, s.tol, s.max_restarts,
                  hybrid=False, assignment=asg)
    rec["double"] = solve_record(dbl, s.x_true)
    print(f"config {c}: double {dbl.total_iterations} its {time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(OUT, f"config{c}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    if c == 0:
        np.savez_compressed(os.path.join(OUT, "config0.npz"), assignment=asg.astype(np.int32),
                            x_hybrid=hyb.x, x_double=dbl.x)


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [0, 1, 4, 2, 3]
    R = Ref()
    for c in cfgs:
        do_config(R, c)


if __name__ == "__main__":
    main()
