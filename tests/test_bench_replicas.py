"""bench.py's multi-GPU path is replicas only: one process
per GPU, each solving its own systems, no collective on the data path; the
process group carries only the barrier and the max-over-ranks time. These
tests run that host-side logic with world_size 2 over gloo on CPU: both ranks
partition their own system (host code, bit-identical to the reference) and
the whole-job ms/system is the slowest rank's time over all systems."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import json, os, sys, time
sys.path.insert(0, sys.argv[1])
import numpy as np
import bench
import paper_2509_09139_b200 as hp
rg = bench.Replicas("gloo")
W = bench.load_workloads()
s = W.generate(0)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
rg.barrier()
t0 = time.perf_counter()
systems = 2 + rg.rank  # unequal work per rank
for _ in range(systems):
    part = hp.partition_graph(a, s.num_blocks, 0.1)
local_ms = (time.perf_counter() - t0) * 1e3 + (50.0 if rg.rank == 1 else 0.0)
agg = rg.aggregate_ms_per_system(local_ms, systems)
mx = rg.max(local_ms)
tot = rg.sum(systems)
with open(os.path.join(sys.argv[2], f"rank{rg.rank}.json"), "w") as f:
    json.dump({"rank": rg.rank, "ws": rg.ws, "local_ms": local_ms, "agg": agg, "max": mx, "tot": tot,
               "asg": int(np.asarray(part.assignment).sum())}, f)
rg.close()
'''


def _run(tmp_path, nproc):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    env = dict(os.environ, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc), str(w), ROOT, str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    return [json.loads((tmp_path / f"rank{k}.json").read_text()) for k in range(nproc)]


def test_replicas_world_size_2_gloo(tmp_path):
    out = _run(tmp_path, 2)
    assert sorted(o["rank"] for o in out) == [0, 1] and all(o["ws"] == 2 for o in out)
    # every rank holds the same whole-job numbers
    assert len({o["agg"] for o in out}) == 1 and len({o["max"] for o in out}) == 1
    mx = max(o["local_ms"] for o in out)
    assert out[0]["max"] == pytest.approx(mx)
    assert out[0]["tot"] == 5  # 2 + 3 systems
    assert out[0]["agg"] == pytest.approx(mx / 5)
    # replicas of the same system partition identically (no data exchanged)
    assert len({o["asg"] for o in out}) == 1


def test_single_process_needs_no_group(tmp_path):
    sys.path.insert(0, ROOT)
    import bench
    rg = bench.Replicas("gloo")
    assert rg.ws == 1 and rg.max(3.5) == 3.5 and rg.aggregate_ms_per_system(10.0, 4) == 2.5
    rg.close()
