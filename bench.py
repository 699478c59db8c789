#!/usr/bin/env python
"""Benchmark: hybrid-precision block-Jacobi GMRES(m) setup + solve on B200.

Metric (BASELINE.json): "GMRES setup+solve ms/system; SpMV & precond-apply
HBM GB/s vs peak". One step = one full system: host graph + partition
(bit-identical to the reference), device Q A Q^T + batched FP32 block LU,
device GMRES(m) to the config's tolerance. Workload = BASELINE config 3, the
largest single-GPU config (160^3 interconnect mesh + long-range couplings,
n = 4,096,000, bs 256, GMRES(100), tol 1e-9; seeded synthetic data); the other
configs are parity cases and the ``--report-all`` table (``--config`` picks
another one).

  value : ms per system with A (device CSR + host CSR for the partitioner)
          and b already resident; device-timed (CUDA events, max over ranks),
          L2 flushed (256 MiB write) between systems.
  e2e   : same metric through the C ABI with HOST buffers: hpbj_set_matrix
          (CSR H2D) + partition + setup + hpbj_gmres (b H2D, x D2H).
  roofline : the dominant device kernel of a system (largest summed time per
          system among the batched LU, the apply-format build and the solve's
          apply / SpMV / orthogonalisation / fused-cycle kernels), from
          per-launch CUDA events in an instrumented host-enqueued repeat of
          the timed steps (the production path runs the restart loop as one
          CUDA graph). Algorithmic bytes per launch: DESIGN.md §5.
          peak = MEASURED_PEAKS.json hbm_gbs; traffic = ncu DRAM bytes of the
          same kernel (profiles/ncu_traffic_config<c>.json).
  cpu_baseline : the reference library (oracle/_ref: the reference sources
          compiled unmodified) on this host's cores through its own stock
          run_spec sequence (graph_from_matrix, partition_graph,
          block_jacobi, hybrid_restart_gmres), in a child process after the
          GPU timing; bounded by --cpu-budget-s (config 3: one system,
          ~9.5 min on the 16-core GPU-box host, 92% of it the reference's
          O(n*s) partition_graph).

``--impl reference`` runs that reference path alone (rank 0 only under
torchrun) with the same config dict, metric and unit: the timed steps are as
many full systems as fit --ref-budget-s (at least one; config 3: one, no
warm-up — one warm-up system would cost another ~9 minutes).

``--report-all`` measures every config (setup ms, solve ms, per-iteration us,
apply / SpMV HBM fractions) with the reference CPU beside each in the same
run: configs 0-3 through the reference's own partitioner, config 4's 64-step
sequence (partition of A_0 reused, block_jacobi + solve per step), plus a
one-thread line and a DoubleOnly line.

Multi-GPU: ``--gpus N`` runs N independent replicas (one system per GPU per
step, no collective on the data path; NCCL only for the barrier and the
max-over-ranks time), scaling "weak". Without torchrun, N > 1 relaunches
itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMRES setup+solve ms/system; SpMV & precond-apply HBM GB/s vs peak"
UNIT = "ms/system"
DEFAULT_CONFIG = 3
WORKLOADS = {
    0: "config0: random MNA circuit n=10,000 (ring + 2 random/node), bs 32, GMRES(30), tol 1e-10",
    1: "config1: 447x447 5-point power-grid mesh + 1% vias, n=199,809, bs 64, GMRES(50), tol 1e-10",
    2: "config2: 1M-node MNA circuit + 50 supply-rail hubs x 10,000, bs 128, GMRES(50), tol 1e-10",
    3: "config3: 160^3 7-point interconnect mesh + 0.5% long-range, n=4,096,000, bs 256, GMRES(100), tol 1e-9",
    4: "config4: transient Newton sequence, 64 steps sharing one pattern, n=100,000, bs 64, GMRES(30), tol 1e-10",
}
KNAMES = ["bj_apply_f32", "spmv_csr_f64", "arnoldi_mgs_f64", "arnoldi_cycle_fused"]
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # B200 CUDA-core FP32 FMA peak at the 1965 MHz max clock


# ---------------------------------------------------------------- inputs
def load_workloads(oracle_copy: bool = False):
    """paper_2509_09139_b200/workloads.py as a standalone module (numpy +
    ctypes only). oracle_copy: generate with oracle/build/libhpbj_gen.so, the
    same generator source built outside the product package, so the reference
    arm's process loads nothing from it."""
    spec = importlib.util.spec_from_file_location(
        "hpbj_workloads", os.path.join(ROOT, "paper_2509_09139_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["hpbj_workloads"] = mod  # dataclasses resolve their module by name
    spec.loader.exec_module(mod)
    if oracle_copy:
        mod.GEN_LIB = os.path.join(ROOT, "oracle", "build", "libhpbj_gen.so")
    return mod


def config_dict(s, c: int) -> dict:
    """The workload, identical in both arms."""
    return {"workload": WORKLOADS[c], "n": int(s.n), "nnz": int(s.nnz), "blocks": int(s.num_blocks),
            "restart_m": int(s.restart_m), "tol": float(s.tol), "max_restarts": int(s.max_restarts)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 20 ms) during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, mx, rs))
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        nv = self.nv
        bits = {"hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        reasons = sorted({name for _, _, r in self.samples for name, b in bits.items() if r & b})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------- replicas
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Replicas:
    """One process per GPU, each solving its own systems: no collective on
    the data path. The process group ("nccl" on the GPU box, "gloo" in the
    CPU tests) only carries the barrier around the timed region and the
    max-over-ranks of the per-rank device time."""

    def __init__(self, backend: str = "nccl"):
        self.ws, self.rank, self.local = dist_env()
        self.backend = backend
        if self.ws > 1:
            import torch.distributed as dist
            if backend == "nccl":
                import torch
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(backend)

    def _t(self, v):
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        return torch.tensor([float(v)], dtype=torch.float64, device=dev)

    def barrier(self):
        if self.ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, v: float) -> float:
        if self.ws == 1:
            return float(v)
        import torch.distributed as dist
        t = self._t(v)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if self.ws == 1:
            return float(v)
        import torch.distributed as dist
        t = self._t(v)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def aggregate_ms_per_system(self, local_total_ms: float, local_systems: int) -> float:
        """Whole-job ms/system: the slowest rank's time over all systems solved."""
        return self.max(local_total_ms) / self.sum(local_systems)

    def close(self):
        if self.ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


# ------------------------------------------------------- reference CPU
def reference_systems(s, budget_s: float, max_systems: int, warmup: int, hybrid: bool = True, assignment=None):
    """The reference library's stock path (run_spec, bjgmres_cli.cpp:125-164:
    graph_from_matrix + partition_graph + block_jacobi + hybrid_restart_gmres)
    on full systems: `warmup` untimed systems, then timed ones until
    max_systems or the budget is reached (at least one)."""
    from oracle import Ref, ref_available
    if not ref_available():
        return None
    R = Ref()

    def one():
        out = R.solve(s.row_ptr, s.col, s.val, s.num_blocks, s.b, s.restart_m, s.tol, s.max_restarts,
                      hybrid=hybrid, cond_estimates=False, assignment=assignment)
        return out, out.timings["setup_ms"] + out.timings["solve_ms"]

    t0 = time.perf_counter()
    done_warm = 0
    for _ in range(warmup):
        if time.perf_counter() - t0 > budget_s / 2:
            break
        one()
        done_warm += 1
    runs, phases, out = [], [], None
    t1 = time.perf_counter()
    while len(runs) < max(1, max_systems):
        out, ms = one()
        runs.append(ms)
        phases.append(dict(out.timings))
        per = (time.perf_counter() - t1) / len(runs)
        if time.perf_counter() - t0 + per > budget_s:
            break
    return {"runs": runs, "ms_per_system": sum(runs) / len(runs), "warmup": done_warm,
            "iterations": int(out.total_iterations), "converged": bool(out.converged),
            "final_residual": float(out.final_residual), "phases_ms": phases[-1]}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if ws > 1 and rank != 0:
        return 0
    cores = os.cpu_count() or 1
    threads = args.ref_threads or cores
    os.environ["OMP_NUM_THREADS"] = str(threads)
    W = load_workloads(oracle_copy=True)
    s = W.generate(args.config)
    res = reference_systems(s, args.ref_budget_s, args.steps, args.warmup, hybrid=not args.ref_double)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbjref.so not built"}))
        return 0
    v = res["ms_per_system"]
    k = len(res["runs"])
    mode = "DoubleOnly" if args.ref_double else "Hybrid"
    sample = (f"{k} full config-{args.config} system(s) through the reference's stock run_spec path "
              f"(graph_from_matrix + partition_graph + block_jacobi + hybrid_restart_gmres, {mode}); "
              f"{res['warmup']} warm-up; bounded by {args.ref_budget_s:.0f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": k,
        "steps_requested": args.steps, "warmup": res["warmup"], "ms_per_step": v, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if not args.ref_double else "f64",
        "data": "synthetic (seeded generator, oracle/build copy)", "config": config_dict(s, args.config),
        "mode": f"reference {mode}", "iterations": res["iterations"], "converged": res["converged"],
        "final_residual": res["final_residual"], "phases_ms": res["phases_ms"], "runs_ms": res["runs"],
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_child(config: int, budget_s: float, threads: int = 0, double: bool = False, steps: int = 1):
    """The reference arm in a child process (after the GPU timing): its JSON line."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", str(config),
           "--steps", str(steps), "--warmup", "0", "--ref-budget-s", str(budget_s)]
    if threads:
        cmd += ["--ref-threads", str(threads)]
    if double:
        cmd += ["--ref-double"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    for ln in reversed(r.stdout.strip().splitlines()):
        try:
            d = json.loads(ln)
            return d if "value" in d else None
        except Exception:
            continue
    return None


# ---------------------------------------------------------- GPU measurement
def kernel_table(kstats, peak):
    out = {}
    for k, nm in enumerate(KNAMES):
        st = kstats[k]
        if st["launches"] == 0:
            continue
        mean_ms = st["total_ms"] / st["launches"]
        gbs = st["total_bytes"] / (st["total_ms"] * 1e-3) / 1e9 if st["total_ms"] > 0 else None
        out[nm] = {"launches": st["launches"], "steps": st["steps"], "mean_us": mean_ms * 1e3,
                   "total_ms": st["total_ms"], "bytes_per_launch": st["bytes_per_launch"],
                   "gbs": gbs, "hbm_frac": (gbs / peak) if gbs else None}
    return out


def profile_kernels(ctx, step_fn, flush, steps, fused):
    """Instrumented repeat of `steps` steps: CUDA events around every kernel
    launch (host-enqueued, same kernels) -> per-kernel durations."""
    import torch
    ctx.set_fused(fused)
    ctx.set_profiling(True)
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        step_fn()
    torch.cuda.synchronize()
    ks = ctx.kernel_stats()
    ctx.set_profiling(False)
    ctx.set_fused(True)
    return ks


def measure_config(c, steps, warmup, local, sampler=None, prof_steps=None):
    """Device-resident measurement of config c through the production path."""
    import torch
    import paper_2509_09139_b200 as hp
    W = load_workloads()

    s = W.generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    cfg = hp.GmresConfig(restart_m=s.restart_m, tol=s.tol, max_restarts=s.max_restarts)
    ctx = hp.Context(local)
    ctx.set_matrix(a)
    d_b = torch.from_numpy(s.b).cuda()
    d_x = torch.zeros_like(d_b)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    infos = []

    def device_step():
        part = hp.partition_graph(a, s.num_blocks, 0.1)
        infos.append(ctx.bj_setup(part, 1e-10))
        _, rep = ctx.gmres(None, cfg, device_ptrs=(d_b.data_ptr(), d_x.data_ptr()))
        return rep

    torch.cuda.synchronize()
    for _ in range(warmup):
        device_step()
    torch.cuda.synchronize()
    l0 = ctx.launches()
    times = []
    infos.clear()
    sampler = sampler or ClockSampler(local)
    with sampler:
        for _ in range(steps):
            flush.zero_()  # L2 flush (256 MiB > 126 MB L2) between systems, outside the event pair
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rep = device_step()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    launches = ctx.launches() - l0
    setup_dev = {"ms_permute": statistics.median(i.ms_permute for i in infos),
                 "ms_lu": statistics.median(i.ms_lu for i in infos),
                 "ms_spk": statistics.median(i.ms_spk for i in infos),
                 "ms_factor": statistics.median(i.ms_factor for i in infos)}

    # breakdown of one more step (host clock, synchronous calls)
    t0 = time.perf_counter()
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    t1 = time.perf_counter()
    ctx.bj_setup(part, 1e-10)
    t2 = time.perf_counter()
    _, rep = ctx.gmres(None, cfg, device_ptrs=(d_b.data_ptr(), d_x.data_ptr()))
    t3 = time.perf_counter()
    x = d_x.cpu().numpy()

    peak, peak_kind = measured_peak()
    ps = prof_steps or steps
    kf = profile_kernels(ctx, device_step, flush, ps, fused=True)
    kern = kernel_table(kf, peak)
    fused = "arnoldi_cycle_fused" in kern
    if fused:  # fused path: the unfused kernels timed separately (the north star's per-kernel fractions)
        ku = profile_kernels(ctx, device_step, flush, ps, fused=False)
        kern.update({k: v for k, v in kernel_table(ku, peak).items() if k != "arnoldi_cycle_fused"})
    dims = np.diff(np.asarray(part.block_starts, dtype=np.float64))
    lu_flops = float(np.sum(2.0 / 3.0 * dims ** 3))  # dense LU of every diagonal block
    return {
        "sys": s, "a": a, "ctx": ctx, "cfg": cfg, "flush": flush, "assignment": part.assignment,
        "lu_flops": lu_flops,
        "value": sum(times) / steps, "times": times, "launches": launches, "rep": rep, "x": x,
        "breakdown_ms": {"partition_host": (t1 - t0) * 1e3, "bj_setup": (t2 - t1) * 1e3,
                         "permute_dev": setup_dev["ms_permute"], "factor_dev": setup_dev["ms_factor"],
                         "lu_dev": setup_dev["ms_lu"], "spk_build_dev": setup_dev["ms_spk"],
                         "solve": (t3 - t2) * 1e3,
                         "per_iteration_us": (t3 - t2) * 1e6 / max(1, rep.total_iterations)},
        "kernels": kern, "peak": peak, "peak_kind": peak_kind, "clocks": sampler.summary(),
        "fused": fused,
    }


def roofline_of(m, config):
    """The dominant device kernel of one system by summed time: the batched
    LU, the apply-format build, or one of the solve's kernels. The solve's
    kernels carry algorithmic bytes (HBM roofline); the LU is reported by its
    time share and FP32 rate (no HBM bound)."""
    kern, peak, peak_kind = m["kernels"], m["peak"], m["peak_kind"]
    its = max(1, m["rep"].total_iterations)
    per_system = {}
    for k, v in kern.items():
        if m["fused"] and k != "arnoldi_cycle_fused":
            continue  # timed for the table only; the production path runs the fused cycle
        per_system[k] = v["total_ms"] / max(1, v["steps"]) * its
    per_system["block_lu_f32"] = m["breakdown_ms"]["lu_dev"]
    per_system["spk_build"] = m["breakdown_ms"]["spk_build_dev"]
    dom_any = max(per_system, key=per_system.get)
    hbm_kernels = {k: t for k, t in per_system.items() if k in kern}
    dom = max(hbm_kernels, key=hbm_kernels.get)
    achieved = kern[dom]["gbs"] or 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_config{config}.json")
    if os.path.exists(tpath):
        try:
            t = json.load(open(tpath))
            traffic = t.get(dom)
            if traffic is not None and dom == "arnoldi_cycle_fused":
                # captured launch = one cycle of t[...steps] steps; scale to this run's mean steps per launch
                per_step = traffic / t.get("arnoldi_cycle_fused_steps", 1)
                traffic = per_step * kern[dom]["steps"] / kern[dom]["launches"]
        except Exception:
            traffic = None
    total = sum(per_system.values())
    lu_ms = m["breakdown_ms"]["lu_dev"]
    lu = {"ms": lu_ms, "flops": m["lu_flops"], "tflops": m["lu_flops"] / (lu_ms * 1e-3) / 1e12 if lu_ms else None,
          "fp32_peak_tflops": FP32_PEAK_TFLOPS,
          "fp32_frac": (m["lu_flops"] / (lu_ms * 1e-3) / 1e12 / FP32_PEAK_TFLOPS) if lu_ms else None,
          "note": "batched FP32 LU on CUDA cores (no tensor-core path: bit-exact FP32 fmaf chains); "
                  "flops = sum (2/3) d^3 over the blocks"}
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_kind, "traffic": traffic,
            "bytes_per_launch": kern[dom]["bytes_per_launch"],
            "device_ms_per_system": {k: round(v, 3) for k, v in per_system.items()},
            "share_of_device_time": round(per_system[dom] / total, 3) if total else None,
            "largest_device_kernel": dom_any, "block_lu_f32": lu}


def run_gpu_arm(args):
    import torch
    rep_group = Replicas("nccl")
    ws, rank, local = rep_group.ws, rep_group.rank, rep_group.local
    torch.cuda.set_device(local)
    import paper_2509_09139_b200 as hp

    rep_group.barrier()
    m = measure_config(args.config, args.steps, args.warmup, local)
    s, a = m["sys"], m["a"]
    value = rep_group.aggregate_ms_per_system(sum(m["times"]), args.steps)

    # ---- e2e through the C ABI with host buffers (CSR, b in; x out)
    flush = m["flush"]

    def e2e_step(c2):
        c2.set_matrix(a)
        part = hp.partition_graph(a, s.num_blocks, 0.1)
        c2.bj_setup(part, 1e-10)
        return c2.gmres(s.b, m["cfg"])

    ctx2 = hp.Context(local)
    e2e_step(ctx2)
    torch.cuda.synchronize()
    e2e_times = []
    rep_group.barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        x2, _ = e2e_step(ctx2)
        e1.record()
        torch.cuda.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
    e2e_value = rep_group.aggregate_ms_per_system(sum(e2e_times), args.steps)
    h2d = s.row_ptr.nbytes + s.col.nbytes + s.val.nbytes + s.b.nbytes
    d2h = x2.nbytes
    roofline = roofline_of(m, args.config)
    del ctx2

    # ---- CPU baseline: the reference library on this host, after the GPU timing
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        d = cpu_baseline_child(args.config, args.cpu_budget_s)
        if d is not None:
            cpu = dict(d["cpu_baseline"])
            cpu.update({"iterations": d["iterations"], "phases_ms": d.get("phases_ms"), "runs_ms": d.get("runs_ms")})

    if rank == 0:
        rep = m["rep"]
        err = float(np.linalg.norm(m["x"] - s.x_true) / np.linalg.norm(s.x_true))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": value * ws, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator)",
            "config": config_dict(s, args.config),
            "timing": {"precond_dtype": "f32", "krylov_dtype": "f64", "l2_flush": "256MiB write between steps",
                       "parallelism": f"replicas x{ws}"},
            "iterations": rep.total_iterations, "converged": rep.converged,
            "final_residual": rep.final_residual, "rel_err_vs_xtrue": err,
            "breakdown_ms": m["breakdown_ms"],
            "kernels": m["kernels"],
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(m["launches"]),
            "clocks": m["clocks"],
        }
        print(json.dumps(line), flush=True)
    rep_group.close()
    return 0


# ---------------------------------------------------------------------------
def run_report_all(args):
    """Per-config table: setup / solve / per-iteration, apply & SpMV HBM
    fractions, the reference CPU beside each config in the same run."""
    import torch
    import paper_2509_09139_b200 as hp
    W = load_workloads()
    torch.cuda.set_device(0)
    cores = os.cpu_count() or 1
    table = {"metric": METRIC, "peak_gbs": measured_peak()[0], "cores": cores, "configs": {}, "reference_extra": {}}
    ref_cfgs = [] if args.no_cpu_baseline else [int(x) for x in args.ref_configs.split(",") if x != ""]
    for c in [int(x) for x in args.configs.split(",")]:
        m = measure_config(c, args.steps, args.warmup, 0, prof_steps=1)
        s, rep = m["sys"], m["rep"]
        row = {"workload": WORKLOADS[c], "n": s.n, "nnz": s.nnz, "blocks": s.num_blocks,
               "ms_per_system": m["value"], "iterations": rep.total_iterations,
               "final_residual": rep.final_residual, "converged": rep.converged,
               "breakdown_ms": m["breakdown_ms"], "kernels": m["kernels"],
               "apply_hbm_frac": m["kernels"].get("bj_apply_f32", {}).get("hbm_frac"),
               "spmv_hbm_frac": m["kernels"].get("spmv_csr_f64", {}).get("hbm_frac"),
               "roofline": roofline_of(m, c), "clocks": m["clocks"]}
        if c == 4:  # the transient sequence: one partition, per step refactor + solve
            ctx, cfg, a = m["ctx"], m["cfg"], m["a"]
            t0 = time.perf_counter()
            part = hp.partition_graph(a, s.num_blocks, 0.1)
            ctx.bj_setup(part, 1e-10)
            t_part = (time.perf_counter() - t0) * 1e3
            per, its = [], []
            for k in range(64):
                sk = W.generate(4, k)
                b = torch.from_numpy(sk.b).cuda()
                x = torch.zeros_like(b)
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.update_values(sk.val)
                ctx.bj_refactor()
                _, r = ctx.gmres(None, cfg, device_ptrs=(b.data_ptr(), x.data_ptr()))
                e1.record()
                torch.cuda.synchronize()
                per.append(e0.elapsed_time(e1))
                its.append(r.total_iterations)
            row["sequence"] = {"steps": 64, "partition_and_first_setup_ms": t_part, "total_ms": sum(per),
                               "per_step_ms_mean": sum(per) / 64, "iterations": its}
        del m
        torch.cuda.empty_cache()
        if c in ref_cfgs:
            if c == 4:
                row["cpu_reference"] = reference_sequence_config4(W, args.cpu_budget_s)
            else:
                d = cpu_baseline_child(c, args.cpu_budget_s, steps=1)
                if d is not None:
                    row["cpu_reference"] = {"ms_per_system": d["value"], "phases_ms": d["phases_ms"],
                                            "iterations": d["iterations"], "cores": d["cpu_baseline"]["cores"],
                                            "kind": "reference", "sample": d["cpu_baseline"]["sample"]}
        table["configs"][str(c)] = row
        print(json.dumps({"config": c, "ms_per_system": row["ms_per_system"], "iterations": row["iterations"],
                          "breakdown_ms": row["breakdown_ms"], "apply_hbm_frac": row["apply_hbm_frac"],
                          "spmv_hbm_frac": row["spmv_hbm_frac"],
                          "cpu_ms": row.get("cpu_reference", {}).get("ms_per_system")}), flush=True)
    if not args.no_cpu_baseline and args.ref_extra:
        for label, threads, double in (("config1_one_thread", 1, False), ("config1_double_only", 0, True)):
            d = cpu_baseline_child(1, args.cpu_budget_s, threads=threads, double=double)
            if d is not None:
                table["reference_extra"][label] = {"ms_per_system": d["value"], "phases_ms": d["phases_ms"],
                                                   "iterations": d["iterations"],
                                                   "cores": d["cpu_baseline"]["cores"], "mode": d["mode"]}
                print(json.dumps({label: table["reference_extra"][label]}), flush=True)
    with open(args.out, "w") as f:
        json.dump(table, f, indent=1, default=float)
    return 0


def reference_sequence_config4(W, budget_s):
    """Config 4 on the reference CPU as its caller would run it: partition of
    A_0 once (graph_from_matrix + partition_graph), then per step
    block_jacobi(A_k) + hybrid_restart_gmres (run_spec's sequence with the
    partition reused)."""
    from oracle import Ref, ref_available
    if not ref_available():
        return None
    R = Ref()
    s0 = W.generate(4, 0)
    asg, _, _, tt = R.partition(s0.row_ptr, s0.col, s0.val, s0.num_blocks)
    per, its = [], []
    t0 = time.perf_counter()
    for k in range(64):
        sk = W.generate(4, k)
        out = R.solve(sk.row_ptr, sk.col, sk.val, sk.num_blocks, sk.b, sk.restart_m, sk.tol, sk.max_restarts,
                      hybrid=True, cond_estimates=False, assignment=asg)
        per.append(out.timings["block_jacobi_ms"] + out.timings["solve_ms"])
        its.append(out.total_iterations)
        if time.perf_counter() - t0 > budget_s:
            break
    return {"steps": len(per), "partition_ms": tt["graph_ms"] + tt["partition_ms"], "total_ms": sum(per),
            "per_step_ms_mean": sum(per) / len(per), "iterations": its, "cores": os.cpu_count(),
            "kind": "reference"}


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 without torchrun: start the N replica processes ourselves."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(args.master_port), os.path.abspath(__file__)]
    cmd += [a for a in sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=900.0,
                    help="wall budget of the reference CPU baseline (at least one full system)")
    ap.add_argument("--ref-budget-s", type=float, default=1500.0,
                    help="--impl reference: wall budget of the timed systems (at least one)")
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--ref-double", action="store_true", help="reference DoubleOnly instead of Hybrid")
    ap.add_argument("--report-all", action="store_true")
    ap.add_argument("--configs", default="0,1,2,3,4")
    ap.add_argument("--ref-configs", default="0,1,2,3,4")
    ap.add_argument("--ref-extra", type=int, default=1, help="report-all: one-thread and DoubleOnly lines")
    ap.add_argument("--master-port", type=int, default=29531)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "per_config.json"))
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.report_all:
        return run_report_all(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
