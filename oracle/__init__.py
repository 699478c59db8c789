"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline. The product path
(``paper_2509_09139_b200``) never imports it and has no CPU fallback.

Two oracles:

* ``Ref``  — the UNMODIFIED reference library (arXiv 2509.09139 artifact)
  compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` into
  ``oracle/_ref/libbjref.so`` together with our C-ABI harness
  ``oracle/ref_driver.cpp``.
* ``Port`` — ``oracle/hpbj_oracle.c``: our plain-C restatement of the same
  algorithm, pinned against ``Ref`` and the committed golden fixtures.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libbjref.so")
PORT_LIB = os.path.join(HERE, "build", "liboracle_port.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


class RefReport(ctypes.Structure):
    _fields_ = [
        ("converged", ctypes.c_int64),
        ("total_iterations", ctypes.c_int64),
        ("restarts", ctypes.c_int64),
        ("final_residual", ctypes.c_double),
        ("breakdown", ctypes.c_int64),
        ("ls_rank_deficient", ctypes.c_int64),
        ("hist_len", ctypes.c_int64),
        ("cyc_len", ctypes.c_int64),
        ("ms_graph", ctypes.c_double),
        ("ms_partition", ctypes.c_double),
        ("ms_block_jacobi", ctypes.c_double),
        ("ms_setup", ctypes.c_double),
        ("ms_solve", ctypes.c_double),
        ("perturbations", ctypes.c_int64),
    ]


@dataclass
class SolveOut:
    x: np.ndarray
    converged: bool
    total_iterations: int
    restarts: int
    final_residual: float
    breakdown: bool
    ls_rank_deficient: bool
    history: np.ndarray  # (k, 3): cycle, iteration, relative residual
    cycle_residuals: np.ndarray
    timings: dict = field(default_factory=dict)
    perturbations: int = 0


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


class Ref:
    """ctypes view of oracle/_ref/libbjref.so (the reference library)."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: build it with `make -C oracle ref`")
        L = ctypes.CDLL(path)
        L.bjref_last_error.restype = ctypes.c_char_p
        self.L = L

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.bjref_last_error().decode())

    @staticmethod
    def _csr(rp, ci, v):
        return (
            np.ascontiguousarray(rp, np.int64),
            np.ascontiguousarray(ci, np.int64),
            np.ascontiguousarray(v, np.float64),
        )

    def mm_read(self, path):
        """The reference's read_matrix_market_file: (nrows, ncols, rp, ci, val)."""
        nr, nc, nz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._chk(self.L.bjref_mm_read(os.fsencode(path), ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nz),
                                       None, None, None))
        rp, ci, v = np.zeros(nr.value + 1, np.int64), np.zeros(nz.value, np.int64), np.zeros(nz.value)
        self._chk(self.L.bjref_mm_read(os.fsencode(path), ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nz),
                                       _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p)))
        return nr.value, nc.value, rp, ci, v

    def mm_write(self, path, rp, ci, v):
        rp, ci, v = self._csr(rp, ci, v)
        self._chk(self.L.bjref_mm_write(os.fsencode(path), ctypes.c_int64(len(rp) - 1), _p(rp, _i64p),
                                        _p(ci, _i64p), _p(v, _f64p)))

    def spmv(self, rp, ci, v, x, fp32=False):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(n)
        self._chk(self.L.bjref_spmv(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                    _p(x, _f64p), _p(y, _f64p), ctypes.c_int(int(fp32))))
        return y

    def graph(self, rp, ci, v):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        cap = int(rp[-1]) * 2 + 1
        st = np.zeros(n + 1, np.int64)
        nb = np.zeros(cap, np.int64)
        w = np.zeros(cap)
        self._chk(self.L.bjref_graph(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                     _p(st, _i64p), _p(nb, _i64p), _p(w, _f64p), ctypes.c_int64(cap)))
        k = int(st[-1])
        return st, nb[:k].copy(), w[:k].copy()

    def partition(self, rp, ci, v, s, tol=0.1):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.zeros(n, np.int64)
        perm = np.zeros(n, np.int64)
        bst = np.zeros(s + 1, np.int64)
        tg, tp = ctypes.c_double(), ctypes.c_double()
        self._chk(self.L.bjref_partition(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                         ctypes.c_int64(s), ctypes.c_double(tol), _p(asg, _i64p),
                                         _p(perm, _i64p), _p(bst, _i64p), ctypes.byref(tg),
                                         ctypes.byref(tp)))
        return asg, perm, bst, {"graph_ms": tg.value, "partition_ms": tp.value}

    def partition_graph(self, starts, nbr, w, s, tol=0.1):
        starts = np.ascontiguousarray(starts, np.int64)
        nbr = np.ascontiguousarray(nbr, np.int64)
        w = np.ascontiguousarray(w, np.float64)
        n = len(starts) - 1
        asg = np.zeros(n, np.int64)
        self._chk(self.L.bjref_partition_graph(ctypes.c_int64(n), _p(starts, _i64p), _p(nbr, _i64p),
                                               _p(w, _f64p), ctypes.c_int64(s), ctypes.c_double(tol),
                                               _p(asg, _i64p)))
        return asg

    def permute(self, rp, ci, v, perm):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        perm = np.ascontiguousarray(perm, np.int64)
        rp2 = np.zeros(n + 1, np.int64)
        ci2 = np.zeros(len(ci), np.int64)
        v2 = np.zeros(len(v))
        self._chk(self.L.bjref_permute(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                       _p(perm, _i64p), _p(rp2, _i64p), _p(ci2, _i64p), _p(v2, _f64p)))
        return rp2, ci2, v2

    def factors(self, rp, ci, v, s, assignment, eps=1e-10, want64=False):
        """Per-block densified factors F = L_strict + U (pivot order)."""
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        dims = np.bincount(asg, minlength=s).astype(np.int64)
        tot = int((dims * dims).sum())
        f32 = np.zeros(tot, np.float32)
        f64 = np.zeros(tot) if want64 else None
        piv = np.zeros(n, np.int64)
        pert = np.zeros(s, np.int64)
        sc = ctypes.c_int64()
        self._chk(self.L.bjref_factors(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                       ctypes.c_int64(s), _p(asg, _i64p), ctypes.c_double(eps),
                                       _p(f32, _f32p), _p(f64, _f64p), _p(piv, _i64p),
                                       _p(pert, _i64p), ctypes.byref(sc)))
        return dims, f32, f64, piv, pert

    def block_stats(self, rp, ci, v, s, assignment, eps=1e-10):
        """(cond_estimate, error_bound, block_nnz) per block, reference Hybrid setup."""
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        cond, eb, bn = np.zeros(s), np.zeros(s), np.zeros(s, np.int64)
        self._chk(self.L.bjref_block_stats(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                           ctypes.c_int64(s), _p(asg, _i64p), ctypes.c_double(eps),
                                           _p(cond, _f64p), _p(eb, _f64p), _p(bn, _i64p)))
        return cond, eb, bn

    def apply(self, rp, ci, v, s, assignment, vin, eps=1e-10, fp32=True):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        vin = np.ascontiguousarray(vin, np.float64)
        z = np.zeros(n)
        self._chk(self.L.bjref_apply(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                     ctypes.c_int64(s), _p(asg, _i64p), ctypes.c_double(eps),
                                     ctypes.c_int(1 if fp32 else 0), _p(vin, _f64p), _p(z, _f64p)))
        return z

    def apply_neumann(self, rp, ci, v, s, assignment, vin, order, k, eps=1e-10, fp32=True):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        vin = np.ascontiguousarray(vin, np.float64)
        z = np.zeros(n)
        self._chk(self.L.bjref_apply_neumann(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                             ctypes.c_int64(s), _p(asg, _i64p), ctypes.c_double(eps),
                                             ctypes.c_int(order), ctypes.c_int(k), ctypes.c_int(1 if fp32 else 0),
                                             _p(vin, _f64p), _p(z, _f64p)))
        return z

    def solve(self, rp, ci, v, s, b, m, tol, max_restarts, hybrid=True, assignment=None,
              absolute_tol=False, eps=1e-10, cond_estimates=False, neumann_order=0):
        self.L.bjref_set_neumann_order(ctypes.c_int(neumann_order))
        try:
            return self._solve(rp, ci, v, s, b, m, tol, max_restarts, hybrid, assignment, absolute_tol, eps,
                               cond_estimates)
        finally:
            self.L.bjref_set_neumann_order(ctypes.c_int(0))

    def _solve(self, rp, ci, v, s, b, m, tol, max_restarts, hybrid, assignment, absolute_tol, eps,
               cond_estimates):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        b = np.ascontiguousarray(b, np.float64)
        asg = None if assignment is None else np.ascontiguousarray(assignment, np.int64)
        x = np.zeros(n)
        rep = RefReport()
        hcap = m * max_restarts + 2
        hist = np.zeros(3 * hcap)
        cyc = np.zeros(max_restarts + 1)
        self._chk(self.L.bjref_solve(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                     ctypes.c_int64(s), _p(asg, _i64p), _p(b, _f64p), ctypes.c_int64(m),
                                     ctypes.c_double(tol), ctypes.c_int64(max_restarts),
                                     ctypes.c_int(int(hybrid)), ctypes.c_int(int(absolute_tol)),
                                     ctypes.c_double(eps), ctypes.c_int(int(cond_estimates)),
                                     _p(x, _f64p), ctypes.byref(rep), _p(hist, _f64p),
                                     ctypes.c_int64(hcap), _p(cyc, _f64p),
                                     ctypes.c_int64(max_restarts + 1)))
        return self._out(x, rep, hist, cyc)

    def ilu0_values(self, rp, ci, v):
        rp, ci, v = self._csr(rp, ci, v)
        out = np.zeros(len(v))
        self._chk(self.L.bjref_ilu0_values(ctypes.c_int64(len(rp) - 1), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                           _p(out, _f64p)))
        return out

    def ilu0_apply(self, rp, ci, v, vin):
        rp, ci, v = self._csr(rp, ci, v)
        vin = np.ascontiguousarray(vin, np.float64)
        z = np.zeros(len(rp) - 1)
        self._chk(self.L.bjref_ilu0_apply(ctypes.c_int64(len(rp) - 1), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                          _p(vin, _f64p), _p(z, _f64p)))
        return z

    def solve_ilu0(self, rp, ci, v, b, m, tol, max_restarts, hybrid=False):
        """run_spec with --precond ilu0 (bjgmres_cli.cpp:128-131)."""
        self.L.bjref_set_alt_precond(ctypes.c_int(1))
        try:
            return self.solve_identity(rp, ci, v, b, m, tol, max_restarts, hybrid)
        finally:
            self.L.bjref_set_alt_precond(ctypes.c_int(0))

    def solve_identity(self, rp, ci, v, b, m, tol, max_restarts, hybrid=False):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(n)
        rep = RefReport()
        hcap = m * max_restarts + 2
        hist = np.zeros(3 * hcap)
        cyc = np.zeros(max_restarts + 1)
        self._chk(self.L.bjref_solve_identity(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p),
                                              _p(v, _f64p), _p(b, _f64p), ctypes.c_int64(m),
                                              ctypes.c_double(tol), ctypes.c_int64(max_restarts),
                                              ctypes.c_int(int(hybrid)), _p(x, _f64p),
                                              ctypes.byref(rep), _p(hist, _f64p), ctypes.c_int64(hcap),
                                              _p(cyc, _f64p), ctypes.c_int64(max_restarts + 1)))
        return self._out(x, rep, hist, cyc)

    @staticmethod
    def _out(x, rep, hist, cyc):
        hl, cl = rep.hist_len, rep.cyc_len
        return SolveOut(
            x=x,
            converged=bool(rep.converged),
            total_iterations=rep.total_iterations,
            restarts=rep.restarts,
            final_residual=rep.final_residual,
            breakdown=bool(rep.breakdown),
            ls_rank_deficient=bool(rep.ls_rank_deficient),
            history=hist[: 3 * hl].reshape(hl, 3).copy(),
            cycle_residuals=cyc[:cl].copy(),
            timings={
                "graph_ms": rep.ms_graph,
                "partition_ms": rep.ms_partition,
                "block_jacobi_ms": rep.ms_block_jacobi,
                "setup_ms": rep.ms_setup,
                "solve_ms": rep.ms_solve,
            },
            perturbations=rep.perturbations,
        )


# ---------------------------------------------------------------------------
class PortReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("converged", "total_iterations", "restarts", "breakdown",
                                              "rank_deficient", "hist_len", "cyc_len")] + [
        ("final_residual", ctypes.c_double), ("singular_block", ctypes.c_int64),
        ("singular_column", ctypes.c_int64)]


MODES = {"double": 0, "hybrid": 1, "mix": 2}


class Port:
    """ctypes view of oracle/build/liboracle_port.so (hpbj_oracle.c): our
    plain-C restatement of the reference algorithm."""

    def __init__(self, path: str = PORT_LIB):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: build it with `make -C oracle port`")
        self.L = ctypes.CDLL(path)

    @staticmethod
    def _csr(rp, ci, v):
        return Ref._csr(rp, ci, v)

    def _chk(self, rc, what):
        if rc != 0:
            raise OracleError(rc, f"{what}: rc={rc}")

    def spmv(self, rp, ci, v, x, fp32=False):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(n)
        self._chk(self.L.orc_spmv(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), _p(x, _f64p),
                                  _p(y, _f64p), ctypes.c_int(int(fp32))), "spmv")
        return y

    def graph(self, rp, ci, v):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        cap = 2 * int(rp[-1]) + 1
        st, nb, w = np.zeros(n + 1, np.int64), np.zeros(cap, np.int64), np.zeros(cap)
        self._chk(self.L.orc_graph(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), _p(st, _i64p),
                                   _p(nb, _i64p), _p(w, _f64p), ctypes.c_int64(cap)), "graph")
        k = int(st[-1])
        return st, nb[:k].copy(), w[:k].copy()

    def partition(self, rp, ci, v, s, tol=0.1):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.zeros(n, np.int64)
        self._chk(self.L.orc_partition(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                       ctypes.c_int64(s), ctypes.c_double(tol), _p(asg, _i64p)), "partition")
        return asg

    def factors(self, rp, ci, v, s, assignment, eps=1e-10):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        dims = np.bincount(asg, minlength=s).astype(np.int64)
        f64 = np.zeros(int((dims * dims).sum()))
        piv = np.zeros(n, np.int64)
        pert = np.zeros(s, np.int64)
        sb, sc = ctypes.c_int64(), ctypes.c_int64()
        rc = self.L.orc_factors(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p), ctypes.c_int64(s),
                                _p(asg, _i64p), ctypes.c_double(eps), _p(f64, _f64p), _p(piv, _i64p),
                                _p(pert, _i64p), ctypes.byref(sb), ctypes.byref(sc))
        if rc == 3:
            raise OracleError(3, f"singular block {sb.value} column {sc.value}")
        self._chk(rc, "factors")
        return dims, f64, piv, pert

    def apply(self, rp, ci, v, s, assignment, vin, eps=1e-10, fp32=True):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        vin = np.ascontiguousarray(vin, np.float64)
        z = np.zeros(n)
        self._chk(self.L.orc_apply(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                   ctypes.c_int64(s), _p(asg, _i64p), ctypes.c_double(eps),
                                   ctypes.c_int(int(fp32)), _p(vin, _f64p), _p(z, _f64p)), "apply")
        return z

    def solve_full(self, rp, ci, v, s, assignment, b, m, tol, max_restarts, mode="hybrid", eps=1e-10):
        rp, ci, v = self._csr(rp, ci, v)
        n = len(rp) - 1
        asg = np.ascontiguousarray(assignment, np.int64)
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(n)
        rep = PortReport()
        hcap = m * max_restarts + 2
        hist = np.zeros(3 * hcap)
        cyc = np.zeros(max_restarts + 1)
        self._chk(self.L.orc_solve(ctypes.c_int64(n), _p(rp, _i64p), _p(ci, _i64p), _p(v, _f64p),
                                   ctypes.c_int64(s), _p(asg, _i64p), _p(b, _f64p), ctypes.c_int64(m),
                                   ctypes.c_double(tol), ctypes.c_int64(max_restarts), ctypes.c_int(MODES[mode]),
                                   ctypes.c_double(eps), _p(x, _f64p), ctypes.byref(rep), _p(hist, _f64p),
                                   ctypes.c_int64(hcap), _p(cyc, _f64p), ctypes.c_int64(max_restarts + 1)),
                  "solve")
        hl, cl = rep.hist_len, rep.cyc_len
        return SolveOut(x=x, converged=bool(rep.converged), total_iterations=rep.total_iterations,
                        restarts=rep.restarts, final_residual=rep.final_residual, breakdown=bool(rep.breakdown),
                        ls_rank_deficient=bool(rep.rank_deficient), history=hist[:3 * hl].reshape(hl, 3).copy(),
                        cycle_residuals=cyc[:cl].copy())

    def solve(self, sysm, assignment, mode="hybrid"):
        """(iterations, x) of a workloads.System — smoke()'s fallback checker."""
        out = self.solve_full(sysm.row_ptr, sysm.col, sysm.val, sysm.num_blocks, assignment, sysm.b,
                              sysm.restart_m, sysm.tol, sysm.max_restarts, mode)
        return out.total_iterations, out.x
