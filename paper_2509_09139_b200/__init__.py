"""B200-native hybrid-precision block-Jacobi GMRES(m) (arXiv 2509.09139 path).

Python mirror of the reference's C++ solver interface
(/root/reference/proj/include/bjgmres), over the C ABI of libhpbj.so
(include/hpbj.h). Names, argument meaning and error behaviour follow the
reference so callers (and our parity tests) read like the reference's own:

=====================================  =====================================
reference (proj/include/bjgmres)        here
=====================================  =====================================
SparseMatrix (sparse_matrix.hpp:23)     SparseMatrix
graph_from_matrix (graph.hpp:30)        graph_from_matrix -> WeightedGraph
partition_graph (partition.hpp:38)      partition_graph -> Partition
partition_from_assignment (:33)         partition_from_assignment
Preconditioner::block_jacobi (:60)      Preconditioner.block_jacobi
Preconditioner::apply<float> (:69)      Preconditioner.apply
GmresConfig (gmres.hpp:89)              GmresConfig
hybrid_restart_gmres (gmres.hpp:145)    hybrid_restart_gmres -> SolveResult
SingularBlockError (lu.hpp:52)          SingularBlockError
=====================================  =====================================

Exceptions: std::invalid_argument -> ValueError, std::logic_error ->
LogicError, std::out_of_range -> IndexError, SingularBlockError ->
SingularBlockError, device failures -> RuntimeError.

Every numerical step runs in sm_100a kernels; only graph partitioning runs on
the host (bit-identical to the reference). There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi

__all__ = [
    "SparseMatrix", "WeightedGraph", "Partition", "BlockJacobiOptions", "Preconditioner", "GmresConfig",
    "SolveReport", "SolveResult", "HistoryPoint", "SingularBlockError", "LogicError", "graph_from_matrix",
    "partition_graph", "partition_from_assignment", "hybrid_restart_gmres", "Context", "library",
    "read_matrix_market", "write_matrix_market", "read_csr_cache", "write_csr_cache", "export_partition",
    "import_partition", "measure_block_nnz", "cut_weight",
]

ROUNDOFF_SINGLE = 2.0 ** -24  # types.hpp:12
ROUNDOFF_DOUBLE = 2.0 ** -53  # types.hpp:13


class LogicError(RuntimeError):
    """std::logic_error."""


class SingularBlockError(RuntimeError):
    """bjgmres::SingularBlockError (lu.hpp:52-60): zero pivot with eps_pivot = 0."""

    def __init__(self, what: str, column: int, block: int = -1):
        super().__init__(what)
        self._column = column
        self.block = block

    def column(self) -> int:
        return self._column


def library():
    return _abi.load()


def _raise(code: int, msg: str, info: Optional[_abi.SetupInfo] = None):
    if code == _abi.HPBJ_EINVAL:
        raise ValueError(msg)
    if code == _abi.HPBJ_ELOGIC:
        raise LogicError(msg)
    if code == _abi.HPBJ_ERANGE:
        raise IndexError(msg)
    if code == _abi.HPBJ_ESINGULAR:
        col = int(info.singular_column) if info is not None else -1
        blk = int(info.singular_block) if info is not None else -1
        raise SingularBlockError(msg, col, blk)
    raise RuntimeError(msg)


def _p(a, t):
    return a.ctypes.data_as(t)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
@dataclass
class SparseMatrix:
    """CSR matrix, FP64 master values (sparse_matrix.hpp:23-62)."""

    nrows: int
    row_starts: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_starts = _i64(self.row_starts)
        self.col_indices = _i64(self.col_indices)
        self.values = _f64(self.values)
        if len(self.row_starts) != self.nrows + 1:
            raise ValueError("sparse matrix: row_starts length")

    @property
    def n(self) -> int:
        return self.nrows

    def rows(self) -> int:
        return self.nrows

    def nnz(self) -> int:
        return int(self.row_starts[-1])

    @staticmethod
    def from_triplets(rows, cols, vals, n: int) -> "SparseMatrix":
        """SparseMatrix::from_triplets (sparse_matrix.cpp:52-88): sort by
        (row, col, value bits), sum duplicates in that order."""
        rows = _i64(rows)
        cols = _i64(cols)
        vals = _f64(vals)
        if len(rows) and (rows.min() < 0 or rows.max() >= n or cols.min() < 0 or cols.max() >= n):
            raise IndexError("from_triplets: index out of range")
        order = np.lexsort((vals.view(np.uint64), cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        out_r, out_c, out_v = [], [], []
        k = 0
        while k < len(rows):
            r, c, s = rows[k], cols[k], 0.0
            while k < len(rows) and rows[k] == r and cols[k] == c:
                s += float(vals[k])
                k += 1
            out_r.append(r)
            out_c.append(c)
            out_v.append(s)
        rs = np.zeros(n + 1, np.int64)
        np.add.at(rs, np.asarray(out_r, np.int64) + 1, 1)
        return SparseMatrix(n, np.cumsum(rs), np.asarray(out_c, np.int64), np.asarray(out_v, np.float64))


@dataclass
class WeightedGraph:
    """graph.hpp:17-25 as CSR adjacency (sorted by neighbour)."""

    num_nodes: int
    start: np.ndarray
    neighbor: np.ndarray
    weight: np.ndarray

    def degree(self, v: int) -> int:
        return int(self.start[v + 1] - self.start[v])

    def num_edges(self) -> int:
        return int(self.start[-1]) // 2


@dataclass
class Partition:
    """partition.hpp:14-28."""

    num_blocks: int
    assignment: np.ndarray
    perm: np.ndarray
    block_starts: np.ndarray

    def num_nodes(self) -> int:
        return len(self.assignment)

    def block_size(self, b: int) -> int:
        return int(self.block_starts[b + 1] - self.block_starts[b])


def graph_from_matrix(a: SparseMatrix) -> WeightedGraph:
    lib = library()
    n = a.n
    cap = 2 * a.nnz() + 1
    st = np.zeros(n + 1, np.int64)
    nb = np.zeros(cap, np.int64)
    w = np.zeros(cap)
    rc = lib.hpbj_graph_from_matrix(n, _p(a.row_starts, _abi.i64p), _p(a.col_indices, _abi.i64p),
                                    _p(a.values, _abi.f64p), _p(st, _abi.i64p), _p(nb, _abi.i64p),
                                    _p(w, _abi.f64p), cap)
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())
    k = int(st[-1])
    return WeightedGraph(n, st, nb[:k].copy(), w[:k].copy())


def partition_graph(g, s: int, imbalance_tol: float = 0.1) -> Partition:
    """partition_graph (partition.hpp:38-39). Accepts a WeightedGraph or, as a
    fused fast path, the SparseMatrix itself (graph_from_matrix + partition)."""
    lib = library()
    if isinstance(g, SparseMatrix):
        n = g.n
        asg, perm, bst = np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(max(s, 0) + 1, np.int64)
        rc = lib.hpbj_partition_graph(n, _p(g.row_starts, _abi.i64p), _p(g.col_indices, _abi.i64p),
                                      _p(g.values, _abi.f64p), s, imbalance_tol, _p(asg, _abi.i64p),
                                      _p(perm, _abi.i64p), _p(bst, _abi.i64p))
    else:
        n = g.num_nodes
        st, nb, w = _i64(g.start), _i64(g.neighbor), _f64(g.weight)
        asg, perm, bst = np.zeros(n, np.int64), np.zeros(n, np.int64), np.zeros(max(s, 0) + 1, np.int64)
        rc = lib.hpbj_partition_adjacency(n, _p(st, _abi.i64p), _p(nb, _abi.i64p), _p(w, _abi.f64p), s,
                                          imbalance_tol, _p(asg, _abi.i64p), _p(perm, _abi.i64p),
                                          _p(bst, _abi.i64p))
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())
    return Partition(s, asg, perm, bst)


def partition_from_assignment(assignment, s: int) -> Partition:
    lib = library()
    asg = _i64(assignment)
    n = len(asg)
    perm, bst = np.zeros(n, np.int64), np.zeros(max(s, 0) + 1, np.int64)
    rc = lib.hpbj_partition_from_assignment(n, _p(asg, _abi.i64p), s, _p(perm, _abi.i64p), _p(bst, _abi.i64p))
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())
    return Partition(s, asg.copy(), perm, bst)


# ---------------------------------------------------------------------------
# Matrix Market / CSR cache / partition files
def _take_arrays(lib, n_rows, prp, pci, pval):
    nnz = int(prp[n_rows]) if n_rows >= 0 else 0
    rp = np.ctypeslib.as_array(prp, (n_rows + 1,)).copy()
    ci = np.ctypeslib.as_array(pci, (max(nnz, 1),))[:nnz].copy()
    val = np.ctypeslib.as_array(pval, (max(nnz, 1),))[:nnz].copy()
    for p_ in (prp, pci, pval):
        lib.hpbj_free(ctypes.cast(p_, ctypes.c_void_p))
    return rp, ci, val


def read_matrix_market(path: str) -> SparseMatrix:
    """read_matrix_market_file (matrix_market.cpp:36-106) for square matrices."""
    lib = library()
    nr, nc = ctypes.c_int64(), ctypes.c_int64()
    prp, pci = ctypes.POINTER(ctypes.c_int64)(), ctypes.POINTER(ctypes.c_int64)()
    pval = ctypes.POINTER(ctypes.c_double)()
    rc = lib.hpbj_mm_read(os.fsencode(path), ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(prp),
                          ctypes.byref(pci), ctypes.byref(pval))
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())
    rp, ci, val = _take_arrays(lib, nr.value, prp, pci, pval)
    if nr.value != nc.value:
        raise ValueError(f"matrix must be square, got {nr.value}x{nc.value}")
    return SparseMatrix(nr.value, rp, ci, val)


def write_matrix_market(path: str, a: SparseMatrix) -> None:
    """write_matrix_market_file (matrix_market.cpp:108-121): real general, %.17g."""
    lib = library()
    rc = lib.hpbj_mm_write(os.fsencode(path), a.n, a.n, _p(a.row_starts, _abi.i64p), _p(a.col_indices, _abi.i64p),
                           _p(a.values, _abi.f64p))
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())


def write_csr_cache(path: str, a: SparseMatrix) -> None:
    """Binary CSR cache ("HPBJCSR1"): the configs / SuiteSparse inputs load without parsing."""
    lib = library()
    rc = lib.hpbj_csr_cache_write(os.fsencode(path), a.n, _p(a.row_starts, _abi.i64p), _p(a.col_indices, _abi.i64p),
                                  _p(a.values, _abi.f64p))
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())


def read_csr_cache(path: str) -> SparseMatrix:
    lib = library()
    n = ctypes.c_int64()
    prp, pci = ctypes.POINTER(ctypes.c_int64)(), ctypes.POINTER(ctypes.c_int64)()
    pval = ctypes.POINTER(ctypes.c_double)()
    rc = lib.hpbj_csr_cache_read(os.fsencode(path), ctypes.byref(n), ctypes.byref(prp), ctypes.byref(pci),
                                 ctypes.byref(pval))
    if rc:
        _raise(rc, lib.hpbj_last_error(None).decode())
    rp, ci, val = _take_arrays(lib, n.value, prp, pci, pval)
    return SparseMatrix(n.value, rp, ci, val)


def export_partition(path: str, p: Partition) -> None:
    """export_partition (partition.cpp:174-176): one block index per line."""
    with open(path, "w") as f:
        f.write("".join(f"{int(b)}\n" for b in p.assignment))


def import_partition(path: str, n: int, s: int) -> Partition:
    """import_partition (partition.cpp:145-172): blank lines skipped, errors name the line."""
    asg = []
    with open(path) as f:
        for line_no, line in enumerate(f, 1):
            tok = line.split()
            if not tok:
                continue
            try:
                b = int(tok[0])
            except ValueError:
                raise RuntimeError(f"partition file: line {line_no}: malformed") from None
            if b < 0 or b >= s:
                raise IndexError(f"partition file: line {line_no}: block index {b} out of range")
            asg.append(b)
    if len(asg) != n:
        raise RuntimeError(f"partition file: expected {n} lines, got {len(asg)}")
    return partition_from_assignment(np.asarray(asg, np.int64), s)


def measure_block_nnz(p: Partition, a: SparseMatrix):
    """measure_block_nnz (partition.cpp:178-195): nnz of each diagonal block and max/mean."""
    rows = np.repeat(np.arange(a.n), np.diff(a.row_starts))
    asg = np.asarray(p.assignment)
    inblk = asg[rows] == asg[a.col_indices]
    bn = np.bincount(asg[rows][inblk], minlength=p.num_blocks).astype(np.int64)
    mean = bn.sum() / p.num_blocks
    return bn, (bn.max() / mean if mean > 0 else 0.0)


def cut_weight(g: "WeightedGraph", p: Partition) -> float:
    """cut_weight (partition.cpp:197-204): sum of w over u < v edges across blocks (u ascending)."""
    asg = np.asarray(p.assignment)
    cut = 0.0
    for u in range(g.num_nodes):
        for k in range(int(g.start[u]), int(g.start[u + 1])):
            v = int(g.neighbor[k])
            if u < v and asg[u] != asg[v]:
                cut += float(g.weight[k])
    return cut


# ---------------------------------------------------------------------------
class Context:
    """Owns one hpbj_ctx (device buffers + CUDA stream)."""

    def __init__(self, device: int = 0):
        self.lib = library()
        h = ctypes.c_void_p()
        rc = self.lib.hpbj_create(ctypes.byref(h), device)
        if rc:
            _raise(rc, self.lib.hpbj_last_error(None).decode())
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.hpbj_destroy(h)
            self.h = None

    def check(self, rc, info=None):
        if rc:
            _raise(rc, self.lib.hpbj_last_error(self.h).decode(), info)

    def set_matrix(self, a: SparseMatrix):
        self.check(self.lib.hpbj_set_matrix(self.h, a.n, _p(a.row_starts, _abi.i64p), _p(a.col_indices, _abi.i64p),
                                            _p(a.values, _abi.f64p)))

    def update_values(self, values):
        v = _f64(values)
        self.check(self.lib.hpbj_update_values(self.h, _p(v, _abi.f64p)))

    def spmv(self, x):
        x = _f64(x)
        y = np.zeros_like(x)
        self.check(self.lib.hpbj_spmv(self.h, _p(x, _abi.f64p), _p(y, _abi.f64p)))
        return y

    def bj_setup(self, part: Partition, eps_pivot: float) -> _abi.SetupInfo:
        info = _abi.SetupInfo()
        perm, bst = _i64(part.perm), _i64(part.block_starts)
        rc = self.lib.hpbj_bj_setup(self.h, part.num_blocks, _p(perm, _abi.i64p), _p(bst, _abi.i64p), eps_pivot,
                                    ctypes.byref(info))
        self.check(rc, info)
        return info

    def bj_refactor(self) -> _abi.SetupInfo:
        info = _abi.SetupInfo()
        self.check(self.lib.hpbj_bj_refactor(self.h, ctypes.byref(info)), info)
        return info

    def apply(self, v):
        v = _f64(v)
        z = np.zeros_like(v)
        self.check(self.lib.hpbj_bj_apply(self.h, _p(v, _abi.f64p), _p(z, _abi.f64p)))
        return z

    def ilu0_setup(self) -> _abi.SetupInfo:
        info = _abi.SetupInfo()
        self.check(self.lib.hpbj_ilu0_setup(self.h, ctypes.byref(info)), info)
        return info

    def identity_setup(self):
        self.check(self.lib.hpbj_identity_setup(self.h))

    def precond_apply(self, v):
        v = _f64(v)
        z = np.zeros_like(v)
        self.check(self.lib.hpbj_precond_apply(self.h, _p(v, _abi.f64p), _p(z, _abi.f64p)))
        return z

    def ilu0_values(self, nnz: int):
        out = np.zeros(nnz)
        self.check(self.lib.hpbj_get_ilu0_values(self.h, _p(out, _abi.f64p)))
        return out

    def set_neumann_order(self, order: int):
        self.check(self.lib.hpbj_bj_set_neumann_order(self.h, int(order)))

    def apply_neumann(self, v, k: int):
        v = _f64(v)
        z = np.zeros_like(v)
        self.check(self.lib.hpbj_bj_apply_neumann(self.h, _p(v, _abi.f64p), _p(z, _abi.f64p), int(k)))
        return z

    def block_factors(self, b: int):
        d = ctypes.c_int64()
        self.check(self.lib.hpbj_get_block_factors(self.h, b, ctypes.byref(d), None, None))
        f = np.zeros(d.value * d.value, np.float32)
        piv = np.zeros(d.value, np.int64)
        self.check(self.lib.hpbj_get_block_factors(self.h, b, ctypes.byref(d), _p(f, _abi.f32p),
                                                   _p(piv, _abi.i64p)))
        return f.reshape(d.value, d.value), piv

    def block_stats(self, s: int):
        dims, pert = np.zeros(s, np.int64), np.zeros(s, np.int64)
        self.check(self.lib.hpbj_get_block_stats(self.h, _p(dims, _abi.i64p), _p(pert, _abi.i64p)))
        return dims, pert

    def block_diagnostics(self, s: int):
        """(cond_estimate[s], error_bound[s]) of the factored blocks (device)."""
        cond, eb = np.zeros(s), np.zeros(s)
        self.check(self.lib.hpbj_get_block_diagnostics(self.h, _p(cond, _abi.f64p), _p(eb, _abi.f64p)))
        return cond, eb

    def launches(self) -> int:
        return int(self.lib.hpbj_kernel_launches(self.h))

    def set_profiling(self, on: bool):
        self.check(self.lib.hpbj_set_profiling(self.h, 1 if on else 0))

    def kernel_stats(self):
        arr = (_abi.KernelStat * _abi.HPBJ_K_COUNT)()
        self.check(self.lib.hpbj_get_kernel_stats(self.h, arr))
        return [dict(launches=s.launches, total_ms=s.total_ms, bytes_per_launch=s.bytes_per_launch, steps=s.steps,
                     total_bytes=s.total_bytes) for s in arr]

    def set_fused(self, on: bool):
        """Whole Arnoldi cycle as one persistent kernel when it fits (default)."""
        self.check(self.lib.hpbj_set_fused(self.h, 1 if on else 0))

    def set_graph(self, on: bool):
        """Solve as one CUDA graph (default) or host-enqueued launches."""
        self.check(self.lib.hpbj_set_graph(self.h, 1 if on else 0))

    def gmres(self, b, cfg: "GmresConfig", device_ptrs=None):
        opts = cfg.to_opts()
        rep = _abi.Report()
        hcap = cfg.restart_m * cfg.max_restarts + 2
        hist = (_abi.HistoryPoint * hcap)()
        cyc = np.zeros(cfg.max_restarts + 1)
        if device_ptrs is not None:
            d_b, d_x = device_ptrs
            rc = self.lib.hpbj_gmres_device(self.h, ctypes.c_void_p(d_b), ctypes.c_void_p(d_x), ctypes.byref(opts),
                                            ctypes.byref(rep), hist, hcap, _p(cyc, _abi.f64p), len(cyc))
            x = None
        else:
            b = _f64(b)
            x = np.zeros_like(b)
            rc = self.lib.hpbj_gmres(self.h, _p(b, _abi.f64p), _p(x, _abi.f64p), ctypes.byref(opts),
                                     ctypes.byref(rep), hist, hcap, _p(cyc, _abi.f64p), len(cyc))
        self.check(rc)
        hl = min(int(rep.history_len), hcap)
        history = [HistoryPoint(int(hist[k].cycle), int(hist[k].iteration), float(hist[k].relative_residual))
                   for k in range(hl)]
        report = SolveReport(
            converged=bool(rep.converged),
            total_iterations=int(rep.total_iterations),
            restarts=int(rep.restarts),
            residual_history=history,
            cycle_residuals=cyc[: int(rep.cycles)].tolist(),
            final_residual=float(rep.final_residual),
            breakdown=bool(rep.breakdown),
            ls_rank_deficient=bool(rep.ls_rank_deficient),
            iterate_seconds=float(rep.ms_solve) / 1e3,
        )
        return x, report


# ---------------------------------------------------------------------------
@dataclass
class BlockJacobiOptions:
    """preconditioner.hpp:32-38 (Hybrid policy only: FP32 factors)."""

    eps_pivot: float = 1e-10
    neumann_order: int = 0  # 0 = direct block solves; k > 0: truncated Neumann series in the solve


class Preconditioner:
    """Preconditioner resident on one B200 (preconditioner.hpp:50-98): block
    Jacobi (FP32 factors), ILU(0) (FP64 factors) or the identity."""

    BLOCK_JACOBI, ILU0, IDENTITY = "block_jacobi", "ilu0", "identity"

    def __init__(self, ctx: Optional[Context], a: Optional[SparseMatrix], part: Optional[Partition],
                 opts: Optional[BlockJacobiOptions], info: Optional[_abi.SetupInfo], kind: str = "block_jacobi",
                 n: Optional[int] = None):
        self.ctx = ctx
        self.matrix = a
        self.partition = part
        self.opts = opts or BlockJacobiOptions()
        self.info = info
        self.kind = kind
        self._n = a.n if a is not None else n

    @staticmethod
    def identity(n: int) -> "Preconditioner":
        """Preconditioner::identity (preconditioner.cpp:90-92); bound to the
        matrix by the solve."""
        return Preconditioner(None, None, None, None, None, kind=Preconditioner.IDENTITY, n=int(n))

    @staticmethod
    def from_ilu0(a: SparseMatrix, device: int = 0, ctx: Optional[Context] = None) -> "Preconditioner":
        """Preconditioner::from_ilu0 (preconditioner.cpp:94-98): ILU(0) on the
        device, FP64 factors in A's pattern."""
        ctx = ctx or Context(device)
        ctx.set_matrix(a)
        info = ctx.ilu0_setup()
        return Preconditioner(ctx, a, None, None, info, kind=Preconditioner.ILU0)

    def ilu0_values(self) -> np.ndarray:
        """The factored values in A's pattern (L strictly lower, then U)."""
        if self.kind != Preconditioner.ILU0:
            raise LogicError("ilu0: factors not set up")
        return self.ctx.ilu0_values(self.matrix.nnz())

    @staticmethod
    def block_jacobi(a: SparseMatrix, partition: Partition, opts: Optional[BlockJacobiOptions] = None,
                     device: int = 0, ctx: Optional[Context] = None) -> "Preconditioner":
        opts = opts or BlockJacobiOptions()
        if partition.num_nodes() != a.n:
            raise ValueError("block_jacobi: partition does not cover the matrix")
        ctx = ctx or Context(device)
        ctx.set_neumann_order(opts.neumann_order)
        ctx.set_matrix(a)
        info = ctx.bj_setup(partition, opts.eps_pivot)
        return Preconditioner(ctx, a, partition, opts, info)

    def dim(self) -> int:
        return self._n

    def apply(self, v) -> np.ndarray:
        """z with M z = v: apply<float> for block Jacobi (FP32 factors, FP32
        arithmetic), apply<double> for ILU(0) and the identity."""
        v = _f64(v)
        if len(v) != self.dim():
            raise ValueError("preconditioner apply: dimension mismatch")
        if self.kind == Preconditioner.IDENTITY:
            return v.copy()
        if self.kind == Preconditioner.ILU0:
            return self.ctx.precond_apply(v)
        return self.ctx.apply(v)

    def neumann_order(self) -> int:
        return self.opts.neumann_order

    def apply_neumann(self, v, k: int) -> np.ndarray:
        """apply_neumann<float> (preconditioner.cpp:200-220): z = sum_{i=0..k}
        (I - Phi^-1 A)^i Phi^-1 v on the matrix the preconditioner was built from."""
        if self.kind != Preconditioner.BLOCK_JACOBI:
            raise LogicError("apply_neumann: block factors not available")
        v = _f64(v)
        if len(v) != self.dim():
            raise ValueError("preconditioner apply: dimension mismatch")
        return self.ctx.apply_neumann(v, k)

    def block_factors(self, b: int):
        return self.ctx.block_factors(b)

    def stats(self, with_cond_estimates: bool = True):
        """PreconditionerStats per block (preconditioner.hpp:14-20); the condition
        estimates / error bounds are computed on the device on first request."""
        s = self.partition.num_blocks
        dims, pert = self.ctx.block_stats(s)
        cond, eb = self.ctx.block_diagnostics(s) if with_cond_estimates else (np.zeros(s), np.zeros(s))
        return [dict(block_dim=int(d), perturbation_count=int(p), cond_estimate=float(c), error_bound=float(e))
                for d, p, c, e in zip(dims, pert, cond, eb)]


@dataclass
class GmresConfig:
    """gmres.hpp:89-97. precision is PrecisionPolicy::mode (types.hpp:15-26):
    "hybrid" (FP32 preconditioner; the default here, the block-Jacobi device
    path) or "double" (FP64 preconditioner: ILU(0), identity). The
    attainable-floor break uses its working roundoff, 2^-24 or 2^-53
    (gmres.cpp:130-145), unless floor_roundoff overrides it."""

    restart_m: int = 50
    tol: float = 1e-8
    max_restarts: int = 40
    absolute_tol: bool = False
    breakdown_tol_factor: float = 1e2
    floor_roundoff: Optional[float] = None
    precision: str = "hybrid"

    def to_opts(self) -> _abi.GmresOpts:
        o = _abi.GmresOpts()
        o.restart_m = int(self.restart_m)
        o.tol = float(self.tol)
        o.max_restarts = int(self.max_restarts)
        o.absolute_tol = 1 if self.absolute_tol else 0
        o.breakdown_tol_factor = float(self.breakdown_tol_factor)
        if self.floor_roundoff is not None:
            o.floor_roundoff = float(self.floor_roundoff)
        else:
            o.floor_roundoff = ROUNDOFF_DOUBLE if self.precision == "double" else ROUNDOFF_SINGLE
        return o


@dataclass
class HistoryPoint:
    cycle: int
    iteration: int
    relative_residual: float


@dataclass
class SolveReport:
    converged: bool = False
    total_iterations: int = 0
    restarts: int = 0
    residual_history: List[HistoryPoint] = field(default_factory=list)
    cycle_residuals: List[float] = field(default_factory=list)
    final_residual: float = 0.0
    breakdown: bool = False
    ls_rank_deficient: bool = False
    setup_seconds: float = 0.0
    iterate_seconds: float = 0.0


@dataclass
class SolveResult:
    x: np.ndarray
    report: SolveReport


def hybrid_restart_gmres(a: SparseMatrix, p: Preconditioner, b, config: GmresConfig) -> SolveResult:
    """hybrid_restart_gmres (gmres.hpp:145-147): FP64 SpMV and Arnoldi, FP32
    block-Jacobi apply, FP64 true residual per restart cycle."""
    b = _f64(b)
    if a.n != len(b):
        raise ValueError("gmres: rhs dimension mismatch")
    if config.restart_m < 1 or config.tol <= 0.0 or config.max_restarts < 1:
        raise ValueError("gmres: invalid config")
    if config.restart_m > 1024:  # before the history buffers are sized from it
        raise ValueError("gmres: restart_m > 1024 unsupported")
    if config.max_restarts > 1 << 24:
        raise ValueError("gmres: max_restarts too large")
    if config.precision not in ("hybrid", "double"):
        raise ValueError("gmres: unknown precision: " + str(config.precision))
    if p.kind == Preconditioner.IDENTITY:
        if p.dim() != a.n:
            raise ValueError("gmres: preconditioner dimension mismatch")
        if p.ctx is None or p.matrix is not a:  # bind the identity to this matrix
            p.ctx = Context(0)
            p.ctx.set_matrix(a)
            p.ctx.identity_setup()
            p.matrix = a
    elif p.matrix is not a:
        raise ValueError("gmres: the preconditioner must be built from this matrix (device-resident)")
    if p.kind == Preconditioner.ILU0 and config.precision == "hybrid":
        # the reference applies ILU(0) through lu_solve<float> on factors that
        # never get binary32 copies (lu.hpp:94-99): Hybrid + ILU(0) throws there
        raise LogicError("values_low requested before materialize_low()")
    if p.kind == Preconditioner.BLOCK_JACOBI and config.precision == "double":
        raise ValueError("gmres: DoubleOnly block Jacobi is not implemented on the GPU path (FP32 factors)")
    x, rep = p.ctx.gmres(b, config)
    return SolveResult(x, rep)
