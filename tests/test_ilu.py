"""ILU(0) and identity preconditioners on the device:
ilu0 (lu.cpp:227-312), Preconditioner::from_ilu0 / identity
(preconditioner.cpp:90-98), their FP64 apply and the DoubleOnly solve. The
known answers are test_lu_kernels.cpp:233-291 and test_preconditioners.cpp:
292-301; parity is against the reference library (oracle/_ref): factors and
applies bit-identical, solves with the same iteration counts."""
import numpy as np
import pytest

import paper_2509_09139_b200 as hp
from oracle import OracleError
from paper_2509_09139_b200.workloads import generate
from tests import fixtures as fx


def _matrices():
    return {
        "diag": fx.diag_csr([2.0, 3.0, 4.0]),
        "tridiag": fx.tridiag(3, -1.0, 2.0, -1.0),
        "lap12": fx.laplacian_2d(12, 12),
        "rdd300": fx.random_dd(300, 5, 21),
        "cd20": fx.convection_diffusion_2d(20, 20, 20.0, -10.0),
    }


def _dense_lu(a, lu):
    """L (unit lower) and U from the in-pattern factored values."""
    n = a.n
    L, U = np.eye(n), np.zeros((n, n))
    for i in range(n):
        for k in range(a.row_starts[i], a.row_starts[i + 1]):
            j = a.col_indices[k]
            (L if j < i else U)[i, j] = lu[k]
    return L, U


# ------------------------------------------------ oracle pins (CPU, no GPU)
def test_reference_ilu0_known_answers(ref):
    a = fx.diag_csr([2.0, 3.0, 4.0])  # DiagonalMatrixIsExact
    assert np.array_equal(ref.ilu0_values(a.row_starts, a.col_indices, a.values), [2.0, 3.0, 4.0])
    a = fx.tridiag(3, -1.0, 2.0, -1.0)  # TridiagonalEqualsExactLu: no fill
    L, U = _dense_lu(a, ref.ilu0_values(a.row_starts, a.col_indices, a.values))
    assert np.allclose(L @ U, fx.to_dense(a), rtol=0, atol=1e-15)
    a = fx.laplacian_2d(3, 3)  # LaplacianKeepsPatternAndLeavesResidual
    L, U = _dense_lu(a, ref.ilu0_values(a.row_starts, a.col_indices, a.values))
    assert np.linalg.norm(fx.to_dense(a) - L @ U) > 1e-8
    bad = hp.SparseMatrix.from_triplets([0, 1], [1, 0], [1.0, 1.0], 2)  # RejectsStructurallyZeroDiagonal
    with pytest.raises(OracleError, match="structurally zero diagonal in row 0"):
        ref.ilu0_values(bad.row_starts, bad.col_indices, bad.values)
    z = hp.SparseMatrix.from_triplets([0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0], 2)  # ReportsZeroPivotRow
    with pytest.raises(OracleError, match="zero diagonal pivot in row 1"):
        ref.ilu0_values(z.row_starts, z.col_indices, z.values)


def test_reference_rejects_hybrid_ilu0(ref):
    """The reference applies ILU(0) through lu_solve<float> on factors without
    binary32 copies: a Hybrid solve throws (the device mirror raises the same)."""
    a = fx.laplacian_2d(6, 6)
    with pytest.raises(OracleError, match="values_low requested before materialize_low"):
        ref.solve_ilu0(a.row_starts, a.col_indices, a.values, fx.ones(a.n), 20, 1e-10, 10, hybrid=True)


# ------------------------------------------------------------- device path
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["diag", "tridiag", "lap12", "rdd300", "cd20"])
def test_ilu0_factors_bit_identical(ref, name):
    a = _matrices()[name]
    p = hp.Preconditioner.from_ilu0(a)
    assert np.array_equal(p.ilu0_values(), ref.ilu0_values(a.row_starts, a.col_indices, a.values))


@pytest.mark.gpu
@pytest.mark.parametrize("config", [0, 1])
def test_ilu0_factors_and_apply_bit_identical_on_workloads(ref, config):
    s = generate(config)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    p = hp.Preconditioner.from_ilu0(a)
    assert np.array_equal(p.ilu0_values(), ref.ilu0_values(s.row_ptr, s.col, s.val))
    v = np.random.default_rng(config).uniform(-1, 1, s.n)
    assert np.array_equal(p.apply(v), ref.ilu0_apply(s.row_ptr, s.col, s.val, v))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["ticketed", "sweep"])
@pytest.mark.parametrize("name", ["lap12", "rdd300", "cd20"])
def test_ilu0_apply_bit_identical_and_repeatable(ref, name, mode, monkeypatch):
    # AppliesForwardBackSolve (test_preconditioners.cpp:292-301), through both
    # apply kernels (the setup normally times them and keeps the faster); the
    # ticketed one reuses its ticket counter and tags across calls (epochs)
    monkeypatch.setenv("HPBJ_ILU_APPLY", mode[0])
    a = _matrices()[name]
    p = hp.Preconditioner.from_ilu0(a)
    rng = np.random.default_rng(5)
    for _ in range(20):
        v = rng.uniform(-1, 1, a.n)
        assert np.array_equal(p.apply(v), ref.ilu0_apply(a.row_starts, a.col_indices, a.values, v))


@pytest.mark.gpu
def test_ilu0_errors():
    bad = hp.SparseMatrix.from_triplets([0, 1], [1, 0], [1.0, 1.0], 2)
    with pytest.raises(ValueError, match="structurally zero diagonal in row 0"):
        hp.Preconditioner.from_ilu0(bad)
    z = hp.SparseMatrix.from_triplets([0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0], 2)
    with pytest.raises(RuntimeError, match="zero diagonal pivot in row 1"):
        hp.Preconditioner.from_ilu0(z)
    a = fx.laplacian_2d(6, 6)
    p = hp.Preconditioner.from_ilu0(a)
    with pytest.raises(hp.LogicError, match="values_low requested before materialize_low"):
        hp.hybrid_restart_gmres(a, p, fx.ones(a.n), hp.GmresConfig(precision="hybrid"))
    with pytest.raises(hp.LogicError):
        p.apply_neumann(fx.ones(a.n), 0)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["ticketed", "sweep"])
@pytest.mark.parametrize("name", ["lap12", "rdd300"])
def test_ilu0_solve_matches_reference(ref, name, mode, monkeypatch):
    monkeypatch.setenv("HPBJ_ILU_APPLY", mode[0])
    a = _matrices()[name]
    b = fx.ones(a.n)
    cfg = hp.GmresConfig(restart_m=20, tol=1e-10, max_restarts=40, precision="double")
    out = hp.hybrid_restart_gmres(a, hp.Preconditioner.from_ilu0(a), b, cfg)
    r = ref.solve_ilu0(a.row_starts, a.col_indices, a.values, b, 20, 1e-10, 40, hybrid=False)
    assert out.report.converged == r.converged
    assert abs(out.report.total_iterations - r.total_iterations) <= 1, (out.report.total_iterations,
                                                                         r.total_iterations)
    if r.converged:
        res = np.linalg.norm(b - fx.to_dense(a) @ out.x) / np.linalg.norm(b)
        assert res <= 1e-10
        assert np.allclose(out.x, r.x, rtol=0, atol=1e-8 * np.abs(r.x).max())


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["double", "hybrid"])
def test_identity_solve_matches_reference(ref, precision):
    a = fx.random_dd(300, 5, 21)
    b = fx.ones(a.n)
    cfg = hp.GmresConfig(restart_m=30, tol=1e-10, max_restarts=40, precision=precision)
    p = hp.Preconditioner.identity(a.n)
    out = hp.hybrid_restart_gmres(a, p, b, cfg)
    assert np.array_equal(p.apply(b), b)
    r = ref.solve_identity(a.row_starts, a.col_indices, a.values, b, 30, 1e-10, 40, hybrid=precision == "hybrid")
    assert out.report.converged and r.converged
    assert abs(out.report.total_iterations - r.total_iterations) <= 1, (out.report.total_iterations,
                                                                         r.total_iterations)


@pytest.mark.gpu
def test_ilu0_solve_on_workload_config1(ref):
    """A 200k-row mesh (config 1 of BASELINE.json): factor + solve in FP64,
    iteration count against the reference's DoubleOnly ILU(0) GMRES."""
    s = generate(1)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    cfg = hp.GmresConfig(restart_m=50, tol=1e-10, max_restarts=40, precision="double")
    out = hp.hybrid_restart_gmres(a, hp.Preconditioner.from_ilu0(a), s.b, cfg)
    r = ref.solve_ilu0(s.row_ptr, s.col, s.val, s.b, 50, 1e-10, 40, hybrid=False)
    assert out.report.converged == r.converged
    assert abs(out.report.total_iterations - r.total_iterations) <= 1, (out.report.total_iterations,
                                                                         r.total_iterations)


@pytest.mark.gpu
def test_switching_preconditioners_on_one_context(ref):
    a = fx.random_dd(300, 5, 21)
    b = fx.ones(a.n)
    ctx = hp.Context(0)
    part = hp.partition_graph(a, 6, 0.1)
    pbj = hp.Preconditioner.block_jacobi(a, part, ctx=ctx)
    it_bj = hp.hybrid_restart_gmres(a, pbj, b, hp.GmresConfig(restart_m=30, tol=1e-10)).report.total_iterations
    pilu = hp.Preconditioner.from_ilu0(a, ctx=ctx)
    it_ilu = hp.hybrid_restart_gmres(a, pilu, b, hp.GmresConfig(restart_m=30, tol=1e-10, precision="double"))
    r = ref.solve_ilu0(a.row_starts, a.col_indices, a.values, b, 30, 1e-10, 40, hybrid=False)
    assert abs(it_ilu.report.total_iterations - r.total_iterations) <= 1
    # back to block Jacobi: same count as before
    pbj2 = hp.Preconditioner.block_jacobi(a, part, ctx=ctx)
    assert hp.hybrid_restart_gmres(a, pbj2, b, hp.GmresConfig(restart_m=30, tol=1e-10)).report.total_iterations \
        == it_bj
