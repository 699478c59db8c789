"""Truncated Neumann-series preconditioning: apply_neumann
(preconditioner.cpp:200-220) and the solve with BlockJacobiOptions::
neumann_order > 0 (preconditioned<T>, gmres.cpp:91-95). The known answers are
test_preconditioners.cpp:213-259; parity is against the reference library
(oracle/_ref) on the same inputs."""
import numpy as np
import pytest

import paper_2509_09139_b200 as hp
from tests import fixtures as fx


# ------------------------------------------------ oracle pins (CPU, no GPU)
def test_reference_neumann_known_answers(ref):
    a = fx.diag_csr([2.0, 4.0, 8.0])  # Phi = A: every correction term vanishes
    for k in range(4):
        z = ref.apply_neumann(a.row_starts, a.col_indices, a.values, 3, [0, 1, 2], [1.0, 1.0, 1.0], 3, k,
                              fp32=False)
        assert np.array_equal(z, [0.5, 0.25, 0.125])
    a = hp.SparseMatrix.from_triplets([0, 0, 1, 1], [0, 1, 0, 1], [2.0, 1.0, 1.0, 2.0], 2)
    z = ref.apply_neumann(a.row_starts, a.col_indices, a.values, 2, [0, 1], [1.0, 0.0], 1, 1, fp32=False)
    assert np.array_equal(z, [0.5, -0.25])


# ------------------------------------------------------------- device path
@pytest.mark.gpu
def test_diagonal_phi_truncates_exactly():
    a = fx.diag_csr([2.0, 4.0, 8.0])
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 1, 2], 3),
                                       hp.BlockJacobiOptions(neumann_order=3))
    for k in range(4):
        assert np.array_equal(p.apply_neumann([1.0, 1.0, 1.0], k), [0.5, 0.25, 0.125])


@pytest.mark.gpu
def test_order_zero_equals_apply():
    a = fx.random_dd(12, 3, 41)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_graph(a, 3, 0.1), hp.BlockJacobiOptions(neumann_order=2))
    v = fx.random_vector(12, 5)
    assert np.array_equal(p.apply_neumann(v, 0), p.apply(v))


@pytest.mark.gpu
def test_first_order_series_example():
    a = hp.SparseMatrix.from_triplets([0, 0, 1, 1], [0, 1, 0, 1], [2.0, 1.0, 1.0, 2.0], 2)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 1], 2),
                                       hp.BlockJacobiOptions(neumann_order=1))
    assert np.array_equal(p.apply_neumann([1.0, 0.0], 1), [0.5, -0.25])


@pytest.mark.gpu
def test_missing_data_errors():
    a = fx.identity_csr(2)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 1], 2))
    with pytest.raises(ValueError, match="order exceeds"):
        p.apply_neumann([1.0, 2.0], 1)
    with pytest.raises(ValueError):
        p.apply_neumann([1.0, 2.0], -1)
    c = hp.Context(0)
    c.set_matrix(a)
    with pytest.raises(hp.LogicError, match="block factors not available"):
        c.apply_neumann(np.array([1.0, 2.0]), 0)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_apply_neumann_matches_reference(ref, k):
    a = fx.random_dd(300, 5, 21)
    part = hp.partition_graph(a, 6, 0.1)
    p = hp.Preconditioner.block_jacobi(a, part, hp.BlockJacobiOptions(neumann_order=3))
    v = np.random.default_rng(3).uniform(-1, 1, a.n)
    z = p.apply_neumann(v, k)
    zr = ref.apply_neumann(a.row_starts, a.col_indices, a.values, 6, part.assignment, v, 3, k, fp32=True)
    zd = ref.apply_neumann(a.row_starts, a.col_indices, a.values, 6, part.assignment, v, 3, k, fp32=False)
    # FP32 series: the reference's binary32 SpMV vs our FP64 SpMV of the FP32 term
    assert np.linalg.norm(z - zr) <= 4e-6 * np.linalg.norm(zr)
    assert np.linalg.norm(z - zd) <= 1e-5 * np.linalg.norm(zd)
    # the series converges towards A^-1 v (rho(I - Phi^-1 A) < 1 for this diagonally dominant A)
    e = np.linalg.solve(fx.to_dense(a), v)
    err = np.linalg.norm(z - e)
    if k > 0:
        z0 = p.apply_neumann(v, k - 1)
        assert err < np.linalg.norm(z0 - e)


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("mat", ["lap20", "rdd300"])
def test_solve_with_neumann_matches_reference(ref, order, fused, mat):
    a, s = (fx.laplacian_2d(20, 20), 8) if mat == "lap20" else (fx.random_dd(300, 5, 21), 6)
    part = hp.partition_graph(a, s, 0.1)
    b = fx.ones(a.n)
    p = hp.Preconditioner.block_jacobi(a, part, hp.BlockJacobiOptions(neumann_order=order))
    p.ctx.set_fused(fused)  # the series runs on the unfused step graph either way
    cfg = hp.GmresConfig(restart_m=30, tol=1e-10, max_restarts=40)
    out = hp.hybrid_restart_gmres(a, p, b, cfg)
    r = out.report
    assert r.converged
    res = np.linalg.norm(b - fx.to_dense(a) @ out.x) / np.linalg.norm(b)
    assert res <= 1e-10
    refout = ref.solve(a.row_starts, a.col_indices, a.values, s, b, 30, 1e-10, 40, hybrid=True,
                       assignment=part.assignment, neumann_order=order)
    assert abs(r.total_iterations - refout.total_iterations) <= 1, (r.total_iterations, refout.total_iterations)
    # a stronger preconditioner: fewer iterations than the direct block solves
    p0 = hp.Preconditioner.block_jacobi(a, part)
    assert r.total_iterations < hp.hybrid_restart_gmres(a, p0, b, cfg).report.total_iterations
