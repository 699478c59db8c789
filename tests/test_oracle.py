"""Pin the CPU oracle (oracle/hpbj_oracle.c, our plain-C restatement of the
reference algorithm) against (a) the real reference library compiled from
/root/reference (oracle/_ref) — bit-exact — and (b) the committed golden
fixtures generated from the reference (tests/golden, make_golden.py)."""
import json
import os

import numpy as np
import pytest

from oracle import Port
from paper_2509_09139_b200.workloads import generate
from tests import fixtures as fx

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def port():
    return Port()


def _cases():
    return [("laplacian32", fx.laplacian_2d(32, 32), 16), ("laplacian16", fx.laplacian_2d(16, 16), 8),
            ("random_dd80", fx.random_dd(80, 4, 55), 4), ("convdiff", fx.convection_diffusion_2d(10, 10, 2.0, 1.0), 4),
            ("random_dd30", fx.random_dd(30, 4, 23), 5), ("tridiag4", fx.tridiag4(), 2)]


@pytest.mark.parametrize("name,a,s", _cases())
def test_port_bit_exact_vs_reference(ref, port, name, a, s):
    rp, ci, v = a.row_starts, a.col_indices, a.values
    x = fx.random_vector(a.n, 3)
    assert np.array_equal(port.spmv(rp, ci, v, x), ref.spmv(rp, ci, v, x))
    assert np.array_equal(port.spmv(rp, ci, v, x, fp32=True), ref.spmv(rp, ci, v, x, fp32=True))
    st, nb, w = port.graph(rp, ci, v)
    st2, nb2, w2 = ref.graph(rp, ci, v)
    assert np.array_equal(st, st2) and np.array_equal(nb, nb2) and np.array_equal(w, w2)
    asg = port.partition(rp, ci, v, s)
    asg2, _, _, _ = ref.partition(rp, ci, v, s)
    assert np.array_equal(asg, asg2)
    dims, f64, piv, pert = port.factors(rp, ci, v, s, asg)
    dims2, _, f64r, piv2, pert2 = ref.factors(rp, ci, v, s, asg, want64=True)
    assert np.array_equal(f64, f64r) and np.array_equal(piv, piv2) and np.array_equal(pert, pert2)
    for fp32 in (False, True):
        assert np.array_equal(port.apply(rp, ci, v, s, asg, x, fp32=fp32),
                              ref.apply(rp, ci, v, s, asg, x, fp32=fp32))
    b = fx.to_dense(a) @ np.ones(a.n)
    for mode, hyb in (("hybrid", True), ("double", False)):
        o = port.solve_full(rp, ci, v, s, asg, b, 50, 1e-8, 40, mode)
        r = ref.solve(rp, ci, v, s, b, 50, 1e-8, 40, hybrid=hyb, assignment=asg)
        assert o.total_iterations == r.total_iterations
        assert np.array_equal(o.x, r.x)
        assert np.array_equal(o.history, r.history) and np.array_equal(o.cycle_residuals, r.cycle_residuals)


def test_port_singular_block_and_regularisation(port):
    a = fx.diag_csr([1e-20, 1.0])  # test_lu_kernels.cpp:95-102
    dims, f64, piv, pert = port.factors(a.row_starts, a.col_indices, a.values, 1, [0, 0])
    assert pert[0] == 1 and f64[0] == 1e-10
    from oracle import OracleError
    b = fx.diag_csr([0.0, 1.0])
    with pytest.raises(OracleError):
        port.factors(b.row_starts, b.col_indices, b.values, 1, [0, 0], eps=0.0)


def test_port_pivot_known_answers(port):
    # test_lu_kernels.cpp:120-141: largest magnitude; ties -> smallest row
    import paper_2509_09139_b200 as hp
    a = hp.SparseMatrix.from_triplets([0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, -3.0, 1.0], 2)
    assert list(port.factors(a.row_starts, a.col_indices, a.values, 1, [0, 0], eps=0.0)[2]) == [1, 0]
    a = hp.SparseMatrix.from_triplets([0, 1, 0, 1], [0, 0, 1, 1], [2.0, -2.0, 1.0, 5.0], 2)
    assert list(port.factors(a.row_starts, a.col_indices, a.values, 1, [0, 0])[2]) == [0, 1]


def test_port_matches_config0_golden(port):
    g = json.load(open(os.path.join(GOLD, "config0.json")))
    npz = np.load(os.path.join(GOLD, "config0.npz"))
    s = generate(0)
    asg = npz["assignment"].astype(np.int64)
    assert np.array_equal(port.partition(s.row_ptr, s.col, s.val, s.num_blocks), asg)
    o = port.solve_full(s.row_ptr, s.col, s.val, s.num_blocks, asg, s.b, s.restart_m, s.tol, s.max_restarts)
    assert o.total_iterations == g["hybrid"]["total_iterations"]
    assert np.array_equal(o.x, npz["x_hybrid"])  # bit-exact with the reference run
    assert list(o.cycle_residuals) == g["hybrid"]["cycle_residuals"]
    d = port.solve_full(s.row_ptr, s.col, s.val, s.num_blocks, asg, s.b, s.restart_m, s.tol, s.max_restarts,
                        "double")
    assert np.array_equal(d.x, npz["x_double"])


@pytest.mark.parametrize("config", [1, 4])
def test_port_matches_golden_iterations(port, config):
    import paper_2509_09139_b200 as hp
    g = json.load(open(os.path.join(GOLD, f"config{config}.json")))
    s = generate(config)
    asg = hp.partition_graph(hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val), s.num_blocks).assignment
    o = port.solve_full(s.row_ptr, s.col, s.val, s.num_blocks, asg, s.b, s.restart_m, s.tol, s.max_restarts)
    assert o.total_iterations == g["hybrid"]["total_iterations"]
    assert o.cycle_residuals.tolist() == g["hybrid"]["cycle_residuals"]
    idx = np.array(g["hybrid"]["x_sample_idx"])
    assert np.array_equal(o.x[idx], np.array(g["hybrid"]["x_sample"]))


def test_mix_mode_iterations_track_hybrid(port):
    """The B200 precision mix (FP64 SpMV/Arnoldi, FP32 preconditioner, floor
    2^-24) reproduces reference Hybrid iteration counts."""
    for c in (0, 4):
        g = json.load(open(os.path.join(GOLD, f"config{c}.json")))
        s = generate(c)
        import paper_2509_09139_b200 as hp
        asg = hp.partition_graph(hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val), s.num_blocks).assignment
        o = port.solve_full(s.row_ptr, s.col, s.val, s.num_blocks, asg, s.b, s.restart_m, s.tol,
                            s.max_restarts, "mix")
        assert o.converged and o.final_residual <= s.tol
        its = g["hybrid"]["total_iterations"]
        assert abs(o.total_iterations - its) <= max(1, 0.05 * its)


def test_golden_inputs_pinned():
    for c in (0, 1, 4):
        g = json.load(open(os.path.join(GOLD, f"config{c}.json")))
        assert generate(c).digest() == g["input_sha256"]
