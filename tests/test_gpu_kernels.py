"""GPU parity of the individual kernels (through the C ABI) against the
reference library (oracle/_ref) and the reference's known-answer tests."""
import numpy as np
import pytest

import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate
from tests import fixtures as fx

pytestmark = pytest.mark.gpu


def _ctx_with(a):
    c = hp.Context(0)
    c.set_matrix(a)
    return c


def _sys_matrix(s):
    return hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)


# ---------------------------------------------------------------- SpMV (K1)
def _spmv_bound(a, x):
    """per-row |dy_i| <= 2 nnz_i 2^-53 sum_j |a_ij x_j| (FP reassociation/FMA)."""
    rs, ci, v = a.row_starts, a.col_indices, a.values
    absrow = np.zeros(a.n)
    np.add.at(absrow, np.repeat(np.arange(a.n), np.diff(rs)), np.abs(v * x[ci]))
    return 2.0 * np.maximum(np.diff(rs), 1) * 2.0 ** -53 * absrow


@pytest.mark.parametrize("config", [0, 1, 4, 2, 3])
def test_spmv_matches_reference(ref, config):
    s = generate(config)
    a = _sys_matrix(s)
    c = _ctx_with(a)
    x = np.random.default_rng(config).uniform(-1, 1, s.n)
    y = c.spmv(x)
    yr = ref.spmv(s.row_ptr, s.col, s.val, x)
    assert np.linalg.norm(y - yr) <= 1e-14 * np.linalg.norm(yr)
    assert np.all(np.abs(y - yr) <= _spmv_bound(a, x) + 1e-300)


def test_spmv_known_answers():
    # test_sparse_core.cpp:153-169
    c = _ctx_with(fx.identity_csr(4))
    assert np.array_equal(c.spmv([1, 2, 3, 4]), [1, 2, 3, 4])
    c = _ctx_with(hp.SparseMatrix.from_triplets([0, 1, 1], [0, 0, 1], [2.0, 1.0, 3.0], 2))
    assert np.array_equal(c.spmv([1.0, 1.0]), [2.0, 4.0])


def test_spmv_deterministic():
    a = fx.laplacian_2d(64, 80)  # test_sparse_core.cpp:204-215
    c = _ctx_with(a)
    x = fx.random_vector(a.n, 9)
    y1, y2 = c.spmv(x), c.spmv(x)
    assert np.array_equal(y1, y2)
    assert np.allclose(y1, fx.to_dense(a) @ x, rtol=0, atol=1e-13)


# ------------------------------------------------- block LU (K2 + K3)
def _factor_parity(ref, s_sys, asg, blocks=None):
    a = _sys_matrix(s_sys)
    s = int(asg.max()) + 1
    part = hp.partition_from_assignment(asg, s)
    p = hp.Preconditioner.block_jacobi(a, part)
    dims, f32, _, piv_ref, pert_ref = ref.factors(s_sys.row_ptr, s_sys.col, s_sys.val, s, asg)
    offs = np.concatenate([[0], np.cumsum(dims * dims)])
    worst = 0.0
    mism = 0
    sel = range(s) if blocks is None else blocks
    for b in sel:
        d = int(dims[b])
        F, piv = p.block_factors(b)
        Fr = f32[offs[b]:offs[b + 1]].reshape(d, d).astype(np.float64)
        o = int(part.block_starts[b])
        if not np.array_equal(piv, piv_ref[o:o + d]):
            mism += 1
            continue
        err = np.linalg.norm(F.astype(np.float64) - Fr) / np.linalg.norm(Fr)
        worst = max(worst, err)
    st = p.stats()
    assert [x["perturbation_count"] for x in st] == list(pert_ref)
    return worst, mism


@pytest.mark.parametrize("config", [0, 1, 4])
def test_block_factors_match_reference(ref, config):
    s = generate(config)
    asg, _, _, _ = ref.partition(s.row_ptr, s.col, s.val, s.num_blocks)
    worst, mism = _factor_parity(ref, s, asg)
    assert mism == 0, f"{mism} blocks with a different pivot sequence"
    assert worst <= 1e-5, worst


@pytest.mark.parametrize("config", [0, 1])
def test_lu_pair_and_warp_kernels_bit_identical(config, monkeypatch):
    """k_block_lu_pair (two warps per block, default) and k_block_lu_warp
    (HPBJ_LU_WARP=1) make the same pivots and the same FMA sequence per
    element: factors and pivot rows bit-identical."""
    s = generate(config)
    a = _sys_matrix(s)
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("HPBJ_LU_WARP", flag)
        p = hp.Preconditioner.block_jacobi(a, part)
        blocks = range(0, s.num_blocks, max(1, s.num_blocks // 40))
        out.append([p.block_factors(b) for b in blocks])
    for (f0, p0), (f1, p1) in zip(*out):
        assert np.array_equal(p0, p1)
        assert np.array_equal(f0.view(np.uint32), f1.view(np.uint32))


@pytest.mark.parametrize("config", [2, 3])
def test_lu_left_looking_bit_identical_to_blocked(config, monkeypatch):
    """k_block_lu_ll (left-looking, L in shared memory; default for
    96 < d <= 288) and k_block_lu_blk (right-looking, L2 scratch tile;
    HPBJ_LU_LL=0) apply the same fmaf chain per element in the same order and
    the same pivot rule: factors and pivot rows bit-identical, incl. the
    largest blocks (d > 256: the 512-thread instance)."""
    s = generate(config)
    a = _sys_matrix(s)
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    dims = np.diff(part.block_starts)
    blocks = sorted(set(range(0, s.num_blocks, max(1, s.num_blocks // 150))) |
                    set(np.argsort(dims)[-20:].tolist()) | set(np.argsort(dims)[:5].tolist()))
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("HPBJ_LU_LL", flag)
        p = hp.Preconditioner.block_jacobi(a, part)
        out.append(([p.block_factors(b) for b in blocks], [x["perturbation_count"] for x in p.stats(False)]))
    (f0, pc0), (f1, pc1) = out
    assert pc0 == pc1
    for b, (F0, P0), (F1, P1) in zip(blocks, f0, f1):
        assert np.array_equal(P0, P1), b
        assert np.array_equal(F0.view(np.uint32), F1.view(np.uint32)), (b, int(dims[b]))


@pytest.mark.slow
@pytest.mark.parametrize("config", [2, 3])
def test_block_factors_all_blocks_large_configs(ref, config):
    """Every block of configs 2 (7,813 blocks, d <= 141) and 3 (16,000
    blocks, d up to 282: k_block_lu_blk<256,1> and, for d > 256,
    k_block_lu_blk<256,2>) against gp_lu (lu.cpp:134-225) cast to FP32: pivot
    sequences equal, normwise factor error <= 1e-5, perturbation counts equal.
    The partition is our host partitioner's, bit-identical to the reference's
    (tests/test_partition.py, goldens)."""
    s = generate(config)
    part = hp.partition_graph(_sys_matrix(s), s.num_blocks, 0.1)
    dims = np.diff(part.block_starts)
    if config == 3:
        assert dims.max() > 256  # the two-tile-row blocked kernel is exercised
    worst, mism = _factor_parity(ref, s, part.assignment)
    assert mism == 0, f"{mism} blocks with a different pivot sequence"
    assert worst <= 1e-5, worst


def test_lu_known_answers(ref):
    # test_lu_kernels.cpp:78-93 tridiagonal, 120-141 pivoting/ties, 95-102 tiny pivot
    a = fx.tridiag(3, -1.0, 2.0, -1.0)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 0, 0], 1))
    F, piv = p.block_factors(0)
    assert list(piv) == [0, 1, 2]
    # reference values are FP64 (then cast); our factors are born FP32: 1-ulp tolerance
    expect = {(0, 0): 2.0, (1, 1): 1.5, (2, 2): 4.0 / 3.0, (1, 0): -0.5, (2, 1): -2.0 / 3.0}
    for (i, j), v in expect.items():
        assert abs(float(F[i, j]) - v) <= 2.0 ** -23 * abs(v), (i, j, F[i, j], v)

    a = hp.SparseMatrix.from_triplets([0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, -3.0, 1.0], 2)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 0], 1), hp.BlockJacobiOptions(0.0))
    assert list(p.block_factors(0)[1]) == [1, 0]

    a = hp.SparseMatrix.from_triplets([0, 1, 0, 1], [0, 0, 1, 1], [2.0, -2.0, 1.0, 5.0], 2)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 0], 1))
    assert list(p.block_factors(0)[1]) == [0, 1]

    a = fx.diag_csr([1e-20, 1.0])
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 0], 1))
    assert p.stats()[0]["perturbation_count"] == 1
    F, _ = p.block_factors(0)
    assert F[0, 0] == np.float32(1e-10)


def test_singular_block_only_with_zero_eps():
    # test_preconditioners.cpp:196-211, test_lu_kernels.cpp:104-118
    a = hp.SparseMatrix.from_triplets([0, 0, 1, 1, 2, 3], [0, 1, 0, 1, 2, 3], [1.0, 1.0, 1.0, 1.0, 3.0, 4.0], 4)
    part = hp.partition_from_assignment([0, 0, 1, 1], 2)
    with pytest.raises(hp.SingularBlockError) as ei:
        hp.Preconditioner.block_jacobi(a, part, hp.BlockJacobiOptions(eps_pivot=0.0))
    assert ei.value.column() == 1
    p = hp.Preconditioner.block_jacobi(a, part)
    st = p.stats()
    assert st[0]["perturbation_count"] == 1 and st[1]["perturbation_count"] == 0

    a = hp.SparseMatrix.from_triplets([0, 1], [0, 0], [1.0, 2.0], 2)  # column 1 structurally empty
    with pytest.raises(hp.SingularBlockError) as ei:
        hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 0], 1), hp.BlockJacobiOptions(0.0))
    assert ei.value.column() == 1 and "column 1" in str(ei.value)


# ------------------------------------------------------------ apply (K4)
def test_apply_known_answers():
    # test_preconditioners.cpp:83-91, 99-115
    d = [2.0, 5.0, 0.25, -4.0]
    p = hp.Preconditioner.block_jacobi(fx.diag_csr(d), hp.partition_from_assignment([0, 0, 1, 1], 2))
    z = p.apply([1.0, 2.0, 3.0, 4.0])
    assert np.array_equal(z, np.float32(np.array([1.0, 2.0, 3.0, 4.0]) / np.array(d)).astype(np.float64))
    a = hp.SparseMatrix.from_triplets([0, 0, 1], [0, 1, 1], [2.0, 1.0, 4.0], 2)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0, 0], 1))
    assert np.array_equal(p.apply([5.0, 8.0]), [1.5, 2.0])


def test_apply_single_block_is_full_inverse():
    a = fx.random_well_conditioned(12, 3)  # test_preconditioners.cpp:54-63 (FP32 tolerance)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_from_assignment([0] * 12, 1))
    b = fx.random_vector(12, 8)
    z = p.apply(b)
    e = np.linalg.solve(fx.to_dense(a), b)
    assert np.linalg.norm(z - e) <= 1e-6 * np.linalg.norm(e)


def test_apply_hybrid_close_to_double():
    # test_preconditioners.cpp:176-194: FP32 apply within 1e-5 of FP64
    a = fx.laplacian_2d(10, 10)
    part = hp.partition_graph(a, 4, 0.1)
    p = hp.Preconditioner.block_jacobi(a, part)
    v = fx.random_vector(a.n, 31)
    zf = p.apply(v)
    M = np.zeros((a.n, a.n))
    D = fx.to_dense(a)
    for b in range(4):
        idx = np.where(part.assignment == b)[0]
        M[np.ix_(idx, idx)] = D[np.ix_(idx, idx)]
    zd = np.linalg.solve(M, v)
    assert np.linalg.norm(zd - zf) / np.linalg.norm(zd) <= 1e-5


@pytest.mark.parametrize("config", [0, 1, 3])
def test_apply_matches_reference(ref, config):
    s = generate(config)
    a = _sys_matrix(s)
    if config == 3:
        part = hp.partition_graph(a, s.num_blocks, 0.1)
        asg = part.assignment
    else:
        asg, _, _, _ = ref.partition(s.row_ptr, s.col, s.val, s.num_blocks)
        part = hp.partition_from_assignment(asg, s.num_blocks)
    p = hp.Preconditioner.block_jacobi(a, part)
    v = np.random.default_rng(7).uniform(-1, 1, s.n)
    z = p.apply(v)
    zr = ref.apply(s.row_ptr, s.col, s.val, s.num_blocks, asg, v, fp32=True)
    zd = ref.apply(s.row_ptr, s.col, s.val, s.num_blocks, asg, v, fp32=False)
    assert np.linalg.norm(z - zr) <= 2e-6 * np.linalg.norm(zr)
    assert np.linalg.norm(z - zd) <= 1e-5 * np.linalg.norm(zd)


@pytest.mark.parametrize("layout", ["0", "1"])
@pytest.mark.parametrize("config", [0, 2])
def test_apply_both_offpanel_layouts(ref, config, layout, monkeypatch):
    """Row-sorted runs (HPBJ_SPK_ROWS=0) and row quads (=1) are two storage
    layouts of the same factors: both match the reference FP32 apply, also
    across the merged last panel ((L U)^-1 tile) and blocks of 1-5 panels."""
    monkeypatch.setenv("HPBJ_SPK_ROWS", layout)
    s = generate(config)
    a = _sys_matrix(s)
    part = hp.partition_graph(a, s.num_blocks, 0.1)  # bit-identical to the reference's (test_partition.py)
    asg = part.assignment
    p = hp.Preconditioner.block_jacobi(a, part)
    v = np.random.default_rng(11).uniform(-1, 1, s.n)
    z = p.apply(v)
    zr = ref.apply(s.row_ptr, s.col, s.val, s.num_blocks, asg, v, fp32=True)
    assert np.linalg.norm(z - zr) <= 2e-6 * np.linalg.norm(zr)
    assert np.array_equal(z, p.apply(v))


@pytest.mark.parametrize("coef", [-0.6, -0.75])
def test_apply_ill_conditioned_tiles(ref, coef):
    """The apply multiplies by explicitly inverted 32x32 diagonal tiles
    (spk.cu). Blocks of 96 rows made of three unit upper-triangular 32x32
    tiles with every upper entry = coef (tile condition ~1e6 / ~1e8) plus weak
    random coupling: no pivoting, so our FP32 factors and the reference's FP32
    cast are the same numbers and only the substitution differs. Our result
    must be as accurate as the reference's apply<float> (sequential FP32
    substitution, lu.hpp:88-112) against the exact solve with those factors."""
    rng = np.random.default_rng(5)
    nb, d = 4, 96
    n = nb * d
    rows, cols, vals = [], [], []
    for b in range(nb):
        o = b * d
        for i in range(d):
            rows.append(o + i), cols.append(o + i), vals.append(1.0)
            for j in range(i + 1, d):
                if i // 32 == j // 32:
                    rows.append(o + i), cols.append(o + j), vals.append(coef)
                elif rng.random() < 0.1:
                    rows.append(o + i), cols.append(o + j), vals.append(float(rng.uniform(-0.05, 0.05)))
    a = hp.SparseMatrix.from_triplets(np.array(rows), np.array(cols), np.array(vals), n)
    asg = np.repeat(np.arange(nb), d)
    part = hp.partition_from_assignment(asg, nb)
    p = hp.Preconditioner.block_jacobi(a, part)
    U = fx.to_dense(a).astype(np.float32).astype(np.float64)  # the FP32 factors (L = I)
    tile = U[:32, :32]
    cond = np.linalg.cond(tile, 1)
    assert 1e5 <= cond <= 1e9, cond
    v = rng.uniform(-1, 1, n)
    v32 = v.astype(np.float32).astype(np.float64)  # both applies round v to FP32 on load
    exact = np.linalg.solve(U, v32)
    z = p.apply(v)
    zr = ref.apply(a.row_starts, a.col_indices, a.values, nb, asg, v, fp32=True)
    err = np.linalg.norm(z - exact) / np.linalg.norm(exact)
    err_ref = np.linalg.norm(zr - exact) / np.linalg.norm(exact)
    print(f"tile cond {cond:.2e}: ours {err:.2e}, reference apply<float> {err_ref:.2e}")
    assert err <= 4.0 * err_ref + 1e-7, (err, err_ref)


def test_apply_deterministic():
    a = fx.laplacian_2d(16, 16)
    p = hp.Preconditioner.block_jacobi(a, hp.partition_graph(a, 8, 0.1))
    v = fx.random_vector(a.n, 12)
    assert np.array_equal(p.apply(v), p.apply(v))


def test_dimension_mismatch_raises():
    p = hp.Preconditioner.block_jacobi(fx.diag_csr([2.0, 4.0, 1.0]), hp.partition_from_assignment([0, 1, 2], 3))
    with pytest.raises(ValueError):
        p.apply([1.0, 2.0])


# ---------------------------------------------------------------------------
# Preconditioner diagnostics: cond_estimate_block /
# block_error_bound on the device vs the reference's FP64 estimates.
@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["small", "large"])
def test_block_condition_estimates_match_reference(ref, shape):
    if shape == "small":  # dims <= 64: exact inverse 1-norm
        a, s = fx.random_dd(300, 5, 13), 6
    else:  # dims > 64: Hager estimator
        a, s = fx.laplacian_2d(24, 24), 4
    part = hp.partition_graph(a, s, 0.1)
    p = hp.Preconditioner.block_jacobi(a, part)
    st = p.stats()
    cond = np.array([x["cond_estimate"] for x in st])
    eb = np.array([x["error_bound"] for x in st])
    rc, reb, _ = ref.block_stats(a.row_starts, a.col_indices, a.values, s, part.assignment)
    # FP64 arithmetic on the FP32 factors vs the reference's FP64 factors
    assert np.allclose(cond, rc, rtol=1e-4), (cond, rc)
    assert np.allclose(eb, reb, rtol=2e-4)
    assert np.all(cond >= 1.0)


def test_left_looking_lu_regularises_and_reports_singular_like_reference(ref):
    """Blocks of 96 < d <= 288 (the left-looking kernel) with tiny and exactly
    zero pivots: Eq. 7 regularisation (lu.cpp:10-20) with the reference's
    perturbation records and factors, and with eps_pivot = 0 the reference's
    SingularBlockError (lu.cpp:190-195) naming the column."""
    rng = np.random.default_rng(11)
    d, nb = 140, 3
    rows, cols, vals = [], [], []
    for blk in range(nb):
        o = blk * d
        for i in range(d):
            js = rng.choice(d, 6, replace=False)
            for j in js:
                if j != i:
                    rows.append(o + i), cols.append(o + int(j)), vals.append(float(rng.uniform(-1, 1)))
            rows.append(o + i), cols.append(o + i), vals.append(8.0)
    r, c, v = np.array(rows), np.array(cols), np.array(vals)
    # block 1: column 7 keeps only its rows above the diagonal and a 1e-14
    # diagonal; block 2: column 11 structurally empty (no update reaches it:
    # a zero pivot)
    o1, o2 = d, 2 * d
    v[(r == o1 + 7) & (c == o1 + 7)] = 1e-14
    keep = ~((r >= o1 + 7) & (r < o1 + d) & (c == o1 + 7) & (r != o1 + 7))
    keep &= ~((c == o2 + 11) & (r >= o2) & (r < o2 + d))
    r, c, v = r[keep], c[keep], v[keep]
    a = hp.SparseMatrix.from_triplets(r, c, v, nb * d)
    asg = np.repeat(np.arange(nb), d)
    part = hp.partition_from_assignment(asg, nb)
    p = hp.Preconditioner.block_jacobi(a, part)
    dims, f32, _, piv_ref, pert_ref = ref.factors(a.row_starts, a.col_indices, a.values, nb, asg)
    st = p.stats(False)
    assert [x["perturbation_count"] for x in st] == list(pert_ref)
    assert sum(pert_ref) >= 2
    offs = np.concatenate([[0], np.cumsum(dims * dims)])
    for b in range(nb):
        F, piv = p.block_factors(b)
        Fr = f32[offs[b]:offs[b + 1]].reshape(d, d).astype(np.float64)
        assert np.array_equal(piv, piv_ref[b * d:(b + 1) * d]), b
        assert np.linalg.norm(F.astype(np.float64) - Fr) <= 1e-5 * np.linalg.norm(Fr), b
    with pytest.raises(hp.SingularBlockError) as ei:
        hp.Preconditioner.block_jacobi(a, part, hp.BlockJacobiOptions(eps_pivot=0.0))
    assert ei.value.column() >= 0
    with pytest.raises(Exception):  # the reference refuses the same matrix
        ref.factors(a.row_starts, a.col_indices, a.values, nb, asg, eps=0.0)
