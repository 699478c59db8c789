"""Host partitioner (graph_from_matrix + partition_graph + partition_from_
assignment, in libhpbj.so) vs the reference library and its known answers
(test_graph_partition.cpp). CPU only: no kernel is launched."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2509_09139_b200 as hp
from paper_2509_09139_b200.workloads import generate
from tests import fixtures as fx

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def path_graph(n, w=1.0):
    st = [0]
    nb, ws = [], []
    for i in range(n):
        for j in (i - 1, i + 1):
            if 0 <= j < n:
                nb.append(j)
                ws.append(w)
        st.append(len(nb))
    return hp.WeightedGraph(n, np.array(st, np.int64), np.array(nb, np.int64), np.array(ws))


def edge_weight(g, u, v):
    for k in range(g.start[u], g.start[u + 1]):
        if g.neighbor[k] == v:
            return g.weight[k]
    return 0.0


def cut_weight(g, part):
    c = 0.0
    for u in range(g.num_nodes):
        for k in range(g.start[u], g.start[u + 1]):
            v = g.neighbor[k]
            if u < v and part.assignment[u] != part.assignment[v]:
                c += g.weight[k]
    return c


# ---------------------------------------------------------------- graph
def test_weight_averages_both_directions():
    a = hp.SparseMatrix.from_triplets([0, 1, 0, 1], [0, 1, 1, 0], [1.0, 1.0, -4.0, 2.0], 2)
    g = hp.graph_from_matrix(a)  # graph.cpp:17-51; test_graph_partition.cpp:55-60
    assert edge_weight(g, 0, 1) == 3.0 and edge_weight(g, 1, 0) == 3.0


def test_one_sided_entry_makes_an_edge():
    a = hp.SparseMatrix.from_triplets([0, 1, 0], [0, 1, 1], [1.0, 1.0, 5.0], 2)
    g = hp.graph_from_matrix(a)  # test_graph_partition.cpp:62-67
    assert edge_weight(g, 0, 1) == 2.5 and edge_weight(g, 1, 0) == 2.5


def test_tridiag_gives_path_graph():
    g = hp.graph_from_matrix(fx.tridiag4())
    assert g.num_nodes == 4 and g.num_edges() == 3
    assert edge_weight(g, 0, 1) == 1.0 and edge_weight(g, 2, 3) == 1.0 and edge_weight(g, 0, 2) == 0.0


def test_zero_valued_pairs_are_dropped():
    a = hp.SparseMatrix.from_triplets([0, 0, 1, 1, 2, 2], [0, 1, 0, 1, 2, 1], [1.0, 0.0, 0.0, 1.0, 1.0, -1.0], 3)
    g = hp.graph_from_matrix(a)  # graph.cpp:41 (w <= 0 skipped)
    assert edge_weight(g, 0, 1) == 0.0 and g.degree(0) == 0
    assert edge_weight(g, 1, 2) == 0.5


@pytest.mark.parametrize("seed", [4, 9, 16])
def test_graph_matches_reference(ref, seed):
    a = fx.random_dd(30, 4, seed)  # unsymmetric pattern -> general (transpose) path
    g = hp.graph_from_matrix(a)
    st, nb, w = ref.graph(a.row_starts, a.col_indices, a.values)
    assert np.array_equal(g.start, st) and np.array_equal(g.neighbor, nb) and np.array_equal(g.weight, w)


@pytest.mark.parametrize("config", [0, 4])
def test_graph_symmetric_fast_path_matches_reference(ref, config):
    s = generate(config)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    g = hp.graph_from_matrix(a)
    st, nb, w = ref.graph(s.row_ptr, s.col, s.val)
    assert np.array_equal(g.start, st) and np.array_equal(g.neighbor, nb)
    assert np.array_equal(g.weight.view(np.uint64), w.view(np.uint64))  # bit-exact


def test_graph_rejects_non_square_or_bad_csr():
    with pytest.raises(ValueError):
        hp.graph_from_matrix(hp.SparseMatrix(2, np.array([0, 1, 2]), np.array([0, 2]), np.array([1.0, 1.0])))
    with pytest.raises(ValueError):  # columns not strictly increasing
        hp.graph_from_matrix(hp.SparseMatrix(2, np.array([0, 2, 2]), np.array([1, 0]), np.array([1.0, 1.0])))


# ---------------------------------------------------------------- partition
def test_single_block_is_degenerate():
    p = hp.partition_graph(path_graph(5), 1, 0.1)
    assert list(p.assignment) == [0] * 5 and list(p.perm) == list(range(5))


def test_four_node_path_splits_in_the_middle():
    g = hp.graph_from_matrix(fx.tridiag4())  # test_graph_partition.cpp:116-123
    p = hp.partition_graph(g, 2, 0.1)
    a = p.assignment
    assert a[0] == a[1] and a[2] == a[3] and a[0] != a[2]
    assert cut_weight(g, p) == 1.0


def test_six_node_path_matches_brute_force():
    g = path_graph(6)
    p = hp.partition_graph(g, 2, 0.1)
    a = p.assignment
    assert list(a) == [a[0]] * 3 + [a[3]] * 3 and a[0] != a[3] and cut_weight(g, p) == 1.0


def test_isolated_nodes_go_to_smallest_blocks():
    p = hp.partition_graph(hp.graph_from_matrix(fx.diag_csr([1, 2, 3, 4, 5, 6])), 3, 0.0)
    assert [p.block_size(b) for b in range(3)] == [2, 2, 2]


def test_s_equals_n_with_zero_tolerance():
    p = hp.partition_graph(path_graph(5), 5, 0.0)
    assert [p.block_size(b) for b in range(5)] == [1] * 5


def test_rejects_bad_arguments():
    g = path_graph(4)
    for s, tol in [(5, 0.1), (0, 0.1), (2, -0.5)]:
        with pytest.raises(ValueError):
            hp.partition_graph(g, s, tol)


@pytest.mark.parametrize("seed", [3, 7])
@pytest.mark.parametrize("s", [2, 3, 5, 8])
def test_partition_matches_reference_random(ref, seed, s):
    a = fx.random_dd(40, 3, seed)  # test_graph_partition.cpp:137-163 cases
    p = hp.partition_graph(a, s, 0.1)
    asg, perm, bst, _ = ref.partition(a.row_starts, a.col_indices, a.values, s)
    assert np.array_equal(p.assignment, asg) and np.array_equal(p.perm, perm)
    assert np.array_equal(p.block_starts, bst)
    q = hp.partition_graph(hp.graph_from_matrix(a), s, 0.1)  # explicit-graph entry point
    assert np.array_equal(q.assignment, asg)


@pytest.mark.parametrize("n,s", [(4, 2), (6, 2), (9, 2), (9, 4), (30, 7)])
def test_partition_of_explicit_graph_matches_reference(ref, n, s):
    g = path_graph(n, 0.5)
    a = hp.partition_graph(g, s, 0.1)
    r = ref.partition_graph(g.start, g.neighbor, g.weight, s, 0.1)
    assert np.array_equal(a.assignment, r)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_explicit_graph_with_nonpositive_weights_matches_reference(ref, seed):
    """A hand-built WeightedGraph may carry w <= 0 edges (graph_from_matrix never
    emits them): partition_graph still grows over and refines with every edge
    (partition.cpp:96-97, :122-125), including touched-twice blocks when
    conn returns to 0.0."""
    rng = np.random.default_rng(seed)
    n = 60
    pairs = {}
    for i in range(n):
        for j in rng.choice(n, 4, replace=False):
            if i != j:
                pairs[(min(i, j), max(i, j))] = float(rng.choice([-1.0, 0.0, 0.5, 1.0, 2.0]))
    adj = [[] for _ in range(n)]
    for (i, j), w in pairs.items():
        adj[i].append((j, w))
        adj[j].append((i, w))
    st, nb, ws = [0], [], []
    for i in range(n):
        for j, w in sorted(adj[i]):
            nb.append(j)
            ws.append(w)
        st.append(len(nb))
    g = hp.WeightedGraph(n, np.array(st, np.int64), np.array(nb, np.int64), np.array(ws))
    for s in (2, 5, 9):
        a = hp.partition_graph(g, s, 0.1)
        r = ref.partition_graph(g.start, g.neighbor, g.weight, s, 0.1)
        assert np.array_equal(a.assignment, r)


def test_laplacian_and_mesh_fixtures_match_reference(ref):
    for a, s in [(fx.laplacian_2d(32, 32), 16), (fx.laplacian_2d(16, 16), 8), (fx.laplacian_2d(8, 8), 4),
                 (fx.convection_diffusion_2d(10, 10, 2.0, 1.0), 4), (fx.random_dd(80, 4, 55), 4)]:
        p = hp.partition_graph(a, s, 0.1)
        asg, _, _, _ = ref.partition(a.row_starts, a.col_indices, a.values, s)
        assert np.array_equal(p.assignment, asg)


def _mesh3d_long_range(k, extra, seed):
    """k^3 7-point mesh plus `extra` random long-range couplings (config 3's shape, small)."""
    rng = np.random.default_rng(seed)
    n = k ** 3
    idx = np.arange(n).reshape(k, k, k)
    r = [idx.ravel()]
    c = [idx.ravel()]
    v = [np.full(n, 8.0)]
    for ax in range(3):
        a = np.take(idx, range(k - 1), axis=ax).ravel()
        b = np.take(idx, range(1, k), axis=ax).ravel()
        w = rng.uniform(0.5, 1.5, a.size)
        r += [a, b]
        c += [b, a]
        v += [-w, -w]
    a, b = rng.integers(0, n, extra), rng.integers(0, n, extra)
    keep = a != b
    w = rng.uniform(0.01, 0.2, int(keep.sum()))
    r += [a[keep], b[keep]]
    c += [b[keep], a[keep]]
    v += [-w, -w]
    r, c, v = np.concatenate(r), np.concatenate(c), np.concatenate(v)
    key = r * n + c
    _, first = np.unique(key, return_index=True)  # drop duplicate long-range pairs
    return hp.SparseMatrix.from_triplets(r[first], c[first], v[first], n)


@pytest.mark.parametrize("T", [2, 3, 7, 16])
def test_parallel_refinement_sweep_matches_reference(ref, monkeypatch, T):
    """The exact parallel refinement sweep (T node ranges, speculative phase +
    in-order resolution, partition.cpp host code) against the reference on
    graphs where block sizes hit the cap (tolerance 0 and 0.1), uniform-weight
    ties (Laplacian), random couplings across ranges and w <= 0 edges."""
    monkeypatch.setenv("HPBJ_REFINE_T", str(T))
    cases = [(fx.laplacian_2d(40, 40), 25, 0.0), (fx.laplacian_2d(40, 40), 25, 0.1),
             (fx.random_dd(400, 3, 9), 20, 0.1), (_mesh3d_long_range(14, 30, 4), 40, 0.0),
             (_mesh3d_long_range(14, 30, 4), 11, 0.1)]
    for a, s, tol in cases:
        p = hp.partition_graph(a, s, tol)
        asg, _, _, _ = ref.partition(a.row_starts, a.col_indices, a.values, s, tol)
        assert np.array_equal(p.assignment, asg), (a.n, s, tol)
    test_explicit_graph_with_nonpositive_weights_matches_reference(ref, 2)


def test_unsymmetric_pattern_with_hub_matches_reference(ref):
    # one-sided couplings (structurally unsymmetric) + a dense hub row
    rng = np.random.default_rng(5)
    n = 300
    t = [(i, i, 4.0) for i in range(n)]
    t += [(i, (i + 1) % n, -1.0) for i in range(n)]
    t += [(0, j, -0.01) for j in rng.choice(np.arange(1, n), 120, replace=False)]
    t += [(int(i), int(j), float(v)) for i, j, v in zip(rng.integers(0, n, 200), rng.integers(0, n, 200),
                                                        rng.uniform(-1, 1, 200)) if i != j]
    r, c, v = zip(*t)
    a = hp.SparseMatrix.from_triplets(r, c, v, n)
    for s in (3, 10, 37):
        p = hp.partition_graph(a, s, 0.1)
        asg, perm, _, _ = ref.partition(a.row_starts, a.col_indices, a.values, s)
        assert np.array_equal(p.assignment, asg) and np.array_equal(p.perm, perm)


@pytest.mark.parametrize("config", [0, 1, 4, 2, 3])
def test_config_partition_bit_identical_to_reference(config):
    """Pinned by tests/golden/config<k>.json (reference partition run once:
    config 3 took ~1000 s in the reference, O(n*s))."""
    g = json.load(open(os.path.join(GOLD, f"config{config}.json")))
    s = generate(config)
    assert s.digest() == g["input_sha256"]
    p = hp.partition_graph(hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val), s.num_blocks, 0.1)
    assert sha(p.assignment) == g["partition"]["assignment_sha256"]
    assert sha(p.perm) == g["partition"]["perm_sha256"]
    assert sha(p.block_starts) == g["partition"]["block_starts_sha256"]


def test_partition_deterministic():
    a = fx.random_dd(40, 3, 7)
    assert np.array_equal(hp.partition_graph(a, 5).assignment, hp.partition_graph(a, 5).assignment)


# ------------------------------------------------ partition_from_assignment
def test_stable_gather():
    p = hp.partition_from_assignment([1, 0, 1, 0], 2)  # test_graph_partition.cpp:212-216
    assert list(p.perm) == [2, 0, 3, 1] and list(p.block_starts) == [0, 2, 4]
    p = hp.partition_from_assignment([0, 0, 1, 1], 2)
    assert list(p.perm) == [0, 1, 2, 3]


def test_assignment_errors():
    with pytest.raises(IndexError):
        hp.partition_from_assignment([0, 0, 2, 1], 2)
    with pytest.raises(ValueError):
        hp.partition_from_assignment([0, 0, 0, 0], 2)
    with pytest.raises(ValueError):
        hp.partition_from_assignment([0, 0], 3)


def _with_zero_entries(a, seed):
    """Explicit off-diagonal zeros: some pairs zero on both sides (no edge,
    graph.cpp:41), some on one side only (an edge of half the other weight)."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(a.n), np.diff(a.row_starts))
    cols = np.asarray(a.col_indices)
    vals = np.array(a.values, dtype=np.float64)
    off = np.nonzero(rows < cols)[0]
    both = rng.choice(off, max(1, off.size // 20), replace=False)
    one = rng.choice(np.setdiff1d(off, both), max(1, off.size // 20), replace=False)
    pos = {(int(r), int(c)): k for k, (r, c) in enumerate(zip(rows, cols))}
    for k in both:
        vals[k] = 0.0
        vals[pos[(int(cols[k]), int(rows[k]))]] = -0.0
    vals[one] = 0.0
    return hp.SparseMatrix(a.n, np.asarray(a.row_starts), cols, vals)


@pytest.mark.parametrize("env", [{"HPBJ_GROW_ELL": "1"}, {"HPBJ_GROW_ELL": "1", "HPBJ_GROW_NOPIPE": "1"},
                                 {"HPBJ_GROW_ELL": "0"}, {"HPBJ_GROW_ELL": "1", "HPBJ_GROW_PF": "0"}])
def test_region_growing_variants_match_reference(ref, monkeypatch, env):
    """Region growing over fixed-stride neighbour records — overlapped with the
    weight/adjacency build on the other cores when A has no explicit
    off-diagonal zero (pipelined), or after it — and over the CSR view,
    against the reference: meshes, long-range couplings, rows longer than a
    record (hubs), explicit zeros (both-sided: no edge; one-sided: an edge)
    and a structurally unsymmetric pattern (the pipelined grow is abandoned)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(3)
    n = 300
    t = [(i, i, 4.0) for i in range(n)] + [(i, (i + 1) % n, -1.0) for i in range(n)]
    t += [(0, j, -0.01) for j in rng.choice(np.arange(1, n), 120, replace=False)]
    r, c, v = zip(*t)
    unsym = hp.SparseMatrix.from_triplets(r, c, v, n)
    hub = fx.random_dd(500, 9, 4)
    # isolated nodes (diagonal-only rows) and two components
    lap = fx.laplacian_2d(12, 12)
    n2 = lap.n + 20
    rr = np.repeat(np.arange(lap.n), np.diff(lap.row_starts))
    r2 = np.concatenate([rr, np.arange(lap.n, n2)])
    c2 = np.concatenate([np.asarray(lap.col_indices), np.arange(lap.n, n2)])
    v2 = np.concatenate([np.asarray(lap.values), np.full(20, 3.0)])
    iso = hp.SparseMatrix.from_triplets(r2, c2, v2, n2)
    cases = [(fx.laplacian_2d(40, 40), 25, 0.1), (_mesh3d_long_range(14, 30, 4), 11, 0.1), (iso, 7, 0.1),
             (hub, 20, 0.1), (_with_zero_entries(fx.laplacian_2d(30, 30), 1), 16, 0.1),
             (_with_zero_entries(_mesh3d_long_range(10, 20, 2), 3), 9, 0.0), (unsym, 10, 0.1)]
    for a, s, tol in cases:
        p = hp.partition_graph(a, s, tol)
        asg, _, _, _ = ref.partition(a.row_starts, a.col_indices, a.values, s, tol)
        assert np.array_equal(p.assignment, asg), (a.n, s, tol)
