"""Matrix Market / CSR cache / partition-file I/O:
the reference's known answers (test_sparse_core.cpp:31-119,
test_graph_partition.cpp import/export) restated, plus bit-exact agreement
with the reference library's reader on generated files. CPU only."""
import os

import numpy as np
import pytest

import paper_2509_09139_b200 as hp
from tests import fixtures as fx


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def value_at(a, i, j):
    for k in range(a.row_starts[i], a.row_starts[i + 1]):
        if a.col_indices[k] == j:
            return a.values[k]
    return 0.0


def test_reads_general_coordinate(tmp_path):  # test_sparse_core.cpp:31-43
    a = hp.read_matrix_market(write(tmp_path, "g.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                                        "2 2 2\n1 1 3.0\n2 2 4.0\n"))
    assert a.n == 2 and a.nnz() == 2 and value_at(a, 0, 0) == 3.0 and value_at(a, 1, 1) == 4.0


def test_expands_symmetric(tmp_path):  # :45-54
    a = hp.read_matrix_market(write(tmp_path, "s.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
                                                        "% a comment\n2 2 1\n2 1 5.0\n"))
    assert value_at(a, 1, 0) == 5.0 and value_at(a, 0, 1) == 5.0


def test_sums_duplicates(tmp_path):  # :56-66
    a = hp.read_matrix_market(write(tmp_path, "d.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                                        "1 1 2\n1 1 1.0\n1 1 2.0\n"))
    assert a.nnz() == 1 and value_at(a, 0, 0) == 3.0


def test_reads_integer_field(tmp_path):  # :68-77
    a = hp.read_matrix_market(write(tmp_path, "i.mtx", "%%MatrixMarket matrix coordinate integer general\n"
                                                        "2 2 2\n1 2 7\n2 1 -3\n"))
    assert value_at(a, 0, 1) == 7.0 and value_at(a, 1, 0) == -3.0


@pytest.mark.parametrize("text,line", [
    ("%%MatrixMarket matrix coordinate pattern general\n", "line 1"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "line 3"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n", "line 1"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "line 4"),
    ("%%MatrixMarket matrix array real general\n", "line 1"),
    ("%%MatrixMarket matrix coordinate real general\n% only a comment\n", "missing size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", "malformed entry"),
])
def test_errors_name_the_line(tmp_path, text, line):  # :79-110
    with pytest.raises(RuntimeError) as e:
        hp.read_matrix_market(write(tmp_path, "bad.mtx", text))
    assert line in str(e.value)


def test_round_trip_is_exact(tmp_path):  # :112-119
    a = fx.random_dd(30, 4, 77)
    p = str(tmp_path / "rt.mtx")
    hp.write_matrix_market(p, a)
    b = hp.read_matrix_market(p)
    assert np.array_equal(a.row_starts, b.row_starts) and np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values.view(np.uint64), b.values.view(np.uint64))


def test_csr_cache_round_trip_and_rejects_garbage(tmp_path):
    a = fx.random_dd(50, 5, 3)
    p = str(tmp_path / "a.csr")
    hp.write_csr_cache(p, a)
    b = hp.read_csr_cache(p)
    assert np.array_equal(a.row_starts, b.row_starts) and np.array_equal(a.values, b.values)
    bad = write(tmp_path, "bad.csr", "not a cache")
    with pytest.raises(RuntimeError):
        hp.read_csr_cache(bad)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_reader_bit_identical_to_reference(ref, tmp_path, seed):
    """Random coordinate files (duplicates with different summation orders,
    symmetric expansion, comments, blank lines, integer field, extra tokens)
    read by both readers: identical CSR, bit for bit."""
    rng = np.random.default_rng(seed)
    n = 40
    symmetric = seed % 2 == 0
    integer = seed == 3
    ent = []
    for _ in range(150):
        i, j = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
        if symmetric and j > i:
            i, j = j, i
        v = int(rng.integers(-9, 10)) if integer else float(rng.standard_normal() * 10.0 ** int(rng.integers(-8, 8)))
        ent.append((i, j, v))
    lines = [f"%%MatrixMarket matrix coordinate {'integer' if integer else 'real'} "
             f"{'symmetric' if symmetric else 'general'}", "% generated", "", f"{n} {n} {len(ent)}"]
    for k, (i, j, v) in enumerate(ent):
        if k % 37 == 5:
            lines.append("% interleaved comment")
        if k % 41 == 7:
            lines.append("   ")
        val = str(v) if integer else repr(v)
        lines.append(f"{i} {j} {val}" + (" trailing" if k % 29 == 3 else ""))
    p = write(tmp_path, "r.mtx", "\n".join(lines) + "\n")
    a = hp.read_matrix_market(p)
    nr, nc, rp, ci, v = ref.mm_read(p)
    assert (nr, nc) == (n, n)
    assert np.array_equal(a.row_starts, rp) and np.array_equal(a.col_indices, ci)
    assert np.array_equal(a.values.view(np.uint64), v.view(np.uint64))


def test_writer_matches_reference_writer(ref, tmp_path):
    a = fx.random_dd(25, 4, 11)
    ours, theirs = str(tmp_path / "o.mtx"), str(tmp_path / "t.mtx")
    hp.write_matrix_market(ours, a)
    ref.mm_write(theirs, a.row_starts, a.col_indices, a.values)
    assert open(ours).read() == open(theirs).read()


def test_partition_file_round_trip_and_errors(tmp_path):
    a = fx.random_dd(40, 3, 7)
    p = hp.partition_graph(a, 5, 0.1)
    path = str(tmp_path / "p.txt")
    hp.export_partition(path, p)
    q = hp.import_partition(path, a.n, 5)
    assert np.array_equal(p.assignment, q.assignment) and np.array_equal(p.perm, q.perm)
    with pytest.raises(IndexError, match="line 2"):
        hp.import_partition(write(tmp_path, "oob.txt", "0\n9\n"), 2, 2)
    with pytest.raises(RuntimeError, match="line 1"):
        hp.import_partition(write(tmp_path, "mal.txt", "x\n"), 1, 1)
    with pytest.raises(RuntimeError, match="expected 3 lines"):
        hp.import_partition(write(tmp_path, "short.txt", "0\n\n1\n"), 3, 2)


def test_block_nnz_and_cut_weight():
    a = fx.laplacian_2d(8, 8)
    p = hp.partition_graph(a, 4, 0.1)
    bn, imb = hp.measure_block_nnz(p, a)
    assert bn.sum() <= a.nnz() and imb >= 1.0
    g = hp.graph_from_matrix(a)
    assert hp.cut_weight(g, p) > 0.0
