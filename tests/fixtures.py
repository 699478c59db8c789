"""Restatement of the reference test fixtures (proj/tests/fixtures.hpp) and
its SplitMix64 generator (proj/tests/oracles.hpp:205-226), so our tests use
the very matrices the reference's known-answer tests use."""
from __future__ import annotations

import numpy as np

from paper_2509_09139_b200 import SparseMatrix

MASK = (1 << 64) - 1


class Rng:
    """oracles.hpp:205-226"""

    def __init__(self, seed: int):
        self.s = seed & MASK

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform_pm1(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53 * 2.0 - 1.0

    def next_below(self, bound: int) -> int:
        return self.next_u64() % bound


def _from_triplets(t, n):
    if not t:
        return SparseMatrix(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    r, c, v = zip(*t)
    return SparseMatrix.from_triplets(r, c, v, n)


def identity_csr(n):
    return _from_triplets([(i, i, 1.0) for i in range(n)], n)


def diag_csr(d):
    return _from_triplets([(i, i, float(x)) for i, x in enumerate(d)], len(d))


def tridiag(n, lo, di, up):
    t = []
    for i in range(n):
        if i > 0:
            t.append((i, i - 1, lo))
        t.append((i, i, di))
        if i + 1 < n:
            t.append((i, i + 1, up))
    return _from_triplets(t, n)


def tridiag4():
    return tridiag(4, -1.0, 2.0, -1.0)


def laplacian_2d(nx, ny):
    t = []
    for iy in range(ny):
        for ix in range(nx):
            c = iy * nx + ix
            t.append((c, c, 4.0))
            if ix > 0:
                t.append((c, c - 1, -1.0))
            if ix + 1 < nx:
                t.append((c, c + 1, -1.0))
            if iy > 0:
                t.append((c, c - nx, -1.0))
            if iy + 1 < ny:
                t.append((c, c + nx, -1.0))
    return _from_triplets(t, nx * ny)


def convection_diffusion_2d(nx, ny, vx, vy):
    t = []
    for iy in range(ny):
        for ix in range(nx):
            c = iy * nx + ix
            t.append((c, c, 4.0 + vx + vy))
            if ix > 0:
                t.append((c, c - 1, -1.0 - vx))
            if ix + 1 < nx:
                t.append((c, c + 1, -1.0))
            if iy > 0:
                t.append((c, c - nx, -1.0 - vy))
            if iy + 1 < ny:
                t.append((c, c + nx, -1.0))
    return _from_triplets(t, nx * ny)


def random_dd(n, extra_per_row, seed):
    rng = Rng(seed)
    t = []
    row_abs = [0.0] * n
    for i in range(n):
        for _ in range(extra_per_row):
            j = rng.next_below(n)
            if j == i:
                continue
            v = rng.uniform_pm1()
            t.append((i, j, v))
            row_abs[i] += abs(v)
    for i in range(n):
        t.append((i, i, row_abs[i] + 1.0 + 0.5 * abs(rng.uniform_pm1())))
    return _from_triplets(t, n)


def random_dense_pattern(n, seed):
    rng = Rng(seed)
    return _from_triplets([(i, j, rng.uniform_pm1()) for i in range(n) for j in range(n)], n)


def random_well_conditioned(n, seed):
    rng = Rng(seed)
    t = []
    for i in range(n):
        for j in range(n):
            v = rng.uniform_pm1()
            if i == j:
                v += float(n)
            t.append((i, j, v))
    return _from_triplets(t, n)


def ones(n):
    return np.ones(n)


def random_vector(n, seed):
    rng = Rng(seed)
    return np.array([rng.uniform_pm1() for _ in range(n)])


def to_dense(a: SparseMatrix) -> np.ndarray:
    d = np.zeros((a.n, a.n))
    for i in range(a.n):
        for k in range(a.row_starts[i], a.row_starts[i + 1]):
            d[i, a.col_indices[k]] += a.values[k]
    return d
