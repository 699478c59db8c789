"""Seeded synthetic systems for the five BASELINE.json configs.

Thin ctypes wrapper over ``lib/libhpbj_gen.so`` (csrc/gen/workloads.cpp).
The generator is deterministic (SplitMix64, the reference's test convention,
proj/tests/oracles.hpp:205-226); every array is copied into numpy.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
GEN_LIB = os.path.join(_HERE, "lib", "libhpbj_gen.so")


class _GenSystem(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.POINTER(ctypes.c_int64)),
        ("col", ctypes.POINTER(ctypes.c_int64)),
        ("val", ctypes.POINTER(ctypes.c_double)),
        ("b", ctypes.POINTER(ctypes.c_double)),
        ("x_true", ctypes.POINTER(ctypes.c_double)),
        ("block_size", ctypes.c_int64),
        ("num_blocks", ctypes.c_int64),
        ("restart_m", ctypes.c_int64),
        ("tol", ctypes.c_double),
        ("maxit", ctypes.c_int64),
        ("max_restarts", ctypes.c_int64),
    ]


@dataclass
class System:
    """One linear system A x = b plus the solver parameters of its config."""

    config: int
    step: int
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray  # int64[nnz]
    val: np.ndarray  # float64[nnz]
    b: np.ndarray  # float64[n]
    x_true: np.ndarray  # float64[n]
    block_size: int
    num_blocks: int
    restart_m: int
    tol: float
    maxit: int
    max_restarts: int

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.row_ptr, self.col, self.val, self.b):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


_lib = None


def _gen():
    global _lib
    if _lib is None:
        if not os.path.exists(GEN_LIB):
            raise RuntimeError(f"{GEN_LIB} missing: run __graft_entry__.build()")
        _lib = ctypes.CDLL(GEN_LIB)
        _lib.hpbj_gen_config.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_GenSystem)]
        _lib.hpbj_gen_config.restype = ctypes.c_int
        _lib.hpbj_gen_free.argtypes = [ctypes.POINTER(_GenSystem)]
    return _lib


def generate(config: int, step: int = 0) -> System:
    lib = _gen()
    s = _GenSystem()
    rc = lib.hpbj_gen_config(config, step, ctypes.byref(s))
    if rc != 0:
        raise ValueError(f"bad config/step {config}/{step}")
    try:
        n, nnz = s.n, s.nnz
        arr = np.ctypeslib.as_array
        return System(
            config=config,
            step=step,
            n=n,
            row_ptr=arr(s.row_ptr, (n + 1,)).copy(),
            col=arr(s.col, (nnz,)).copy(),
            val=arr(s.val, (nnz,)).copy(),
            b=arr(s.b, (n,)).copy(),
            x_true=arr(s.x_true, (n,)).copy(),
            block_size=s.block_size,
            num_blocks=s.num_blocks,
            restart_m=s.restart_m,
            tol=s.tol,
            maxit=s.maxit,
            max_restarts=s.max_restarts,
        )
    finally:
        lib.hpbj_gen_free(ctypes.byref(s))
