"""ctypes declarations of include/hpbj.h (libhpbj.so).

The library is loaded from this package's ``lib/`` directory only; a missing
library is a hard error (there is no CPU fallback for any numerical step).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libhpbj.so")

HPBJ_OK = 0
HPBJ_EINVAL = 1
HPBJ_ELOGIC = 2
HPBJ_ESINGULAR = 3
HPBJ_ECUDA = 4
HPBJ_ENOMEM = 5
HPBJ_ERANGE = 6
HPBJ_ENODEV = 7
HPBJ_EIO = 8
HPBJ_ERUNTIME = 9

HPBJ_K_APPLY = 0
HPBJ_K_SPMV = 1
HPBJ_K_MGS = 2
HPBJ_K_CYCLE = 3
HPBJ_K_COUNT = 4

i64 = ctypes.c_int64
f64 = ctypes.c_double
i64p = ctypes.POINTER(ctypes.c_int64)
f64p = ctypes.POINTER(ctypes.c_double)
f32p = ctypes.POINTER(ctypes.c_float)
vp = ctypes.c_void_p


class SetupInfo(ctypes.Structure):
    _fields_ = [
        ("num_blocks", i64),
        ("dim_min", i64),
        ("dim_max", i64),
        ("perturbations", i64),
        ("singular_block", i64),
        ("singular_column", i64),
        ("factor_bytes", i64),
        ("ms_permute", f64),
        ("ms_factor", f64),
        ("ms_lu", f64),
        ("ms_spk", f64),
    ]


class GmresOpts(ctypes.Structure):
    _fields_ = [
        ("restart_m", i64),
        ("tol", f64),
        ("max_restarts", i64),
        ("absolute_tol", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("breakdown_tol_factor", f64),
        ("floor_roundoff", f64),
    ]


class Report(ctypes.Structure):
    _fields_ = [
        ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("ls_rank_deficient", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("total_iterations", i64),
        ("restarts", i64),
        ("history_len", i64),
        ("cycles", i64),
        ("final_residual", f64),
        ("ms_solve", f64),
    ]


class HistoryPoint(ctypes.Structure):
    _fields_ = [("cycle", i64), ("iteration", i64), ("relative_residual", f64)]


class KernelStat(ctypes.Structure):
    _fields_ = [("launches", i64), ("total_ms", f64), ("bytes_per_launch", f64), ("steps", i64),
                ("total_bytes", f64)]


# name -> (restype, argtypes); exactly the symbols include/hpbj.h declares
SIGNATURES = {
    "hpbj_create": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_int]),
    "hpbj_destroy": (None, [vp]),
    "hpbj_last_error": (ctypes.c_char_p, [vp]),
    "hpbj_kernel_launches": (i64, [vp]),
    "hpbj_set_profiling": (ctypes.c_int, [vp, ctypes.c_int]),
    "hpbj_get_kernel_stats": (ctypes.c_int, [vp, ctypes.POINTER(KernelStat)]),
    "hpbj_set_fused": (ctypes.c_int, [vp, ctypes.c_int]),
    "hpbj_set_graph": (ctypes.c_int, [vp, ctypes.c_int]),
    "hpbj_get_block_diagnostics": (ctypes.c_int, [vp, ctypes.POINTER(f64), ctypes.POINTER(f64)]),
    "hpbj_mm_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                    ctypes.POINTER(ctypes.POINTER(i64)), ctypes.POINTER(ctypes.POINTER(i64)),
                                    ctypes.POINTER(ctypes.POINTER(f64))]),
    "hpbj_mm_write": (ctypes.c_int, [ctypes.c_char_p, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                     ctypes.POINTER(f64)]),
    "hpbj_csr_cache_write": (ctypes.c_int, [ctypes.c_char_p, i64, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                            ctypes.POINTER(f64)]),
    "hpbj_csr_cache_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(i64),
                                           ctypes.POINTER(ctypes.POINTER(i64)), ctypes.POINTER(ctypes.POINTER(i64)),
                                           ctypes.POINTER(ctypes.POINTER(f64))]),
    "hpbj_free": (None, [vp]),
    "hpbj_graph_from_matrix": (ctypes.c_int, [i64, i64p, i64p, f64p, i64p, i64p, f64p, i64]),
    "hpbj_partition_graph": (ctypes.c_int, [i64, i64p, i64p, f64p, i64, f64, i64p, i64p, i64p]),
    "hpbj_partition_adjacency": (ctypes.c_int, [i64, i64p, i64p, f64p, i64, f64, i64p, i64p, i64p]),
    "hpbj_partition_from_assignment": (ctypes.c_int, [i64, i64p, i64, i64p, i64p]),
    "hpbj_set_matrix": (ctypes.c_int, [vp, i64, i64p, i64p, f64p]),
    "hpbj_update_values": (ctypes.c_int, [vp, f64p]),
    "hpbj_spmv": (ctypes.c_int, [vp, f64p, f64p]),
    "hpbj_bj_setup": (ctypes.c_int, [vp, i64, i64p, i64p, f64, ctypes.POINTER(SetupInfo)]),
    "hpbj_bj_refactor": (ctypes.c_int, [vp, ctypes.POINTER(SetupInfo)]),
    "hpbj_bj_apply": (ctypes.c_int, [vp, f64p, f64p]),
    "hpbj_bj_set_neumann_order": (ctypes.c_int, [vp, ctypes.c_int]),
    "hpbj_ilu0_setup": (ctypes.c_int, [vp, ctypes.c_void_p]),
    "hpbj_identity_setup": (ctypes.c_int, [vp]),
    "hpbj_precond_apply": (ctypes.c_int, [vp, f64p, f64p]),
    "hpbj_get_ilu0_values": (ctypes.c_int, [vp, f64p]),
    "hpbj_bj_apply_neumann": (ctypes.c_int, [vp, f64p, f64p, ctypes.c_int]),
    "hpbj_get_block_factors": (ctypes.c_int, [vp, i64, i64p, f32p, i64p]),
    "hpbj_get_block_stats": (ctypes.c_int, [vp, i64p, i64p]),
    "hpbj_gmres_default_opts": (None, [ctypes.POINTER(GmresOpts)]),
    "hpbj_gmres": (ctypes.c_int, [vp, f64p, f64p, ctypes.POINTER(GmresOpts), ctypes.POINTER(Report),
                                  ctypes.POINTER(HistoryPoint), i64, f64p, i64]),
    "hpbj_gmres_device": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(GmresOpts), ctypes.POINTER(Report),
                                         ctypes.POINTER(HistoryPoint), i64, f64p, i64]),
}

_lib = None


def load():
    """Load libhpbj.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                               " (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
