"""The C ABI library loads and exports exactly what include/hpbj.h declares;
CPU-only behaviour (no device -> HPBJ_ENODEV, no silent CPU fallback)."""
import ctypes
import os
import re

import pytest

from paper_2509_09139_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hpbj.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(hpbj_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "hpbj_gmres" in names and "hpbj_bj_setup" in names and "hpbj_partition_graph" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_abi.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared_functions()) == set(_abi.SIGNATURES)


def test_no_device_is_a_hard_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _abi.load()
    h = ctypes.c_void_p()
    assert lib.hpbj_create(ctypes.byref(h), 0) == _abi.HPBJ_ENODEV
    assert b"no CPU fallback" in lib.hpbj_last_error(None)


def test_default_options_match_gmres_config():
    # GmresConfig defaults (gmres.hpp:89-97); floor roundoff 2^-24 (FP32 preconditioner)
    o = _abi.GmresOpts()
    _abi.load().hpbj_gmres_default_opts(ctypes.byref(o))
    assert (o.restart_m, o.tol, o.max_restarts, o.absolute_tol) == (50, 1e-8, 40, 0)
    assert o.breakdown_tol_factor == 1e2 and o.floor_roundoff == 2.0 ** -24


def test_null_context_is_rejected():
    lib = _abi.load()
    assert lib.hpbj_set_matrix(None, 0, None, None, None) == _abi.HPBJ_EINVAL
    assert lib.hpbj_gmres(None, None, None, None, None, None, 0, None, 0) == _abi.HPBJ_EINVAL


def test_struct_layouts(tmp_path):
    """ctypes mirrors of the hpbj.h structs: sizes and field offsets equal the
    C compiler's."""
    import subprocess
    structs = {"hpbj_gmres_opts": _abi.GmresOpts, "hpbj_report": _abi.Report, "hpbj_setup_info": _abi.SetupInfo,
               "hpbj_history_point": _abi.HistoryPoint, "hpbj_kernel_stat": _abi.KernelStat}
    src = ["#include <stdio.h>", "#include <stddef.h>", '#include "hpbj.h"', "int main(void) {"]
    for cname, py in structs.items():
        src.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            src.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    src.append("return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I" + os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True,
                                                    check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)
