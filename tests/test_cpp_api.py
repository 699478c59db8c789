"""The C++ mirror API (include/bjgmres_b200.hpp) drives libhpbj.so like the
reference's own tests drive the reference library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2509_09139_b200", "lib")
EXE = os.path.join(ROOT, "paper_2509_09139_b200", "build_obj", "test_api")


def build_exe():
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(os.path.getmtime(SRC), os.path.getmtime(
            os.path.join(ROOT, "include", "bjgmres_b200.hpp"))):
        subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), SRC, "-L" + LIBDIR,
                        "-lhpbj", "-Wl,-rpath," + LIBDIR, "-o", EXE], check=True)
    return EXE


def test_cpp_api_compiles():
    assert os.path.exists(build_exe())


@pytest.mark.gpu
def test_cpp_api_reference_scenarios():
    r = subprocess.run([build_exe()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
