"""The C++ drop-in header (include/qgemm_b200.hpp) compiles as C++20 against
the C ABI (CPU), and its reference-style parity program passes on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_0803_1975_b200", "_lib")
SRC = os.path.join(ROOT, "tests", "cpp", "shim_parity.cpp")
EXE = os.path.join(ROOT, "build", "shim_parity")


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", EXE,
                    "-L", LIBDIR, "-lqgemm_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_shim_compiles_and_links():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_shim_parity_on_gpu():
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all passed" in out.stdout
