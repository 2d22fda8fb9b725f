"""The C++ facade (include/asyncdiff_b200.hpp) compiles against the C ABI and
drives it the way the reference's own C++ callers do."""
import os
import subprocess

import pytest

from paper_2406_06911_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "facade_demo.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "build", "facade_demo")


def build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    libdir = os.path.dirname(_lib.SO_PATH)
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(os.path.getmtime(SRC), os.path.getmtime(_lib.SO_PATH)):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), SRC, "-o", EXE,
                               f"-L{libdir}", "-l:libasyncdiff_b200.so", f"-Wl,-rpath,{libdir}"])
    return EXE


def test_facade_host_mode():
    out = subprocess.run([build(), "host"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host ok" in out.stdout


@pytest.mark.gpu
def test_facade_gpu_golden():
    out = subprocess.run([build(), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
