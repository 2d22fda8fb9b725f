"""The C++ facade (include/asyncdiff_b200.hpp) compiles against the C ABI and
drives it the way the reference's own C++ callers do: tests/cpp/run_one.cpp is
the reference's run_one (experiment.cpp:238-290) with only the namespace
switched; tests/cpp/vec_adapter.cpp uses a non-std vector type (the Eigen
adapter's contract); tests/cpp/facade_demo.cpp is the minimal caller."""
import os
import subprocess

import pytest

from paper_2406_06911_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(name):
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    exe = os.path.join(ROOT, "tests", "cpp", "build", name)
    hdr = os.path.join(ROOT, "include", "asyncdiff_b200.hpp")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    libdir = os.path.dirname(_lib.SO_PATH)
    if not os.path.exists(exe) or os.path.getmtime(exe) < max(os.path.getmtime(src), os.path.getmtime(hdr),
                                                               os.path.getmtime(_lib.SO_PATH)):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                               src, "-o", exe, f"-L{libdir}", "-l:libasyncdiff_b200.so", f"-Wl,-rpath,{libdir}"])
    return exe


@pytest.mark.parametrize("name", ["facade_demo", "run_one", "vec_adapter"])
def test_facade_host_mode(name):
    out = subprocess.run([build(name), "host"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok" in out.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["facade_demo", "run_one", "vec_adapter"])
def test_facade_gpu(name):
    out = subprocess.run([build(name), "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    print(out.stdout)
