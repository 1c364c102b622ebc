"""The C++ mirror header (include/vmt19937_b200.hpp) over the C ABI:
tests/cpp/acceptance_b200.cpp compiles against it on CPU and passes every
criterion on the GPU."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "acceptance_b200.cpp")
LIBDIR = os.path.join(ROOT, "paper_2309_16682_b200")


def build(out):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ unavailable")
    cmd = [gxx, "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR,
           "-l:libvmt19937_b200.so", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_header_compiles(tmp_path):
    build(str(tmp_path / "acc"))


@pytest.mark.gpu
def test_cpp_acceptance_on_gpu(tmp_path):
    exe = build(str(tmp_path / "acc"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
