"""The C++ drop-in shim (include/difform_b200.hpp): compiles here against the
C-ABI; on the GPU box the compiled test program runs reference-style calls."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
PKG = os.path.join(ROOT, "paper_2404_01249_b200")


def build(tmp_path):
    exe = str(tmp_path / "shim_test")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-I",
                           os.path.join(ROOT, "include"), SRC, "-o", exe, "-L", PKG,
                           "-ldifform_cuda", "-Wl,-rpath," + PKG])
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shim_runs_on_device(tmp_path):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
