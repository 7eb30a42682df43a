"""The C++ facade (include/qlra_gpu.hpp) compiles with g++ against the C-ABI
library without a GPU; on a GPU it runs the reference's one-pass flow."""
import os
import subprocess
import sysconfig

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path):
    from paper_2404_14783_b200 import build
    lib = build.build()
    nccl_inc, _ = build._nccl_dirs()
    exe = str(tmp_path / "facade_demo")
    cmd = ["g++", "-std=c++17", "-O2", os.path.join(ROOT, "examples", "facade_demo.cpp"), "-o", exe,
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-I", nccl_inc,
           lib, f"-Wl,-rpath,{os.path.dirname(lib)}", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_facade_runs_one_pass(tmp_path):
    exe = _compile(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "rel_error=" in out.stdout
