"""The C++ facade (include/qlra_gpu.hpp) compiles with g++ against the C-ABI
library without a GPU -- with its own copy of the reference's error types, and
(where the reference's headers exist, i.e. in the build container) against
the reference's own proj/include/qlra/errors.hpp, so a reference caller's
catch (const qlra::RankError&) sees the GPU path's errors.  On a GPU the demo
runs the reference's one-pass flow end to end (sketch, QB stage, truncation,
sketch_from_source, qb_stage_with_psi, orthonormal_range, host in/out)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INCLUDE = "/root/reference/proj/include"


def _compile(tmp_path, extra_include=None, name="facade_demo"):
    from paper_2404_14783_b200 import build
    lib = build.build()
    nccl_inc, _ = build._nccl_dirs()
    exe = str(tmp_path / name)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", os.path.join(ROOT, "examples", "facade_demo.cpp"),
           "-o", exe, "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-I", nccl_inc]
    if extra_include:
        cmd += ["-I", extra_include]
    cmd += [lib, f"-Wl,-rpath,{os.path.dirname(lib)}", "-L/usr/local/cuda/lib64", "-lcudart",
            "-Wl,-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers only in the build container")
def test_facade_compiles_against_reference_errors_hpp(tmp_path):
    """With the reference's include tree on the path the facade uses
    qlra/errors.hpp itself (one definition of qlra::RankError & co.)."""
    src = tmp_path / "both.cpp"
    src.write_text('#include <qlra/errors.hpp>\n#include "qlra_gpu.hpp"\n'
                   'static_assert(std::is_base_of<qlra::Error, qlra::gpu::DeviceError>::value, "");\n'
                   'int main() { try { throw qlra::SingularMatrixError("x", 2.0); }\n'
                   '  catch (const qlra::Error& e) { return std::string(e.what()) == '
                   '"x (estimated condition 2.000000)" ? 0 : 1; } }\n')
    from paper_2404_14783_b200 import build
    nccl_inc, _ = build._nccl_dirs()
    exe = str(tmp_path / "both")
    subprocess.run(["g++", "-std=c++17", str(src), "-o", exe, "-I", REF_INCLUDE, "-I",
                    os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-I", nccl_inc], check=True)
    assert subprocess.run([exe]).returncode == 0
    assert os.path.exists(_compile(tmp_path, REF_INCLUDE, "facade_demo_ref"))


@pytest.mark.gpu
def test_facade_runs_one_pass(tmp_path):
    exe = _compile(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "rel_error=" in out.stdout and "ok=1" in out.stdout
