"""In-tree build of libqlra_cuda.so (sm_100a) -- the product's native library.

    python -m paper_2404_14783_b200.build        # or __graft_entry__.build()

Compiles every csrc/*.cu with nvcc for `-gencode arch=compute_100a,code=sm_100a`
(cross-compiles on a GPU-less host) and links NCCL from the torch-bundled
nvidia-nccl wheel (the same libnccl.so.2 torch loads, so one NCCL per process).
Incremental: objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libqlra_cuda.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_LIB = "/usr/local/cuda/lib64"


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    nvcc = _nvcc()
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_mtime = max((os.path.getmtime(h) for h in headers), default=0.0)
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                    "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_inc,
                    "-Xptxas", "-v" if verbose else "-O3"]
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
            continue
        cmd = [nvcc, "-c", src, "-o", obj] + flags
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    newest = max(os.path.getmtime(o) for o in objs)
    if not (os.path.exists(LIB) and os.path.getmtime(LIB) >= newest):
        cmd = [nvcc, "-shared", "-o", LIB] + objs + ARCH + [
            "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}", "-lcudart",
            # cuBLASLt: the int8 engine's batched IMMA GEMMs (ozaki.cu)
            "-L", CUDA_LIB, "-lcublasLt", "-Xlinker", f"-rpath={CUDA_LIB}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
