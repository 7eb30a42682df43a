"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU and exports every symbol include/qlra_cuda.h declares (no compute calls)."""
import ctypes
import os

from paper_2404_14783_b200 import _lib, build


def test_library_builds_and_exports_every_header_symbol():
    path = build.build()
    assert os.path.exists(path)
    lib = ctypes.CDLL(path)
    names = _lib.exported_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_header_is_plain_c():
    import re
    hdr = open(os.path.join(os.path.dirname(build.HERE), "include", "qlra_cuda.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    for forbidden in ("torch", "std::", "template", "class "):
        assert forbidden not in hdr


def test_kernel_name_without_gpu():
    assert _lib.lib().qlra_sketch_kernel_name().decode()
