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


def test_local_group_lifecycle_without_gpu():
    """qlra_group_t is host-side state: creation limits and destruction need no
    device (its contexts do)."""
    L = _lib.lib()
    h = ctypes.c_void_p()
    assert L.qlra_group_create(ctypes.byref(h), 0) == 2  # QLRA_ERR_PARAMETER
    assert L.qlra_group_create(ctypes.byref(h), 17) == 2
    assert L.qlra_group_create(ctypes.byref(h), 4) == 0 and h.value
    assert L.qlra_group_destroy(h) == 0
    assert L.qlra_group_destroy(None) == 0


def _qskt(path, y_shape, w_shape, s, l, truncate=0):
    """A QSKT1 file (io.cpp:116-128) with the given embedded shapes."""
    import struct

    def spec(kind, rows, cols, seed):
        return struct.pack("<IQQQd", kind, rows, cols, seed, 1.0)
    b = b"QSKT1\0" + spec(0, 9, s, 1) + spec(0, l, 9, 2) + struct.pack("<QQQ", 1, s, l)
    for r, c in (y_shape, w_shape):
        b += b"QMAT1\0" + struct.pack("<QQ", r, c) + bytes(32 * r * c)
    with open(path, "wb") as f:
        f.write(b[:len(b) - truncate] if truncate else b)


def test_sketch_file_dims_validates_before_allocating(tmp_path):
    """read_sketch sizes Y and W from their own QMAT1 headers and applies the
    reference's consistency test (io.cpp:130-145) -- no device, no context."""
    L = _lib.lib()
    dims = (ctypes.c_int64 * 4)()
    p = tmp_path / "ok.qskt"
    _qskt(p, (9, 3), (6, 9), 3, 6)
    assert L.qlra_sketch_file_dims(str(p).encode(), dims) == 0 and list(dims) == [9, 3, 6, 9]
    # y rows need not equal the Psi spec's cols (the reference reads headers)
    _qskt(p, (5, 3), (6, 9), 3, 6)
    assert L.qlra_sketch_file_dims(str(p).encode(), dims) == 0 and dims[0] == 5
    _qskt(p, (9, 4), (6, 9), 3, 6)  # y.cols != s
    assert L.qlra_sketch_file_dims(str(p).encode(), dims) == 6  # QLRA_ERR_IO
    _qskt(p, (9, 3), (6, 9), 3, 6, truncate=40)
    assert L.qlra_sketch_file_dims(str(p).encode(), dims) == 6
    with open(p, "r+b") as f:  # absurd header: huge rows -> IoError, not an allocation
        import struct
        _qskt(p, (9, 3), (6, 9), 3, 6)
        f.seek(6 + 72 + 24 + 6)
        f.write(struct.pack("<Q", 1 << 60))
    assert L.qlra_sketch_file_dims(str(p).encode(), dims) == 6


def test_residue_gemm_kernel_is_tcgen05_and_tma():
    """The int8 engine's residue GEMM (csrc/i8gemm.cu) is the repo's own
    tcgen05 kernel: its sm_100a SASS holds the int8 UMMA (UTCIMMA, 1-CTA and
    .2CTA), TMA loads (UTMALDG), TMA stores and reduce-adds (UTMASTG /
    UTMAREDG.ADD), TMEM loads (LDTM) and tcgen05.commit (UTCBAR) -- checked
    on the object nvcc built here, no GPU needed."""
    import shutil
    import subprocess
    build.build()
    obj = os.path.join(build.BUILD, "i8gemm.cu.o")
    assert os.path.exists(obj)
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([cuobjdump, "-sass", obj], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in sass
    for mnemonic in ("UTCIMMA", "UTCIMMA.2CTA", "UTMALDG.3D", "UTMASTG.3D", "UTMAREDG.3D.ADD", "LDTM.x32",
                     "UTCBAR", "UTCBAR.2CTA.MULTICAST", "SYNCS.PHASECHK.TRANS64.TRYWAIT"):
        assert mnemonic in sass, mnemonic
