"""GPU CLI (paper_2404_14783_b200/cli.py) against the oracle: the reference
CLI's sketch / update / approx workflows (qlra_main.cpp:103-208) on QMAT1 /
QSKT1 files."""
import csv
import io
import struct

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import random_gaussian, rel_diff


def _write_qmat(path, a):  # QMAT1 per proj/include/qlra/io.hpp:15-18
    with open(path, "wb") as f:
        f.write(b"QMAT1\0" + struct.pack("<QQ", a.shape[1], a.shape[2]))
        f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def _read_sketch_np(path):  # QSKT1 per io.hpp:20-44
    b = open(path, "rb").read()
    assert b[:6] == b"QSKT1\0"
    off = 6 + 2 * (4 + 8 * 4) + 3 * 8
    mats = []
    for _ in range(2):
        assert b[off:off + 6] == b"QMAT1\0"
        r, c = struct.unpack("<QQ", b[off + 6:off + 22])
        off += 22
        mats.append(np.frombuffer(b[off:off + 32 * r * c], dtype="<f8").reshape(4, r, c))
        off += 32 * r * c
    return mats


def test_cli_parser_accepts_reference_flags():
    from paper_2404_14783_b200 import cli
    a = cli.parser().parse_args(["approx", "--input", "A.qmat", "-r", "5", "10", "--rangefinder", "both",
                                 "--embedding", "sparse-gaussian", "--density", "0.2", "--trials", "2"])
    assert a.rank == [5, 10] and a.trials == 2 and a.sketch_s == -1
    a = cli.parser().parse_args(["sketch", "--input", "A.qmat", "-r", "3", "--out", "s.qskt"])
    assert a.block_rows == 256 and a.seed == 1
    a = cli.parser().parse_args(["update", "--sketch", "s", "--input", "d", "--out", "o"])
    assert a.row0 == -1


@pytest.mark.gpu
def test_cli_sketch_update_approx(ctx, tmp_path, capsys):
    from paper_2404_14783_b200 import cli
    a = random_gaussian(300, 120, 61)
    _write_qmat(tmp_path / "A.qmat", a)
    # sketch: s = r + 5, l = 2 s, seeds (seed, seed + 1) -- qlra_main.cpp:104-108
    assert cli.main(["sketch", "--input", str(tmp_path / "A.qmat"), "-r", "5", "--seed", "7",
                     "--block-rows", "64", "--out", str(tmp_path / "A.qskt")]) == 0
    y, w = _read_sketch_np(tmp_path / "A.qskt")
    yo, wo = O.make_sketch(a, 5, 10, 20, 7, 8)
    assert rel_diff(y, yo) < 1e-13 and rel_diff(w, wo) < 1e-13
    # update: additive delta of the full shape equals sketching A + D
    d = random_gaussian(300, 120, 62)
    _write_qmat(tmp_path / "D.qmat", d)
    assert cli.main(["update", "--sketch", str(tmp_path / "A.qskt"), "--input", str(tmp_path / "D.qmat"),
                     "--out", str(tmp_path / "AD.qskt")]) == 0
    y2, w2 = _read_sketch_np(tmp_path / "AD.qskt")
    yo2, wo2 = O.make_sketch(a + d, 5, 10, 20, 7, 8)
    assert rel_diff(y2, yo2) < 1e-13 and rel_diff(w2, wo2) < 1e-13
    # approx from the matrix and from the checkpoint: CSV with the reference header
    out = tmp_path / "r.csv"
    assert cli.main(["approx", "--input", str(tmp_path / "A.qmat"), "-r", "5", "--rangefinder", "both",
                     "--out", str(out)]) == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert [r["rangefinder"] for r in rows] == ["pseudo-qr", "pseudo-svd"]
    assert all(0.0 < float(r["rel_error"]) < 1.5 for r in rows)
    assert cli.main(["approx", "--sketch", str(tmp_path / "A.qskt"), "-r", "5"]) == 0
    printed = capsys.readouterr().out.splitlines()
    assert printed[0] == cli.APPROX_CSV_HEADER and printed[1].split(",")[3] == "nan"
    # exactly one of --input / --sketch; failures print "error: <what>" and
    # exit 2 (qlra_main.cpp:508-511)
    assert cli.main(["approx", "-r", "5"]) == 2
    assert capsys.readouterr().err.startswith("error: approx: pass exactly one of --input or --sketch")
    # t_solve_s is measured (the rangefinder and the solve are timed apart)
    assert all(float(r["t_solve_s"]) > 0.0 for r in rows)
