"""Command-line front end on the GPU path -- the `sketch`, `update` and
`approx` subcommands of the reference CLI (proj/tools/qlra_main.cpp:103-208,
445-477), with the same flags, defaults, seeds and CSV report, reading and
writing the reference's QMAT1 / QSKT1 files (io.cpp:77-145).  `synth`,
`verify` and `compress-image` (planted-spectrum generators, Monte-Carlo
suites, image I/O) are outside the hot path (DESIGN 7).

    python -m paper_2404_14783_b200.cli sketch --input A.qmat -r 10 --out A.qskt
    python -m paper_2404_14783_b200.cli update --sketch A.qskt --input D.qmat --row0 0 --out A2.qskt
    python -m paper_2404_14783_b200.cli approx --input A.qmat -r 10 --rangefinder both
    python -m paper_2404_14783_b200.cli approx --sketch A.qskt -r 10

Every subcommand fails like the reference's: "error: <what>" on stderr and
exit status 2 (qlra_main.cpp:502-512).
"""
from __future__ import annotations

import argparse
import math
import sys

APPROX_CSV_HEADER = ("rank,rangefinder,seed,rel_error,qb_residual,kappa_h,correction_steps,"
                     "t_sketch_s,t_rangefinder_s,t_solve_s,t_truncate_s")


def _kind(Q, name):
    # test_matrix_kind_from_string (sketching.cpp:90-96)
    kinds = {"gaussian": Q.GAUSSIAN, "rademacher": Q.RADEMACHER, "sparse-gaussian": Q.SPARSE_GAUSSIAN,
             "sparse-rademacher": Q.SPARSE_RADEMACHER}
    if name not in kinds:
        raise Q.ParameterError("unknown embedding kind: " + name)
    return kinds[name]


def _methods(Q, name):
    if name == "both":
        return [Q.PSEUDO_QR, Q.PSEUDO_SVD]
    if name == "pseudo-qr":
        return [Q.PSEUDO_QR]
    if name == "pseudo-svd":
        return [Q.PSEUDO_SVD]
    raise Q.ParameterError("unknown rangefinder: " + name)


def _method_name(Q, m):
    return "pseudo-qr" if m == Q.PSEUDO_QR else "pseudo-svd"


def _fmt(v):
    if v is None or (isinstance(v, float) and math.isnan(v)):
        return "nan"
    return f"{v:.12g}" if isinstance(v, float) else str(v)


def _emit(os_, Q, rank, method, seed, res):
    d = res.diagnostics
    t = d["times"]
    os_.write(",".join([str(rank), _method_name(Q, method), str(seed), _fmt(d["relative_error"]),
                        _fmt(d["qb_residual"]), _fmt(float(d["kappa_h"])), str(d["correction_steps"]),
                        _fmt(float(t["sketch_s"])), _fmt(float(t["rangefinder_s"])),
                        _fmt(float(t["solve_s"])), _fmt(float(t["truncate_s"]))]) + "\n")


def run_sketch(a, Q):
    """run_sketch (qlra_main.cpp:103-115): s = r + 5, l = 2 s, seeds (seed,
    seed + 1); A streams from the file through the device pipeline."""
    s = a.rank + 5 if a.sketch_s < 0 else a.sketch_s
    l = 2 * s if a.sketch_l < 0 else a.sketch_l
    st = Q.sketch_from_qmat_file(a.input, a.rank, s, l, a.seed, a.seed + 1, _kind(Q, a.embedding), a.density,
                                 a.block_rows)
    Q.write_sketch(a.out, st)
    sys.stderr.write(f"sketched {st.y.shape[1]}x{st.w.shape[2]} -> Y {st.y.shape[1]}x{st.y.shape[2]}, "
                     f"W {st.w.shape[1]}x{st.w.shape[2]}\n")
    return 0


def run_update(a, Q):
    """run_update (qlra_main.cpp:117-133): row-block update with --row0,
    additive full-shape update without."""
    st = Q.read_sketch(a.sketch)
    block = Q.read_qmat(a.input)
    if a.row0 < 0:
        Q.sketch_update(st, block)
    else:
        Q.sketch_update_rows(st, a.row0, block)
    Q.write_sketch(a.out, st)
    return 0


def run_approx(a, Q):
    """run_approx (qlra_main.cpp:152-208)."""
    if (a.input is None) == (a.sketch is None):
        raise Q.ParameterError("approx: pass exactly one of --input or --sketch")
    os_ = open(a.out, "w") if a.out else sys.stdout
    try:
        os_.write(APPROX_CSV_HEADER + "\n")
        methods = _methods(Q, a.rangefinder)
        if a.sketch is not None:
            # one-pass from a checkpoint: the data matrix is never opened
            st = Q.read_sketch(a.sketch)
            for rank in a.rank:
                for m in methods:
                    o = Q.OnePassOptions(r=rank, rangefinder=m, rangefinder_seed=a.seed)
                    _emit(os_, Q, rank, m, a.seed, Q.one_pass_approx_from_sketch(st, o))
            return 0
        mat = Q.read_qmat(a.input)
        for rank in a.rank:
            for m in methods:
                for t in range(a.trials):
                    seed = a.seed + 2 * t
                    o = Q.OnePassOptions(r=rank, s=a.sketch_s, l=a.sketch_l, rangefinder=m,
                                         embedding=_kind(Q, a.embedding), density=a.density, omega_seed=seed,
                                         psi_seed=seed + 1, rangefinder_seed=seed)
                    _emit(os_, Q, rank, m, seed, Q.one_pass_approx(mat, o))
        return 0
    finally:
        if os_ is not sys.stdout:
            os_.close()


def parser():
    p = argparse.ArgumentParser(prog="qlra-gpu", description="one-pass quaternion LRA on the GPU")
    sub = p.add_subparsers(dest="cmd", required=True)
    sk = sub.add_parser("sketch", help="build a two-sketch checkpoint from a matrix file")
    sk.add_argument("--input", required=True)
    sk.add_argument("--rank", "-r", type=int, required=True)
    sk.add_argument("--sketch-s", type=int, default=-1)
    sk.add_argument("--sketch-l", type=int, default=-1)
    sk.add_argument("--embedding", default="gaussian")
    sk.add_argument("--density", type=float, default=0.1)
    sk.add_argument("--seed", type=int, default=1)
    sk.add_argument("--block-rows", type=int, default=256)
    sk.add_argument("--out", required=True)
    up = sub.add_parser("update", help="fold a linear update into a sketch checkpoint")
    up.add_argument("--sketch", required=True)
    up.add_argument("--input", required=True, help="update block (QMAT1)")
    up.add_argument("--row0", type=int, default=-1, help="first row of a row-block update; omit for additive")
    up.add_argument("--out", required=True)
    ap = sub.add_parser("approx", help="one-pass rank-r approximation")
    ap.add_argument("--input", default=None, help="data matrix (QMAT1)")
    ap.add_argument("--sketch", default=None, help="sketch checkpoint (QSKT1)")
    ap.add_argument("--rank", "-r", type=int, nargs="+", required=True)
    ap.add_argument("--sketch-s", type=int, default=-1)
    ap.add_argument("--sketch-l", type=int, default=-1)
    ap.add_argument("--rangefinder", default="pseudo-qr", help="pseudo-qr|pseudo-svd|both")
    ap.add_argument("--embedding", default="gaussian")
    ap.add_argument("--density", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--trials", type=int, default=1)
    ap.add_argument("--out", default=None, help="CSV report path (default stdout)")
    p.add_argument("--device", type=int, default=0)
    return p


def main(argv=None):
    a = parser().parse_args(argv)
    from paper_2404_14783_b200 import qlra as Q
    Q.set_default_context(Q.Context(a.device))
    try:
        return {"sketch": run_sketch, "update": run_update, "approx": run_approx}[a.cmd](a, Q)
    except Q.Error as e:  # qlra_main.cpp:508-511
        sys.stderr.write(f"error: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
