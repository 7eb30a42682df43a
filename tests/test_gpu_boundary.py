"""The boundary entries added for the reference's public API
(proj/include/qlra/{sketching,rangefinders}.hpp) and the host-memory paths:
qb_stage_with_psi with an injected Psi, orthonormal_range, pageable host A
(staged through pinned buffers), the QMAT1 file source as one pipeline, and
the error contract of the host-in/host-out call."""
import time

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.helpers import largest_principal_angle, orthonormality_defect, random_gaussian, rel_diff

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def identity(n):
    e = np.zeros((4, n, n))
    e[0][np.arange(n), np.arange(n)] = 1.0
    return e


def test_qb_stage_with_injected_identity_psi_is_exact(ctx):  # test_sketching.cpp:170-183
    from paper_2404_14783_b200 import qlra as Q
    m, n, s, l = 20, 30, 4, 20
    h = O.orthonormal_range(random_gaussian(m, s, 41))
    a = O.qmat_mul(h, random_gaussian(s, n, 42))
    st = Q.empty_sketch(m, n, s, s, l, 1, 2)
    Q.sketch_update(st, dev(a), ctx)
    st.w = dev(a)  # Psi = I implies W = A
    qb = Q.qb_stage_with_psi(st, dev(identity(m)), Q.PSEUDO_SVD, ctx=ctx)
    assert rel_diff(O.qmat_mul(host(qb.h), host(qb.x)), a) < 1e-10
    # the oracle's qb_stage_with_psi on the same inputs
    qo = O.qb_stage(host(st.y), a, 2, O.PSEUDO_SVD, psi=identity(m))
    assert rel_diff(O.qmat_mul(qo["h"], qo["x"]), a) < 1e-10


@pytest.mark.parametrize("method", [0, 1])
def test_qb_stage_with_regenerated_psi_equals_qb_stage(ctx, method):
    """Injecting the Psi the spec generates reproduces qb_stage (HX: the
    basis-independent product)."""
    from paper_2404_14783_b200 import configs, qlra as Q
    cfg = configs.CONFIGS["C1"]
    a = configs.build_matrix(cfg, ctx=ctx)
    st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, ctx=ctx)
    ref = Q.qb_stage(st, method, ctx=ctx)
    psi = Q.gen_test_matrix(Q.TestMatrixSpec(Q.GAUSSIAN, cfg.l, cfg.m, 2, 1.0), ctx)
    got = Q.qb_stage_with_psi(st, psi, method, ctx=ctx)
    assert rel_diff(O.qmat_mul(host(got.h), host(got.x)), O.qmat_mul(host(ref.h), host(ref.x))) < 1e-10
    # the oracle fed the same Y, W and this Psi
    qo = O.qb_stage(host(st.y), host(st.w), 2, method, psi=host(psi))
    r_d, an = Q.residual_fro(a, got.h, got.x, ctx)
    r_o, _ = Q.residual_fro(a, dev(qo["h"]), dev(qo["x"]), ctx)
    assert abs(r_d / r_o - 1) < 1e-10
    with pytest.raises(Q.ShapeError):
        Q.qb_stage_with_psi(st, psi[:, :, :10], method, ctx=ctx)


def test_orthonormal_range_vs_oracle(ctx):  # rangefinders.cpp:160-164
    from paper_2404_14783_b200 import qlra as Q
    y = random_gaussian(90, 12, 7)
    h = host(Q.orthonormal_range(dev(y), ctx=ctx))
    assert orthonormality_defect(h) < 1e-12
    assert largest_principal_angle(h, O.orthonormal_range(y)) < 1e-12
    sq = random_gaussian(6, 6, 8)  # rows == cols is allowed (pseudo_svd refuses it)
    assert orthonormality_defect(host(Q.orthonormal_range(dev(sq), ctx=ctx))) < 1e-12
    with pytest.raises(Q.ParameterError):
        Q.pseudo_svd(dev(sq), ctx=ctx)
    with pytest.raises(Q.ParameterError):
        Q.orthonormal_range(dev(random_gaussian(3, 5, 9)), ctx=ctx)


@pytest.mark.parametrize("method", [0, 1])
def test_one_pass_host_pageable_equals_pinned(ctx, method):
    """A pageable host A (the reference QMatrix's std::vector planes) goes
    through the staged pipeline and gives the pinned path's result."""
    from paper_2404_14783_b200 import configs, qlra as Q
    cfg = configs.CONFIGS["C2"]
    a = configs.build_matrix(cfg, ctx=ctx)
    opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method)
    pinned = a.cpu().pin_memory()
    pageable = a.cpu()
    assert not pageable.is_pinned()
    del a
    r1 = Q.one_pass_qb_host(pinned, opts, ctx=ctx)
    r2 = Q.one_pass_qb_host(pageable, opts, ctx=ctx)
    assert torch.equal(r1.h, r2.h) and torch.equal(r1.x, r2.x)  # same chunks, same arithmetic
    st = Q.make_sketch_host(pageable, cfg.s - 5, cfg.s, cfg.l, 1, 2, ctx=ctx)
    st1 = Q.make_sketch_host(pinned, cfg.s - 5, cfg.s, cfg.l, 1, 2, ctx=ctx)
    assert torch.equal(st.y, st1.y) and torch.equal(st.w, st1.w)


def test_one_pass_host_singular_solve_leaves_no_copy_in_flight(ctx):
    """The core solve raises SingularMatrixError (Psi H rank-deficient: a
    very sparse Psi); the call must not return while its side-stream copy of
    H can still write the caller's buffer, and the context stays usable."""
    from paper_2404_14783_b200 import qlra as Q
    a = dev(random_gaussian(200, 60, 5))
    a_host = a.cpu().pin_memory()
    opts = Q.OnePassOptions(r=5, s=10, l=20, rangefinder=Q.PSEUDO_SVD, embedding=Q.SPARSE_GAUSSIAN,
                            density=2e-4)
    h_out = torch.full((4, 200, 10), 7.0, dtype=torch.float64).pin_memory()
    x_out = torch.zeros((4, 10, 60), dtype=torch.float64).pin_memory()
    with pytest.raises((Q.SingularMatrixError, Q.RankError)) as e:
        Q.one_pass_qb_host(a_host, opts, ctx=ctx, h_out=h_out, x_out=x_out)
    if isinstance(e.value, Q.SingularMatrixError):
        assert "(estimated condition " in str(e.value)
    snap = h_out.clone()
    time.sleep(0.2)
    assert torch.equal(snap, h_out)  # nothing lands after the call returned
    ok = Q.one_pass_qb_host(a_host, Q.OnePassOptions(r=5, s=10, l=20), ctx=ctx)
    assert torch.isfinite(ok.x).all()


def _np_write_qmat(path, a):  # QMAT1 per proj/include/qlra/io.hpp:15-18
    import struct
    with open(path, "wb") as f:
        f.write(b"QMAT1\0" + struct.pack("<QQ", a.shape[1], a.shape[2]))
        f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


@pytest.mark.parametrize("block_rows", [1, 7, 256, 5000])
def test_sketch_from_qmat_file_one_pipeline(ctx, tmp_path, block_rows):
    """The file source (QmatFileSource, io.cpp:213-239) feeds ONE row
    pipeline (Omega built once) for any read granularity; equals the
    in-memory sketch."""
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(700, 90, 31)
    _np_write_qmat(tmp_path / "a.qmat", a)
    n0 = ctx.launch_count()
    st = Q.sketch_from_qmat_file(tmp_path / "a.qmat", 5, 10, 20, 3, 4, block_rows=block_rows, ctx=ctx)
    launches = ctx.launch_count() - n0
    ref = Q.make_sketch(dev(a), 5, 10, 20, 3, 4, ctx=ctx)
    assert rel_diff(host(st.y), host(ref.y)) < 1e-13 and rel_diff(host(st.w), host(ref.w)) < 1e-13
    assert launches < 40, launches  # not one Omega generation per 256-row block
