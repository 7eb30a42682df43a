"""The product's multi-rank code path on one GPU: 2 and 4
ranks, one host thread and Context each, joined by the in-process
communicator (qlra_group_t) -- the same sharded code NCCL drives across GPUs:
row shards of A with their global row0, the rank's own Psi column slice,
all-reduced W, Grams, Psi H and residual norms, replicated small
factorisations.  The sharded one-pass must reproduce the 1-rank result:
Y (concatenated shards) and W to 1e-13, the QB error to 1e-10 relative, the
range of H (concatenated) to a principal angle <= 1e-8, and X must be
bit-identical on every rank."""
import threading

import numpy as np
import pytest
import torch

from tests.helpers import largest_principal_angle, rel_diff

pytestmark = pytest.mark.gpu


def host(t):
    return t.detach().cpu().numpy()


def run_ranks(nranks, fn):
    """fn(rank, ctx) on `nranks` threads, each with its own CUDA stream and a
    Context attached to one LocalGroup; returns the per-rank results."""
    from paper_2404_14783_b200 import qlra as Q
    group = Q.LocalGroup(nranks)
    out, errs = [None] * nranks, []

    def body(r):
        ctx = None
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = Q.Context(0, r, nranks, local_group=group)
                out[r] = fn(r, ctx)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))
        finally:
            if ctx is not None:
                ctx.close()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    group.close()
    if errs:
        raise errs[0][1]
    return out


@pytest.mark.parametrize("cfg_name,nranks,method", [("C1", 2, 0), ("C1", 4, 0), ("C1", 2, 1), ("C1", 4, 1),
                                                    ("C2", 2, 0), ("C2", 4, 0), ("C2", 4, 1)])
def test_sharded_one_pass_equals_single_rank(ctx, cfg_name, nranks, method):
    from paper_2404_14783_b200 import configs, qlra as Q
    cfg = configs.CONFIGS[cfg_name]
    a = configs.build_matrix(cfg, ctx=ctx)
    opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method)
    one = Q.one_pass_qb(a, opts, ctx=ctx)
    torch.cuda.synchronize()

    def rank_fn(r, c):
        r0, r1 = Q.shard_rows(cfg.m, nranks, r)
        ar = a[:, r0:r1].contiguous()
        res = Q.one_pass_qb(ar, opts, ctx=c, row0=r0, m_global=cfg.m)
        return dict(r0=r0, y=host(res.state.y), w=host(res.state.w), h=host(res.qb.h), x=host(res.qb.x),
                    err=res.qb_residual / res.a_fro, steps=res.qb.report.correction_steps_used,
                    kappa=res.qb.report.kappa_before)

    outs = run_ranks(nranks, rank_fn)
    y = np.concatenate([o["y"] for o in outs], axis=1)
    h = np.concatenate([o["h"] for o in outs], axis=1)
    assert rel_diff(y, host(one.state.y)) < 1e-13
    for o in outs:
        assert rel_diff(o["w"], host(one.state.w)) < 1e-13
        assert np.array_equal(o["w"], outs[0]["w"])  # replicated: bit-identical on every rank
        assert np.array_equal(o["x"], outs[0]["x"])
        assert o["err"] == outs[0]["err"] and o["steps"] == outs[0]["steps"]
    err1 = one.qb_residual / one.a_fro
    print(f"{cfg_name} x{nranks} method {method}: QB err sharded {outs[0]['err']:.15e} single {err1:.15e} "
          f"kappa {outs[0]['kappa']:.6e} vs {one.qb.report.kappa_before:.6e}")
    assert abs(outs[0]["err"] / err1 - 1) <= 1e-10
    assert outs[0]["steps"] == one.qb.report.correction_steps_used
    assert largest_principal_angle(h, host(one.qb.h)) <= 1e-8


def test_collective_order_and_sizes_checked(ctx):
    """A collective whose sizes differ across ranks is an error on every rank,
    not a hang or a silent partial sum."""
    from paper_2404_14783_b200 import qlra as Q

    def rank_fn(r, c):
        w = Q.qzeros(3 + r, 5)
        st = Q.SketchState(Q.qzeros(2, 2), w, Q.TestMatrixSpec(), Q.TestMatrixSpec(), 1, 1, 1)
        with pytest.raises(Q.DeviceError):
            Q.sketch_allreduce(st, c)
        return True

    assert all(run_ranks(2, rank_fn))


def test_group_allreduce_sums_in_rank_order(ctx):
    from paper_2404_14783_b200 import qlra as Q
    eps = 2.0 ** -53
    vals = [1.0, eps, eps, -1.0]

    def rank_fn(r, c):
        w = Q.qzeros(7, 9)
        w.fill_(vals[r])
        w[2, 3, 4] = r + 0.5
        st = Q.SketchState(Q.qzeros(2, 2), w, Q.TestMatrixSpec(), Q.TestMatrixSpec(), 1, 1, 1)
        Q.sketch_allreduce(st, c)
        return host(w)

    outs = run_ranks(4, rank_fn)
    # rank order: ((1 + e) + e) - 1 = 0 exactly (each + e rounds back to 1);
    # any other order that adds the two e first gives 2^-52
    expect = ((vals[0] + vals[1]) + vals[2]) + vals[3]
    assert expect == 0.0
    for o in outs:
        assert np.array_equal(o, outs[0])
        assert o[0, 0, 0] == expect
        assert o[2, 3, 4] == 0.5 + 1.5 + 2.5 + 3.5
