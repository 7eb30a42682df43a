"""World-size-2 CPU (gloo) test of the multi-GPU decomposition: each rank owns
the row shard given by the product's shard_rows, computes its partial sketch
and Gram / Psi*H partials (CPU oracle standing in for the device kernels),
and the all-reduced results equal the monolithic ones."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_14783_b200.qlra import shard_rows
    m, n, s, l = 37, 23, 4, 8
    a = O.random_gaussian(m, n, 99)
    r0, r1 = shard_rows(m, world, rank)
    y = np.zeros((4, m, s))
    w = np.zeros((4, l, n))
    O.sketch_update_rows(y, w, r0, np.ascontiguousarray(a[:, r0:r1]), 5, 6)
    wt = torch.from_numpy(w)
    dist.all_reduce(wt)                               # qlra_sketch_allreduce
    h = y[:, r0:r1]                                   # local rows of Y (stand-in for H)
    g = torch.from_numpy(O.qmat_mul(O.adjoint(h), h))
    dist.all_reduce(g)                                # Gram all-reduce
    psi = O.gen_block(O.GAUSSIAN, l, m, 6, 0, l, r0, r1)  # rank's Psi column slice
    ph = torch.from_numpy(O.qmat_mul(psi, np.ascontiguousarray(h)))
    dist.all_reduce(ph)                               # Psi H all-reduce
    if rank == 0:
        out.put((wt.numpy(), g.numpy(), ph.numpy()))
    # every rank holds a distinct, covering, ordered row range
    rng = torch.tensor([r0, r1])
    allr = [torch.zeros(2, dtype=rng.dtype) for _ in range(world)]
    dist.all_gather(allr, rng)
    if rank == 0:
        out.put([tuple(x.tolist()) for x in allr])
    dist.destroy_process_group()


def test_row_sharded_reductions_equal_monolithic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    w, g, ph = q.get(timeout=120)
    ranges = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m, n, s, l = 37, 23, 4, 8
    a = O.random_gaussian(m, n, 99)
    y_full, w_full = O.make_sketch(a, 2, s, l, 5, 6)
    assert np.allclose(w, w_full, rtol=1e-13, atol=1e-13)
    assert np.allclose(g, O.qmat_mul(O.adjoint(y_full), y_full), rtol=1e-12, atol=1e-12)
    psi = O.gen_test_matrix(O.GAUSSIAN, l, m, 6)
    assert np.allclose(ph, O.qmat_mul(psi, y_full), rtol=1e-12, atol=1e-12)
    assert ranges[0][0] == 0 and ranges[-1][1] == m
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))

